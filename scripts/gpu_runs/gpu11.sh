timeout 600 python -m pytest tests -q -m gpu --tb=short -k "tapmajor or tap_major or channels_last or pack_unpack" 2>&1 | tail -25
python scripts/prof_step.py --profiled 3 2>&1 | tail -2
python scripts/prof_step.py --profiled 3 --nchw 2>&1 | tail -2
