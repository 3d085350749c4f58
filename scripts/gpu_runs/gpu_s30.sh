python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python scripts/overlap_probe.py 2>&1 | tail -14
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['ms_per_step_serialized'], d['stages_ms'])"
