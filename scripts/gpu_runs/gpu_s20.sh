python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python scripts/host_time.py 2>&1 | head -6
python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['ms_per_step_serialized'], d['stages_ms'], d['e2e']['ms_per_iter'])"
