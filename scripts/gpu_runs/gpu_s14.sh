python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python scripts/kbench.py 2>&1 | sed -n 9,18p
DPK_MN3=0 python scripts/kbench.py 2>&1 | sed -n 9,18p
python scripts/spd_bench.py | head -1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['ms_per_step_serialized'], d['stages_ms'])"
