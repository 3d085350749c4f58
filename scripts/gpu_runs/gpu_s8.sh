python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python scripts/inv_one.py
DPK_PDL=0 python scripts/inv_one.py
python scripts/ts_group.py
DPK_PDL=0 python scripts/ts_group.py
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'])"
