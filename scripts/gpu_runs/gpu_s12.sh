python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python scripts/spd_bench.py
SPD_ONLY=4608 python scripts/spd_bench.py | head -1
python scripts/inv_one.py
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/inv_launches3.csv python scripts/inv_one.py 1 > /dev/null 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'])"
