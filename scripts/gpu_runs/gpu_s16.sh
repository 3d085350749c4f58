python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python scripts/syrk_one.py 4608 1568 k
python scripts/syrk_one.py 576 100352 k
python scripts/syrk_one.py 576 100352 mn
python scripts/syrk_one.py 1152 25088 mn
python scripts/syrk_one.py 147 401408 mn
python scripts/spd_bench.py | head -1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['ms_per_step_serialized'], d['stages_ms'])"
