python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python scripts/gemm_one.py 4608 4608 4608 tf32
python scripts/gemm_one.py 8192 8192 8192 tf32
python scripts/gemm_one.py 8192 8192 8192 3xtf32
python scripts/gemm_one.py 4608 4608 4608 3xtf32
python scripts/kbench.py 2>&1 | head -18
python scripts/spd_bench.py
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'])"
