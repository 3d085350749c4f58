timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 120 python scripts/gemm_one.py 4608 4608 4608 tf32
timeout 120 python scripts/gemm_one.py 8192 8192 8192 tf32
timeout 120 env DPK_DYN=0 python scripts/gemm_one.py 4608 4608 4608 tf32
timeout 120 python scripts/gemm_one.py 4608 4608 4608 3xtf32
timeout 120 env DPK_DYN=0 python scripts/gemm_one.py 4608 4608 4608 3xtf32
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['ms_per_step_serialized'], d['stages_ms'])"
