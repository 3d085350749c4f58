timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 120 python scripts/gemm_one.py 4608 4608 4608 tf32
timeout 120 python scripts/syrk_one.py 576 100352 mn
timeout 120 env DPK_DYN=0 python scripts/syrk_one.py 576 100352 mn
timeout 120 python scripts/inv_factor_one.py
timeout 120 env DPK_DYN=0 python scripts/inv_factor_one.py
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['ms_per_step_serialized'], d['stages_ms'])"
timeout 300 env DPK_DYN=0 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['ms_per_step_serialized'], d['stages_ms'])"
