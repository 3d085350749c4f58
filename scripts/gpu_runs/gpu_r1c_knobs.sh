for env in "X=1" "DPK_PDL=1" "DPK_LEAF_W=8" "DPK_DYN=0"; do
echo "== $env"
env $env SPD_ONLY=4608 timeout 120 python scripts/inv_factor_one.py 20 2>&1 | tail -1
env $env timeout 120 python scripts/inv_factor_one.py 20 2>&1 | tail -1
env $env timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bk.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bk.json')); print('bench', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3))"
done
timeout 300 python scripts/host_profile.py 2>&1 | head -4
