mkdir -p gpurun_out/r32
DPK_PROFILE_TIMED=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r32/launches.csv python bench.py --model resnet32 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r32/ncu_launch.log 2>&1; echo "rc=$?"
python scripts/launch_summary.py gpurun_out/r32/launches.csv | head -30
python - <<'PY'
import torch, sys
sys.path.insert(0, '.')
import bench_models as BM
m = BM.WORKLOADS['resnet32'][0]()
geom = BM.layer_geometry(m, BM.WORKLOADS['resnet32'][2], BM.WORKLOADS['resnet32'][1])
for g in geom: print(g)
PY
