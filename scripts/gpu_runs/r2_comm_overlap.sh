# comm_overlap (bucketed reduce-scatter from the backward hooks): tests, P=2 parity, N=2 e2e
mkdir -p gpurun_out/co
python -m pytest tests/test_gpu_dpkfac.py -x -q -k "comm_overlap or early" 2>&1 | tail -5
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 \
  scripts/multi_gpu_parity.py > gpurun_out/co/parity_p2.log 2>&1; tail -2 gpurun_out/co/parity_p2.log
for co in "" "--comm-overlap" "--comm-overlap --bucket-mb 4" "--comm-overlap --early"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 \
    bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline $co 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('$co', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_iter'],3))"
done
