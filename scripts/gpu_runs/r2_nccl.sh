mkdir -p gpurun_out/nccl
run() { echo "== $*" >> gpurun_out/nccl/out.txt; env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29711 scripts/nccl_probe.py >> gpurun_out/nccl/out.txt 2>&1; }
run X=1
run NCCL_MIN_NCHANNELS=32
run NCCL_PROTO=Simple
run NCCL_ALGO=Ring
run NCCL_ALGO=NVLS
run NCCL_NVLS_ENABLE=0
NCCL_DEBUG=INFO python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29712 scripts/nccl_probe.py > gpurun_out/nccl/debug.txt 2>&1
grep -i "nvls\|algo\|channels" gpurun_out/nccl/debug.txt | head -20 >> gpurun_out/nccl/out.txt
cat gpurun_out/nccl/out.txt
