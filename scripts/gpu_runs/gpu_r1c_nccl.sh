run() { timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 scripts/nccl_probe.py 2>&1 | grep "P=" ; }
run 4 29551
NCCL_NVLS_ENABLE=1 run 4 29552
NCCL_ALGO=Ring run 4 29553
NCCL_ALGO=NVLS run 4 29554
NCCL_DEBUG=INFO timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29555 scripts/nccl_probe.py 2>&1 | grep -iE "NVLS|algo|channel|Using network|P2P|NCCL INFO Connected all" | head -12
run 2 29556
