# multi-GPU: NCCL parity vs the oracle's P-worker step (PARITY OK logs) + bench at N
N=${1:-2}
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611 scripts/multi_gpu_parity.py > gpurun_out/parity_p${N}.log 2>&1; echo "parity rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/bench_n${N}.json 2> gpurun_out/bench_n${N}.err; echo "bench rc=$?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus $N --steps 20 --warmup 5 --assignment round_robin --no-e2e > gpurun_out/bench_n${N}_rr.json 2> gpurun_out/bench_n${N}_rr.err; echo "bench rr rc=$?"
tail -5 gpurun_out/parity_p${N}.log; head -c 700 gpurun_out/bench_n${N}.json; echo; head -c 500 gpurun_out/bench_n${N}_rr.json
