set -x
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/bench_r01c_n4.json 2> gpurun_out/bench_r01c_n4.err; echo rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 --steps 10 --warmup 3 --assignment balanced > gpurun_out/bench_r01c_n4_bal.json 2> gpurun_out/bench_r01c_n4_bal.err; echo rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 bench.py --impl reference --gpus 4 --steps 2 --warmup 1 > gpurun_out/bench_ref_r01c_n4.json 2> gpurun_out/bench_ref_r01c_n4.err; echo rc=$?
timeout 300 python -m pytest tests/test_exchange_gloo.py -q 2>&1 | tail -3
cat gpurun_out/bench_r01c_n4.json gpurun_out/bench_r01c_n4_bal.json gpurun_out/bench_ref_r01c_n4.json
tail -5 gpurun_out/bench_r01c_n4.err
