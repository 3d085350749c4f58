python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e > gpurun_out/n2.json 2> gpurun_out/n2.err; echo rc=$?
cat gpurun_out/n2.json
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --assignment balanced > gpurun_out/n2b.json 2>> gpurun_out/n2.err; echo rc=$?
cat gpurun_out/n2b.json
tail -5 gpurun_out/n2.err
