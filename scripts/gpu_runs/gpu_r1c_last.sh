timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
CUDA_VISIBLE_DEVICES=0 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py > gpurun_out/bench_last.json 2> gpurun_out/bench_last.err; echo bench=$?
python -c "import json; d=json.load(open('gpurun_out/bench_last.json')); print(round(d['ms_per_step'],3), round(d['value']), d['e2e']['ms_per_iter'], d['cpu_baseline']['value'], d['gpu_launches'], d['clocks'])"
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29601 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_last_n2.json 2>> gpurun_out/bench_last.err; echo n2=$?
python -c "import json; d=json.load(open('gpurun_out/bench_last_n2.json')); print('n2', round(d['ms_per_step'],3), round(d['value']), d['e2e']['ms_per_iter'])"
