timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python scripts/host_profile.py 2>&1 | head -3
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bhost.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bhost.json')); print('bench', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), 'e2e', round(d['e2e']['ms_per_iter'],2))"
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bhost_n2.json 2> /dev/null; echo n2=$?
python -c "import json; d=json.load(open('gpurun_out/bhost_n2.json')); print('n2', round(d['ms_per_step'],3), round(d['value']), 'e2e', round(d['e2e']['ms_per_iter'],2))"
