timeout 600 python -m pytest tests/test_gpu_dpkfac.py -x -q -k "multi_gpu" 2>&1 | tail -2
for a in dp_kfac; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/bench_r01c_n4_final.json 2> gpurun_out/n4final.err; echo n4=$?
python -c "import json; d=json.load(open('gpurun_out/bench_r01c_n4_final.json')); print('n4', d['config']['assignment'], round(d['ms_per_step'],3), round(d['value']), {k: round(v,3) for k,v in d['stages_ms'].items()}, 'e2e', round(d['e2e']['ms_per_iter'],2))"
done
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_r01c_n2_final.json 2> gpurun_out/n2final.err; echo n2=$?
python -c "import json; d=json.load(open('gpurun_out/bench_r01c_n2_final.json')); print('n2', round(d['ms_per_step'],3), round(d['value']), {k: round(v,3) for k,v in d['stages_ms'].items()}, 'e2e', round(d['e2e']['ms_per_iter'],2))"
