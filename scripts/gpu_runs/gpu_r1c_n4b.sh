for a in dp_kfac mpd_kfac_co mpd_kfac_mo; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --steps 10 --warmup 3 --algorithm $a > gpurun_out/bench_r01c_n4_$a.json 2> gpurun_out/bench_r01c_n4_$a.err; echo $a=$?
python -c "import json; d=json.load(open('gpurun_out/bench_r01c_n4_$a.json')); print('$a', d['config']['assignment'], round(d['ms_per_step'],3), round(d['value']), {k: round(v,3) for k,v in d['stages_ms'].items()}, 'e2e', round(d['e2e']['ms_per_iter'],2))"
done
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_r01c_n2_balanced.json 2> gpurun_out/n2b.err; echo n2=$?
python -c "import json; d=json.load(open('gpurun_out/bench_r01c_n2_balanced.json')); print('n2 balanced', round(d['ms_per_step'],3), round(d['value']), 'e2e', round(d['e2e']['ms_per_iter'],2))"
for m in resnet32 densenet201; do
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py --model $m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r01c_$m.json 2> gpurun_out/$m.err; echo $m=$?
python -c "import json; d=json.load(open('gpurun_out/bench_r01c_$m.json')); print('$m', round(d['ms_per_step'],3), round(d['value']), round(d['ms_per_step_serialized'],3), {k: round(v,3) for k,v in d['stages_ms'].items()}, 'e2e', round(d['e2e']['ms_per_iter'],2))"
done
