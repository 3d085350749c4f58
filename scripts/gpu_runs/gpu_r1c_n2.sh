timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for a in dp_kfac mpd_kfac_co mpd_kfac_mo; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e --algorithm $a > gpurun_out/bench_r01c_n2_$a.json 2> gpurun_out/bench_r01c_n2_$a.err; echo $a=$?
python -c "import json; d=json.load(open('gpurun_out/bench_r01c_n2_$a.json')); print('$a', round(d['ms_per_step'],3), round(d['value']), {k: round(v,3) for k,v in d['stages_ms'].items()})"
done
