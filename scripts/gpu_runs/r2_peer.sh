# NVLink peer-copy all-gather: P=2/4 parity, then N=2/4 bench with and without it
mkdir -p gpurun_out/peer
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 $TR --nproc-per-node 2 --master-port 29721 scripts/multi_gpu_parity.py > gpurun_out/peer/parity_p2.log 2>&1; echo "parity2 rc=$?"; tail -1 gpurun_out/peer/parity_p2.log
timeout 300 $TR --nproc-per-node 4 --master-port 29722 scripts/multi_gpu_parity.py > gpurun_out/peer/parity_p4.log 2>&1; echo "parity4 rc=$?"; tail -1 gpurun_out/peer/parity_p4.log
for n in 2 4; do
  for pg in "" "--peer-gather"; do
    timeout 400 $TR --nproc-per-node $n --master-port 2973$n bench.py --gpus $n --steps 20 --warmup 5 $pg > gpurun_out/peer/bench_n${n}${pg:+_peer}.json 2> gpurun_out/peer/bench_n${n}${pg:+_peer}.err; echo "bench$n $pg rc=$?"
    python -c "import json;d=json.load(open('gpurun_out/peer/bench_n${n}${pg:+_peer}.json'));print('n=$n $pg', round(d['ms_per_step'],3), round(d['value'],1), {k:round(v,3) for k,v in d['stages_ms'].items()}, round(d['e2e']['ms_per_iter'],2), d['config'].get('all_gather'))"
  done
done
