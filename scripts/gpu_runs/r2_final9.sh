# (HEAD: cp.async latency path, one capture hook per layer, leaf row skip) 4 GPUs: full gpu suite (incl. the NCCL test at P=2/4), N=1/2/4 bench lines, P=4 parity with KL-clip
mkdir -p gpurun_out/final
python scripts/tf32_peak.py gpurun_out/final/tf32_peak.json > /dev/null 2>&1; echo "tf32 peak rc=$?"
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final/gputest.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/final/gputest.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651 scripts/multi_gpu_parity.py > gpurun_out/final/parity_p4.log 2>&1; echo "parity4 rc=$?"; tail -1 gpurun_out/final/parity_p4.log
python bench.py --steps 20 --warmup 5 > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; echo "bench1 rc=$?"
for n in 2 4; do python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2966$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/final/bench_n$n.json 2> gpurun_out/final/bench_n$n.err; echo "bench$n rc=$?"; done
for n in 2 4; do python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2967$n bench.py --gpus $n --steps 20 --warmup 5 --assignment round_robin --no-e2e > gpurun_out/final/bench_n${n}_rr.json 2>/dev/null; echo "bench$n rr rc=$?"; done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29681 bench.py --gpus 4 --impl reference --steps 10 --warmup 2 > gpurun_out/final/bench_ref_n4.json 2>/dev/null; echo "ref4 rc=$?"
for m in resnet32 densenet201 inception_v4; do python bench.py --model $m --no-cpu-baseline > gpurun_out/final/bench_$m.json 2>/dev/null; echo "$m rc=$?"; done
for f in bench bench_n2 bench_n4 bench_n2_rr bench_n4_rr bench_resnet32 bench_densenet201 bench_inception_v4; do python -c "import json;d=json.load(open('gpurun_out/final/$f.json'));print('$f', round(d['ms_per_step'],3), round(d['value'],1), (d.get('e2e') or {}).get('ms_per_iter'), d.get('clocks',{}).get('sm_mhz'), d.get('clocks',{}).get('reasons'))"; done
python bench.py --inv-type eigen --steps 5 --warmup 3 --e2e-steps 5 --no-cpu-baseline > gpurun_out/final/bench_eigen.json 2>/dev/null; echo "eigen rc=$?"
DPK_PROFILE_TIMED=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/final/launches_timed_step.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/final/ncu_launch.log 2>&1; echo "launch list rc=$?"
