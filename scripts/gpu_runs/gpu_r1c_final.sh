nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
CUDA_VISIBLE_DEVICES=0 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r01c_final.json 2> gpurun_out/final.err; echo bench=$?
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r01c_final.json 2>> gpurun_out/final.err; echo ref=$?
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_r01c_final_n2.json 2>> gpurun_out/final.err; echo n2=$?
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29582 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/bench_r01c_final_n4.json 2>> gpurun_out/final.err; echo n4=$?
CUDA_VISIBLE_DEVICES=0 DPK_PROFILE_TIMED=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01c_final_launches_timed_step.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo launches=$?
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:im2col_k16 -s 1 -c 1 -o gpurun_out/prof_im2col_k16 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu_k16=$?
for f in bench_r01c_final bench_r01c_final_n2 bench_r01c_final_n4; do python -c "import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['n_gpus'], round(d['ms_per_step'],3), round(d['value']), 'serial', round(d['ms_per_step_serialized'],3), 'e2e', round(d['e2e']['ms_per_iter'],2), d['clocks'])"; done
