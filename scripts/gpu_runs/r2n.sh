# e2e at N=4 with and without hook-time launch (early) of the big classes' factor/inverse pipelines
for v in "" "--early" "--early --early-priority low"; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29621 bench.py --gpus 4 --steps 20 --warmup 5 --e2e-steps 30 $v > gpurun_out/e2e4.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/e2e4.json'));print('N=4 $v', round(d['ms_per_step'],3), round(d['e2e']['ms_per_iter'],3))"
done
