run() { python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('$*', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3))"; }
for m in resnet50 densenet201 inception_v4; do for c in 0 112 96; do run --model $m --side-cap $c; done; done
for n in 2 4; do for c in 0 112; do python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2975$n bench.py --gpus $n --steps 20 --warmup 3 --no-e2e --side-cap $c 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('N=$n side-cap $c', round(d['ms_per_step'],3))"; done; done
