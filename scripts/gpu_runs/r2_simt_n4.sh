for n in 2 4; do for v in 1.5e8 5e7 1.5e8 5e7; do DPK_SIMT_FMA=$v python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2976$n bench.py --gpus $n --steps 20 --warmup 3 --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('N=$n SIMT $v', round(d['ms_per_step'],3))"; done; done
