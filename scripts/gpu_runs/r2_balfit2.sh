for cfg in "DPK_NOP=1" "DPK_BAL_SYRK=400e12" "DPK_BAL_SYRK=500e12" "DPK_BAL_SYRK=700e12" "DPK_BAL_SYRK=1000e12" "DPK_BAL_SYRK=500e12 DPK_BAL_CHAIN=0.7e-6"; do
  for n in 2 4; do env $cfg python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2978$n bench.py --gpus $n --steps 20 --warmup 3 --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('N=$n $cfg', round(d['ms_per_step'],3))"; done; done
