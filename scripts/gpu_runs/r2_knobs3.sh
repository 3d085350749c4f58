run() { env "$@" python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('$*', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), {k:round(v,3) for k,v in d['stages_ms'].items()})"; }
run DPK_NOP=1
run DPK_SIMT_FMA=0
run DPK_SIMT_FMA=5e7
run DPK_SIMT_FMA=3e8
run DPK_SPLIT_MIN=32
run DPK_SPLIT_MIN=128
run DPK_NOP=1
run DPK_GEMM_FORK=0
run DPK_CG2=0
run DPK_NOP=1
