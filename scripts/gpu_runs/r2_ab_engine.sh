for i in 1 2; do
for lib in old new; do
  if [ $lib = old ]; then export DPK_LIB_PATH=$PWD/exp_so/libdpkfac_old.so; else unset DPK_LIB_PATH; fi
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('$lib resnet50', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), {k:round(v,3) for k,v in d['stages_ms'].items()})"
done; done
for lib in old new; do
  if [ $lib = old ]; then export DPK_LIB_PATH=$PWD/exp_so/libdpkfac_old.so; else unset DPK_LIB_PATH; fi
  for m in densenet201 inception_v4 resnet32; do python bench.py --model $m --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('$lib $m', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), {k:round(v,3) for k,v in d['stages_ms'].items()})"; done
done
