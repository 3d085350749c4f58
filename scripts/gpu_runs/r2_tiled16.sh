python -m pytest tests/test_gpu_kernels.py -x -q -k "f16_patches or implicit_f16 or prescale or tapmajor" 2>&1 | tail -4
python scripts/im2col16_one.py 64 56 20
python scripts/im2col16_one.py 16 32 20
for m in resnet32 resnet50; do python bench.py --model $m --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('$m', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), {k:round(v,3) for k,v in d['stages_ms'].items()})"; done
