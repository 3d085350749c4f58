timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for v in 0 1 0 1; do for m in resnet50; do DPK_CHUNK_FORK=$v python bench.py --model $m --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('fork $v $m', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3))"; done; done
for m in densenet201 inception_v4 resnet32; do python bench.py --model $m --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('fork 1 $m', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3))"; done
