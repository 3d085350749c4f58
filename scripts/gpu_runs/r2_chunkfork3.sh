timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
for v in 0 1 0 1; do DPK_CHUNK_FORK=$v python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('fork $v resnet50', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3))"; done
for v in 0 1; do for m in densenet201 inception_v4; do DPK_CHUNK_FORK=$v python bench.py --model $m --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); print('fork $v $m', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3))"; done; done
