timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "f16" 2>&1 | tail -2
timeout 300 python scripts/f16_one.py 2>&1 | tail -5
for pd in f32 f16; do
timeout 300 python - <<PY > gpurun_out/bpd_$pd.txt 2>&1
import sys; sys.argv=['bench.py','--steps','20','--warmup','3','--no-cpu-baseline','--no-e2e']
import paper_2206_15143_b200.dpkfac as D
orig = D.DPKFAC.__init__
def init(self, *a, **k):
    k['patch_dtype'] = '$pd'; orig(self, *a, **k)
D.DPKFAC.__init__ = init
import runpy; runpy.run_path('bench.py', run_name='__main__')
PY
python -c "import json; d=json.loads(open('gpurun_out/bpd_$pd.txt').read().strip().splitlines()[-1]); print('$pd bench', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3), {k: round(v,3) for k,v in d['stages_ms'].items()})"
done
