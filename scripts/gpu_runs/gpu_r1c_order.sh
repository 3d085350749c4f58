for fo in 0 1 2 0 1 2; do
timeout 300 python -c "
import sys; sys.path.insert(0, '.')
import paper_2206_15143_b200.dpkfac as D
D.DPKFAC.FACTOR_ORDER = $fo
sys.argv = ['bench.py', '--steps', '20', '--warmup', '3', '--no-cpu-baseline', '--no-e2e']
import runpy; runpy.run_path('bench.py', run_name='__main__')" > gpurun_out/ord.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ord.json')); print('order $fo', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3))"
done
