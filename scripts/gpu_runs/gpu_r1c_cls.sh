for cfg in "3 0.6" "2 0.6" "4 0.6" "3 0.4" "4 0.4" "3 0.8" "4 0.8"; do
set -- $cfg
timeout 300 python -c "
import sys; sys.path.insert(0, '.')
import paper_2206_15143_b200.dpkfac as D
D.DPKFAC.MAX_CLASSES, D.DPKFAC.CLASS_RATIO = $1, $2
sys.argv = ['bench.py', '--steps', '20', '--warmup', '3', '--no-cpu-baseline', '--no-e2e']
import runpy; runpy.run_path('bench.py', run_name='__main__')" > gpurun_out/cls.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/cls.json')); print('$1 $2', round(d['ms_per_step'],3), round(d['ms_per_step_serialized'],3))"
done
