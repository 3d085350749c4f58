import sys, json, runpy, io, contextlib
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_15143_b200.dpkfac as D
res = []
for mc, ratio in ((3, 0.6), (2, 0.6), (4, 0.6), (3, 0.4), (4, 0.4), (3, 0.8)):
    D.DPKFAC.MAX_CLASSES, D.DPKFAC.CLASS_RATIO = mc, ratio
    sys.argv = ["bench.py", "--steps", "20", "--warmup", "3", "--no-cpu-baseline", "--no-e2e"]
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        try:
            runpy.run_path("bench.py", run_name="__main__")
        except SystemExit:
            pass
    d = json.loads(buf.getvalue().strip().splitlines()[-1])
    print(mc, ratio, round(d["ms_per_step"], 3), round(d["ms_per_step_serialized"], 3), flush=True)
