timeout 600 python -m pytest tests -m gpu -x -q -k "eig" 2>&1 | tail -2
timeout 400 python bench.py --steps 5 --warmup 3 --inv-type eigen --no-cpu-baseline --no-e2e > gpurun_out/bench_r01c_eigen2.json 2> gpurun_out/eig.err; echo eigen=$?
python -c "import json; d=json.load(open('gpurun_out/bench_r01c_eigen2.json')); print(round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages_ms'].items()})"
python - <<'PY'
import torch, time
for n in (4608, 2304, 1152, 576, 256):
    a = torch.randn(n, n, device="cuda"); a = a @ a.T / n
    torch.linalg.eigh(a); torch.cuda.synchronize()
    t = time.time(); torch.linalg.eigh(a); torch.cuda.synchronize(); print(n, "eigh fp32 %.1f ms" % ((time.time() - t) * 1000))
PY
