import torch, time
dev = torch.device("cuda", 0)
for n, k in ((256, 24), (512, 16), (576, 6), (1024, 8), (2304, 6), (4608, 3)):
    a = torch.randn(k, n, n, device=dev); a = a @ a.transpose(1, 2) / n
    torch.linalg.eigh(a[:1]); torch.cuda.synchronize()
    t = time.time(); torch.linalg.eigh(a); torch.cuda.synchronize(); tb = time.time() - t
    t = time.time()
    for i in range(k): torch.linalg.eigh(a[i])
    torch.cuda.synchronize(); ts = time.time() - t
    print(f"n={n} k={k}: batched {tb*1e3:.1f} ms, loop {ts*1e3:.1f} ms", flush=True)
