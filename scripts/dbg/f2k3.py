"""Debug: C1 DPKFAC F=2/K=3 vs oracle, per-step diagnostics."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch, torch.nn as nn, torch.nn.functional as F
from oracle import kfac_ref as K, mlp_ref as MLP
from paper_2206_15143_b200 import DPKFAC

def torch_mlp(weights, dev):
    mods = []
    for i, w in enumerate(weights):
        lin = nn.Linear(w.shape[1] - 1, w.shape[0])
        with torch.no_grad():
            lin.weight.copy_(torch.from_numpy(w[:, :-1])); lin.bias.copy_(torch.from_numpy(w[:, -1]))
        mods.append(lin)
        if i < len(weights) - 1: mods.append(nn.ReLU())
    return nn.Sequential(*mods).to(dev), [m for m in mods if isinstance(m, nn.Linear)]

def rel(a, b): return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
inv = sys.argv[1] if len(sys.argv) > 1 else "eigen"
ff, kk = int(sys.argv[2]) if len(sys.argv) > 2 else 2, int(sys.argv[3]) if len(sys.argv) > 3 else 3
dev = torch.device("cuda", 0)
spec = MLP.MlpSpec((784, 512, 256, 10), "relu", "softmax_cross_entropy", True)
h = K.Hyper(gamma=0.03, xi=0.95, inv_type=inv, f_freq=ff, k_freq=kk)
cl = MLP.build_cluster(spec, 1, seed=0)
model, lins = torch_mlp([w.copy() for w in cl.weights], dev)
kf = DPKFAC(model, inv_type=inv, f_freq=ff, k_freq=kk)
opt = torch.optim.SGD(model.parameters(), lr=0.05, momentum=0.9)
rng = np.random.default_rng(4321)
for t in range(8):
    x = rng.standard_normal((784, 64)); y = rng.integers(0, 10, size=64)
    _, pre = MLP.dp_kfac_step(cl, MLP.shard(x, y, 1), h, 0.05, 0.9, t)
    opt.zero_grad()
    F.cross_entropy(model(torch.from_numpy(x.T.copy()).float().to(dev)), torch.from_numpy(y).to(dev)).backward()
    kf.step(); torch.cuda.synchronize()
    errs = []
    for i, lin in enumerate(lins):
        got = torch.cat([lin.weight.grad, lin.bias.grad[:, None]], 1).double().cpu().numpy()
        st = cl.states[0][i]; ly = kf.layers[i]
        e = [rel(got, pre[i]), rel(ly.a_cov.double().cpu().numpy(), st.a_cov), rel(ly.g_cov.double().cpu().numpy(), st.g_cov)]
        if inv == "eigen":
            q = ly.a_q.double().cpu().numpy(); e.append(float(np.abs(q.T @ q - np.eye(q.shape[0])).max()))
            e.append(rel(ly.a_w.double().cpu().numpy(), st.a_eig.values))
            qg = ly.g_q.double().cpu().numpy(); e.append(float(np.abs(qg.T @ qg - np.eye(qg.shape[0])).max()))
            e.append(rel(ly.g_w.double().cpu().numpy(), st.g_eig.values))
        errs.append(["%.2e" % v for v in e])
    print(t, errs, flush=True)
    opt.step()
