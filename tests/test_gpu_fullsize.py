"""Full-size parity through size-independent properties (BASELINE configs C2-C4 at
their real shapes, where the float64 CPU oracle would take minutes per step).

After the first DP-KFAC step (t = 0: the factors are exactly A = X X^T / M and
G = Gamma Gamma^T / M, kfac.py:85-125) -- or after t >= 1, where they are the
running average of the per-step factors -- for every checked layer:
  * factor action on a random vector:  A v == X (X^T v) / M  and  G v == Gamma (Gamma^T v) / M,
    X / Gamma built in float64 from the captured activations / output gradients with
    F.unfold in the reference (C, kh, kw) order;
  * preconditioned gradient:  out == (G + sqrt(g)/pi I)^-1 grad (A + pi sqrt(g) I)^-1
    (kfac.py:128-171), the right-hand side solved in float64 from the exported factors.
Tolerance: relative Frobenius error <= 1e-3 (fp32 path, BASELINE north_star).
"""

import numpy as np
import pytest
import torch
import torch.nn as nn
import torch.nn.functional as F

pytestmark = pytest.mark.gpu
TOL = 1e-3


def _rel(a, b):
    return float(torch.linalg.norm(a - b) / torch.linalg.norm(b).clamp_min(1e-300))


def _record(model):
    rec, hooks = {}, []
    for name, m in model.named_modules():
        if isinstance(m, (nn.Conv2d, nn.Linear)):
            def pre(mod, inp, name=name):
                rec.setdefault(name, {})["x"] = inp[0].detach()

            def fwd(mod, inp, out, name=name):
                out.register_hook(lambda g, name=name: rec[name].__setitem__("g", g.detach()))
            hooks += [m.register_forward_pre_hook(pre), m.register_forward_hook(fwd)]
    return rec, hooks


def _x_cols(m, x):
    x = x.double()
    if isinstance(m, nn.Conv2d):
        c = F.unfold(x.contiguous(), m.kernel_size, dilation=m.dilation, padding=m.padding, stride=m.stride)
        X = c.permute(1, 0, 2).reshape(c.shape[1], -1)
    else:
        X = x.reshape(-1, x.shape[-1]).T
    if m.bias is not None:
        X = torch.cat([X, torch.ones(1, X.shape[1], dtype=X.dtype, device=X.device)])
    return X


def _g_cols(m, g, batch):
    g = g.double()
    G = g.permute(1, 0, 2, 3).reshape(g.shape[1], -1) if isinstance(m, nn.Conv2d) else g.reshape(-1, g.shape[-1]).T
    return G * batch  # B_local * dL/ds: per-sample gradients (model.py:9-12, 243)


def _precond_want(A, G, grad, gamma, inv_type):
    """float64 right-hand side from the exported factors: kfac.py:165-171 (inverse,
    pi-split damping) or kfac.py:174-191 (eigen, exact (A (x) G + gamma I)^-1)."""
    dev = A.device
    if inv_type == "eigen":
        va, qa = torch.linalg.eigh(0.5 * (A + A.T))
        vg, qg = torch.linalg.eigh(0.5 * (G + G.T))
        d = vg.clamp_min(0)[:, None] * va.clamp_min(0)[None, :] + gamma
        return qg @ ((qg.T @ grad @ qa) / d) @ qa.T
    r = gamma ** 0.5
    pi = float(torch.sqrt((torch.trace(A) / A.shape[0]) / (torch.trace(G) / G.shape[0])))
    la = torch.linalg.cholesky(A + pi * r * torch.eye(A.shape[0], device=dev, dtype=torch.float64))
    lg = torch.linalg.cholesky(G + r / pi * torch.eye(G.shape[0], device=dev, dtype=torch.float64))
    return torch.cholesky_solve(torch.cholesky_solve(grad, lg).T, la).T


def _run(model_name, every=1, gamma=0.002, steps=1, inv_type="inverse", xi=0.95):
    """``steps`` DP-KFAC steps on fresh synthetic batches (no weight update in
    between); the checks run after the last one.  steps >= 2 exercises the
    running average F = xi F_new + (1 - xi) F_old (kfac.py:107-125) and the
    refresh on the blended factors."""
    torchvision = pytest.importorskip("torchvision")  # noqa: F841
    import bench_models as BM
    from paper_2206_15143_b200 import DPKFAC
    dev = torch.device("cuda", 0)
    ctor, batch, shape, classes = BM.WORKLOADS[model_name]
    torch.manual_seed(0)
    model = ctor().to(dev).to(memory_format=torch.channels_last)
    kf = DPKFAC(model, gamma=gamma, xi=xi, inv_type=inv_type)
    mods = [(n, m) for n, m in model.named_modules() if isinstance(m, (nn.Conv2d, nn.Linear))]
    gen = torch.Generator().manual_seed(1234)
    recs = []
    for t in range(steps):
        rec, hooks = _record(model)
        x = torch.randn(batch, *shape, generator=gen).to(dev).contiguous(memory_format=torch.channels_last)
        y = torch.randint(0, classes, (batch,), generator=gen).to(dev)
        model.zero_grad()
        F.cross_entropy(model(x), y).backward()
        for h in hooks:
            h.remove()
        recs.append(rec)
        grads = []
        for _, m in mods:
            w = m.weight.grad.double().reshape(m.weight.shape[0], -1)
            if m.bias is not None:
                w = torch.cat([w, m.bias.grad.double()[:, None]], 1)
            grads.append(w)
        kf.step()
    torch.cuda.synchronize()
    sd = kf.state_dict()["layers"]
    gen_v = torch.Generator(device=dev).manual_seed(7)
    worst = {}
    for i, (name, m) in enumerate(mods):
        if i % every:
            continue
        A, G = sd[i]["a_cov"].double(), sd[i]["g_cov"].double()
        va = torch.randn(A.shape[0], generator=gen_v, device=dev, dtype=torch.float64)
        vg = torch.randn(G.shape[0], generator=gen_v, device=dev, dtype=torch.float64)
        want_a = torch.zeros_like(va)
        want_g = torch.zeros_like(vg)
        for t, rec in enumerate(recs):  # the running average of the per-step factor actions
            w = 1.0 if t == 0 else xi
            want_a.mul_(1.0 - (0.0 if t == 0 else xi))
            want_g.mul_(1.0 - (0.0 if t == 0 else xi))
            X = _x_cols(m, rec[name]["x"])
            Gm = _g_cols(m, rec[name]["g"], batch)
            M = X.shape[1]
            want_a += w * (X @ (X.T @ va)) / M
            want_g += w * (Gm @ (Gm.T @ vg)) / M
            del X, Gm
        ea = _rel(A @ va, want_a)
        eg = _rel(G @ vg, want_g)
        want = _precond_want(A, G, grads[i], gamma, inv_type)
        got = m.weight.grad.double().reshape(m.weight.shape[0], -1)
        if m.bias is not None:
            got = torch.cat([got, m.bias.grad.double()[:, None]], 1)
        ep = _rel(got, want)
        worst[name] = (ea, eg, ep)
        assert ea <= TOL and eg <= TOL and ep <= TOL, (name, ea, eg, ep)
    kf.remove_hooks()
    return worst


def test_resnet50_config3_fullsize_properties():
    w = _run("resnet50")
    assert len(w) == 54


def test_resnet32_config2_fullsize_properties():
    w = _run("resnet32")
    assert len(w) >= 31


def test_densenet201_config4_fullsize_properties():
    w = _run("densenet201", every=3)
    assert len(w) >= 60


def test_resnet50_config3_fullsize_running_average_t2():
    """Third step (t = 2): factors are the xi-blend of three batches' factors."""
    w = _run("resnet50", steps=3)
    assert len(w) == 54


def test_resnet50_config3_fullsize_eigen_mode():
    """Eigen mode (the reference default) at full size, after the EMA step: the
    preconditioned gradient equals the exact (A (x) G + gamma I)^-1 solve."""
    w = _run("resnet50", steps=2, inv_type="eigen", every=2)
    assert len(w) == 27


def test_inception_v4_config5_fullsize_properties():
    """Config C5 at its real shapes (B=16, 299x299): 1x7/7x1 and 1x3/3x1 convs with
    asymmetric padding, 1537-dim fc factor."""
    w = _run("inception_v4", every=4)
    assert len(w) >= 37
