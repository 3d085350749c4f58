#!/usr/bin/env python
"""Benchmark of the DP-KFAC second-order update (BASELINE.json metric) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--model resnet50|resnet32|densenet201|mlp] [--inv-type inverse|eigen]

A "step" is one DP-KFAC second-order update (kfaclab distsim.dp_kfac_step's
second-order part, distsim.py:300-337): Kronecker-factor SYRK + running
average, damped inversion, gradient reduce-scatter, preconditioning,
all-gather -- over one synthetic batch per GPU (ResNet-50: 32 x 3x224x224,
random init, synthetic data) whose layer captures and gradients are resident in
HBM when the timed region starts (they total > 1.4 GB, larger than L2, so no
flush is needed).  ``value`` = samples/s of that update for the whole job
(iter/s x 32 x N); ``e2e`` = the same through the public API for full training
iterations (pinned-host batch H2D, forward, backward, DPKFAC.step(),
optimizer.step(), loss D2H).

``--impl reference`` times the reference algorithm on the host CPU (the
float64 oracle port of kfaclab's kfac.py, all host threads): each step is a
bounded, rotating 1/9 of the layers; the full-update time is the sum of every
layer's median MEASURED time (no cost-model extrapolation).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DP-KFAC 2nd-order update ms/iter + iter/s, ResNet-50 at 1/2/4/8 B200 vs CPU"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--inv-type", default="inverse", choices=["inverse", "eigen"])
    ap.add_argument("--gamma", type=float, default=0.002)
    ap.add_argument("--xi", type=float, default=0.95)      # reference default (kfac.py:61)
    ap.add_argument("--precision", default="auto", choices=["auto", "tf32", "3xtf32"])
    ap.add_argument("--nchw", action="store_true",
                    help="keep the conv model NCHW (default: channels_last, the B200-native layout)")
    # north_star: "layers are assigned to GPUs by a load balancer" -> the LPT balancer
    # (SURVEY 8(f)1); "round_robin" is the reference's bit-exact default partition
    ap.add_argument("--assignment", default="balanced")
    ap.add_argument("--im2col", default="materialize", choices=["materialize", "auto", "implicit", "implicit16"])
    ap.add_argument("--algorithm", default="dp_kfac", choices=["dp_kfac", "mpd_kfac_co", "mpd_kfac_mo"],
                    help="dp_kfac (the product) or the paper's MPD-KFAC comparators on the same kernels")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-overlap", action="store_true", help="run every stage on one stream")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--early", action="store_true",
                    help="e2e: launch the larger size classes' factor/inverse pipeline from the backward hooks")
    ap.add_argument("--max-classes", type=int, default=None, help="tuning: DPKFAC.MAX_CLASSES")
    ap.add_argument("--class-ratio", type=float, default=None, help="tuning: DPKFAC.CLASS_RATIO")
    ap.add_argument("--factor-order", type=int, default=None, help="tuning: DPKFAC.FACTOR_ORDER")
    ap.add_argument("--side-cap", type=int, default=None, help="tuning: DPKFAC.SIDE_CAP")
    ap.add_argument("--comm-overlap", action="store_true",
                    help="bucketed gradient reduce-scatter launched from the backward hooks (e2e)")
    ap.add_argument("--bucket-mb", type=float, default=16.0)
    ap.add_argument("--peer-gather", action="store_true",
                    help="closing all-gather as one NVLink peer-copy kernel (IPC-mapped chunks) instead of NCCL")
    ap.add_argument("--early-priority", default="high", choices=["high", "low"],
                    help="e2e with --early: stream priority of the hook-launched pipelines")
    ap.add_argument("--ncu-step", action="store_true",
                    help="profiling helper: after warm-up run ONE serialized step between cudaProfilerStart/Stop "
                         "with NVTX stage ranges (DPK_NVTX) and exit without a result line")
    return ap.parse_args()


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region
    (B200_PROFILING.md clocks line): NVML polled every ~2 ms from a thread (a timed
    region of 10 steps lasts only ~50-90 ms), nvidia-smi -lms 200 as the fallback."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.nv = []
        self.proc = None
        self.stop = threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_sm = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            reasons = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                N.nvmlDeviceGetCurrentClocksThrottleReasons

            def poll():
                while not self.stop.is_set():
                    try:
                        self.nv.append((N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM), int(reasons(h))))
                    except Exception:  # noqa: BLE001 -- sampling must never break the bench
                        pass
                    time.sleep(0.002)

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return self
        except Exception:  # noqa: BLE001 -- no NVML: nvidia-smi
            pass
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        elif self.t is not None:
            self.t.join(timeout=1)

    def summary(self):
        if self.nv:
            sm = [c for c, _ in self.nv]
            reasons = sorted({n for _, r in self.nv for n, b in self.BITS.items() if r & b})
            return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_sm, "reasons": reasons,
                    "samples": len(self.nv), "source": "nvml"}
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "source": "nvidia-smi"}


# ----------------------------------------------------------------- CPU reference (oracle port)
def cpu_reference_layers(geom, layers, inv_type: str, gamma: float, xi: float, seed: int = 0):
    """Time the reference algorithm (float64 oracle port of kfaclab kfac.py:
    kfac_layer_step = factor SYRK + running-average blend, damped inverses or
    eigendecompositions, preconditioning) on each listed layer, synthetic captures
    of the exact unfolded shapes.  Returns {layer index: seconds} -- every number
    measured, nothing extrapolated."""
    import numpy as np

    from oracle import kfac_ref as K  # bench.py's cpu_baseline / reference leg only

    h = K.Hyper(gamma=gamma, xi=xi, inv_type=inv_type)
    out = {}
    for i in layers:
        _, d_in, d_out, m, _ = geom[i]
        rng = np.random.default_rng(seed + i)
        x = np.maximum(rng.standard_normal((d_in, m)), 0.0)
        x[-1] = 1.0
        g = rng.standard_normal((d_out, m)) * 1e-2
        grad = rng.standard_normal((d_out, d_in)) * 1e-3
        st = K.LayerState()
        a0, g0 = K.compute_factors(x[:, : min(m, 64)], g[:, : min(m, 64)])
        K.update_running_average(st, a0, g0, xi, 0)  # initialised state: the timed update blends
        t0 = time.perf_counter()
        K.kfac_layer_step(st, x, g, grad, h, 1)
        out[i] = time.perf_counter() - t0
        del x, g
    return out


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count()


def run_reference(args, rank, world):
    """--impl reference: rank 0 times the CPU reference.  Step s runs the layers
    i % G == s % G (G = 9 groups for the 54-layer ResNet-50, so one step is ~1/9
    of an update and the whole run fits a few minutes); the full-update time is
    the SUM over all layers of each layer's median measured time (layers the
    timed steps did not reach are measured after them), never a model estimate."""
    if rank != 0:
        return
    import bench_models as BM

    ctor, batch, shape, classes = BM.WORKLOADS[args.model]
    geom = BM.layer_geometry(ctor(), shape, batch)
    n = len(geom)
    groups = 9 if n > 20 else 1
    per_layer: dict = {}
    step_ms = []
    for s in range(args.warmup + args.steps):
        layers = [i for i in range(n) if i % groups == s % groups]
        t0 = time.perf_counter()
        got = cpu_reference_layers(geom, layers, args.inv_type, args.gamma, args.xi)
        wall = time.perf_counter() - t0
        if s >= args.warmup:
            step_ms.append(1000.0 * wall)
            for i, sec in got.items():
                per_layer.setdefault(i, []).append(sec)
    missing = [i for i in range(n) if i not in per_layer]
    extra = cpu_reference_layers(geom, missing, args.inv_type, args.gamma, args.xi)
    for i, sec in extra.items():
        per_layer.setdefault(i, []).append(sec)
    ms_iter = 1000.0 * sum(statistics.median(v) for v in per_layer.values())
    # P ranks of the simulated cluster run their owned layers sequentially (distsim.py:310-329),
    # so the reference's whole-job iteration time does not shrink with P: samples/s = B*P / t.
    value = batch * world / (ms_iter / 1000.0)
    sample = (f"step s = layers i % {groups} == s % {groups} of {n} (synthetic captures of the exact unfolded "
              "shapes), kfac_layer_step in float64 numpy/scipy (OpenBLAS, all host threads); value = one "
              "full update = sum over all layers of each layer's median measured seconds "
              f"({min(len(v) for v in per_layer.values())}-{max(len(v) for v in per_layer.values())} "
              f"samples per layer{'; ' + str(len(missing)) + ' layers measured after the timed steps' if missing else ''})")
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.median(step_ms),
        "ms_per_iter": ms_iter, "iter_per_s": 1000.0 / ms_iter,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.model} DP-KFAC 2nd-order update, batch {batch}/GPU, {args.inv_type}",
                   "model": args.model, "global_batch": batch * world, "parallelism": f"dp{world}",
                   "step": f"one bounded sample = 1/{groups} of the layers; ms_per_iter = the full update"},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": host_threads(), "kind": "port",
                         "ms_per_iter": ms_iter, "sample": sample},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


# ----------------------------------------------------------------- ours
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist
    import torch.nn.functional as F

    import bench_models as BM
    from paper_2206_15143_b200 import DPKFAC, _lib

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    torch.backends.cudnn.benchmark = True
    lib = _lib.load()
    ctor, batch, shape, classes = BM.WORKLOADS[args.model]
    torch.manual_seed(0)
    model = ctor().to(dev)
    geom = BM.layer_geometry(model, shape, batch)
    conv = len(shape) == 3
    mf = torch.contiguous_format if (args.nchw or not conv) else torch.channels_last
    if conv:
        model = model.to(memory_format=mf)
    kf = DPKFAC(model, gamma=args.gamma, xi=args.xi, inv_type=args.inv_type, f_freq=1, k_freq=1,
                assignment=args.assignment, precision=args.precision, check_numerics="deferred",
                overlap=not args.no_overlap, early=False, algorithm=args.algorithm, im2col=args.im2col,
                comm_overlap=args.comm_overlap, bucket_mb=args.bucket_mb,
                peer_gather=args.peer_gather)  # captures are replayed below; e2e turns early on
    for attr, val in (("MAX_CLASSES", args.max_classes), ("CLASS_RATIO", args.class_ratio),
                      ("FACTOR_ORDER", args.factor_order), ("SIDE_CAP", args.side_cap)):
        if val is not None:
            setattr(kf, attr, val)
    opt = torch.optim.SGD(model.parameters(), lr=1e-3, momentum=0.9)
    gen = torch.Generator().manual_seed(1234 + rank)
    x_host = torch.randn(batch, *shape, generator=gen)
    if conv:
        x_host = x_host.contiguous(memory_format=mf)
    x_host = x_host.pin_memory()
    y_host = torch.randint(0, classes, (batch,), generator=gen).pin_memory()
    x = x_host.to(dev)
    y = y_host.to(dev)

    def sync_barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # one forward/backward: captures + gradients resident in HBM
    model.zero_grad(set_to_none=False)
    F.cross_entropy(model(x), y).backward()
    kf.step()  # first step builds buffers/balance; captures are consumed
    model.zero_grad(set_to_none=False)
    F.cross_entropy(model(x), y).backward()
    capt = kf.layers if args.algorithm != "dp_kfac" else kf.owned
    saved_caps = {ly.index: (ly.a_in, ly.g_out, ly.batch) for ly in capt}
    layer_params = [p for ly in kf.layers for p in ([ly.module.weight] + ([ly.module.bias] if ly.has_bias else []))]
    saved_grads = [p.grad.clone() for p in layer_params]

    def restore():
        for ly in capt:
            ly.a_in, ly.g_out, ly.batch = saved_caps[ly.index]
        torch._foreach_copy_([p.grad for p in layer_params], saved_grads)

    for _ in range(args.warmup):
        restore()
        kf.step()
    kf.check()
    sync_barrier()
    if args.ncu_step:  # ncu --profile-from-start off --nvtx --nvtx-include "<stage>/" ...
        kf.overlap = False
        restore()
        kf.step()
        sync_barrier()
        kf.nvtx = True
        restore()
        torch.cuda.cudart().cudaProfilerStart()
        kf.step()
        sync_barrier()
        torch.cuda.cudart().cudaProfilerStop()
        kf.check()
        kf.remove_hooks()
        return
    launches0 = lib.dpk_launch_count()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # DPK_PROFILE_TIMED=1: bracket exactly the timed steps for `ncu --profile-from-start off`
    prof = os.environ.get("DPK_PROFILE_TIMED") == "1"
    with ClockSampler(local_rank) as clocks:
        sync_barrier()
        if prof:
            torch.cuda.cudart().cudaProfilerStart()
        start.record()
        for _ in range(args.steps):
            restore()
            kf.step()
        end.record()
        sync_barrier()
        if prof:
            torch.cuda.cudart().cudaProfilerStop()
    kf.check()
    launches = lib.dpk_launch_count() - launches0
    ms_local = start.elapsed_time(end) / args.steps
    # per-stage split: the same steps with the stages serialized on one stream
    # (the timed steps above overlap the largest layers' pipeline with the rest)
    overlap = kf.overlap
    kf.overlap = False
    for _ in range(2):
        restore()
        kf.step()
    sync_barrier()
    kf.enable_stage_timing(True)
    s1, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s1.record()
    for _ in range(args.steps):
        restore()
        kf.step()
    e1.record()
    sync_barrier()
    kf.check()
    ms_serial = s1.elapsed_time(e1) / args.steps
    stages = {k: v / args.steps for k, v in kf.stage_ms().items()}
    kf.enable_stage_timing(False)
    kf.overlap = overlap
    t = torch.tensor([ms_local], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = batch * world / (ms / 1000.0)

    # ---- roofline of the dominant stage's kernel(s)
    peaks = {}
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        with open(pk) as f:
            peaks = json.load(f)
    bf16 = peaks.get("bf16_tflops") or 1590.0  # f16 and bf16 issue at the same kind::f16 rate
    bf16_src = "MEASURED_PEAKS.json bf16_tflops" if peaks.get("bf16_tflops") else "B200_PROFILING.md fallback"
    tf32_peak, tf32_src = bf16 / 2.0, bf16_src + " / 2 (kind::tf32 issues at half the f16 rate)"
    tp = os.path.join(ROOT, "profiles", "tf32_peak.json")  # scripts/tf32_peak.py, measured on a B200
    if os.path.exists(tp):
        with open(tp) as f:
            tpj = json.load(f)
        tf32_peak = tpj["tf32_peak_tflops"]
        tf32_src = ("profiles/tf32_peak.json: measured 8192^3 TF32 matmul, best of 10 (max of cuBLAS "
                    f"{tpj['cublas_tf32_tflops']:.0f} and this engine {tpj['dpk_tf32_tflops']:.0f} TF/s)")
    own = [geom[ly.index] for ly in kf.owned]
    f16_a = {ly.index for ly in kf.layers if ly.patch16 is not None or ly.nhwc16 is not None}  # conv A factors on kind::f16
    built = geom if args.algorithm != "dp_kfac" else own  # MPD: every rank builds every layer's factors
    built_idx = range(len(geom)) if args.algorithm != "dp_kfac" else [ly.index for ly in kf.owned]
    syrk_f16 = sum(geom[i][1] * (geom[i][1] + 1) * geom[i][3] for i in built_idx if i in f16_a)
    syrk_all = sum(d_in * (d_in + 1) * m + d_out * (d_out + 1) * m for _, d_in, d_out, m, _ in built)
    fac_passes = 3.0 if kf.precision == "3xtf32" else 1.0
    flops = {
        "factors": syrk_all,
        # inverse mode: Cholesky n^3/3 + triangular inverse n^3/3 (the optimizer keeps
        # A^-1 = X^T X factored, so potri's X^T X product is not part of the step)
        "inversion": sum((2.0 / 3.0) * (float(d_in) ** 3 + float(d_out) ** 3) for _, d_in, d_out, m, _ in own)
        if args.inv_type == "inverse" else sum(9.0 * (float(d_in) ** 3 + float(d_out) ** 3) for _, d_in, d_out, m, _ in own),
        "precondition": sum(2.0 * (d_out * d_out * d_in + d_out * d_in * d_in) * (1 if args.inv_type == "inverse" else 2)
                            for _, d_in, d_out, m, _ in own),
    }
    # ideal (roofline) time of each stage at the peak of the precision its MMAs run in:
    # factors = kind::f16 conv patches at the f16 peak + the rest at tf32 (x3 passes if
    # 3xtf32); inversion / precondition = 3xTF32 products (tf32 peak / 3)
    ideal_ms = {"factors": 1e3 * (syrk_f16 / (bf16 * 1e12) + fac_passes * (syrk_all - syrk_f16) / (tf32_peak * 1e12)),
                "inversion": 1e3 * 3.0 * flops["inversion"] / (tf32_peak * 1e12),
                "precondition": 1e3 * 3.0 * flops["precondition"] / (tf32_peak * 1e12)}
    compute_stages = {k: stages.get(k, 0.0) for k in flops}
    dom = max(compute_stages, key=compute_stages.get)
    achieved = flops[dom] / (compute_stages[dom] / 1000.0) / 1e12 if compute_stages[dom] > 0 else 0.0
    traffic, traffic_src = None, None
    prof = os.path.join(ROOT, "profiles", "stage_traffic.json")  # scripts/stage_traffic.sh (ncu, HEAD)
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                tj = json.load(f)
            st_ = tj.get("stages", {}).get(dom)
            if st_ and tj.get("model") == args.model and tj.get("inv_type") == args.inv_type and world == 1:
                traffic = st_["dram_bytes"]
                traffic_src = (f"profiles/stage_traffic.json: sum of dram__bytes_read+write over the "
                               f"{st_['launches']} kernels of the {dom} stage of one serialized step (ncu, "
                               f"commit {tj.get('commit', '?')})")
        except (OSError, ValueError, KeyError):
            traffic = None
    three_pass = dom in ("inversion", "precondition")
    roofline = {"bound": "tensor", "achieved": achieved, "peak": tf32_peak, "unit": "TFLOP/s",
                "frac": achieved / tf32_peak, "traffic": traffic, "traffic_source": traffic_src, "kernel": dom,
                "peak_source": tf32_src,
                "frac_of_3xtf32_ceiling": (3.0 * achieved / tf32_peak) if three_pass else None,
                "frac_of_stage_roofline": ideal_ms[dom] / compute_stages[dom] if compute_stages[dom] > 0 else None,
                "note": ("fp32-grade stage: every product is 3 tf32 MMA passes (3xTF32), so its tensor-core "
                         "ceiling is peak/3" if three_pass else "mixed kind::f16 / tf32 stage"),
                "algorithmic_work": f"{dom}: {flops[dom] / 1e12:.4f} TFLOP per step (SURVEY 8(d) conventions)"}
    stage_roofline = {k: {"ms": compute_stages[k], "tflops": (flops[k] / (compute_stages[k] / 1000.0) / 1e12)
                          if compute_stages[k] > 0 else None,
                          "frac_of_tf32": ((flops[k] / (compute_stages[k] / 1000.0) / 1e12) / tf32_peak)
                          if compute_stages[k] > 0 else None,
                          "ideal_ms": ideal_ms[k],
                          "frac_of_stage_roofline": ideal_ms[k] / compute_stages[k] if compute_stages[k] > 0 else None}
                      for k in flops}
    stage_roofline["factors"]["f16_flops_share"] = syrk_f16 / syrk_all if syrk_all else 0.0
    stage_roofline["peaks_tflops"] = {"f16": bf16, "tf32": tf32_peak, "3xtf32": tf32_peak / 3.0}

    # ---- e2e through the public API: pinned H2D + fwd + bwd + DPKFAC.step() + SGD + loss D2H
    e2e = None
    if not args.no_e2e:
        k_e2e = args.e2e_steps or args.steps
        for ly in capt:
            ly.a_in = ly.g_out = None
        del saved_caps, saved_grads

        def train_step():
            xb = x_host.to(dev, non_blocking=True)
            yb = y_host.to(dev, non_blocking=True)
            opt.zero_grad(set_to_none=False)
            loss = F.cross_entropy(model(xb), yb)
            loss.backward()
            kf.step()
            opt.step()
            return loss.item()

        kf.early = args.early and not args.no_overlap  # hook-time launch of the larger classes' pipelines
        kf.early_priority = args.early_priority
        for _ in range(2):
            train_step()
        sync_barrier()
        s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s2.record()
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            train_step()
        e2.record()
        sync_barrier()
        e2e_ms = torch.tensor([s2.elapsed_time(e2) / k_e2e], device=dev)
        if world > 1:
            dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
        e2e_ms = float(e2e_ms.item())
        e2e = {"value": batch * world / (e2e_ms / 1000.0), "unit": "samples/s", "ms_per_iter": e2e_ms,
               "h2d_bytes_per_step": x_host.numel() * x_host.element_size() + y_host.numel() * y_host.element_size(),
               "d2h_bytes_per_step": 4,
               "what": "full training iteration: pinned-host batch H2D, forward, backward, DPKFAC.step(), "
                       "SGD step, loss.item()"}

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # every layer once (the same per-layer measurement as --impl reference): ~15 s
        # of host work for ResNet-50 in inverse mode
        per = cpu_reference_layers(geom, range(len(geom)), args.inv_type, args.gamma, args.xi)
        cpu_ms = 1000.0 * sum(per.values())
        cpu_baseline = {"value": batch / (cpu_ms / 1000.0), "unit": "samples/s", "cores": host_threads(),
                        "kind": "port", "ms_per_iter": cpu_ms,
                        "sample": f"all {len(geom)} layers once (synthetic captures of the exact unfolded shapes), "
                                  "float64 kfac_layer_step (oracle port of kfaclab kfac.py, numpy/scipy "
                                  "OpenBLAS, all host threads), summed -- measured, not extrapolated"}

    if kf.precision == "tf32":
        dtype_label = ("f32 (conv A-factor patches as fp16 with an exact power-of-two prescale from a fused amax "
                       "-> tcgen05 kind::f16 SYRK, fp32 accumulate; other factors 1-pass RN tf32; inverse and "
                       "precondition 3xtf32)" if f16_a else "f32 (1-pass RN tf32 factors; 3xtf32 inverse/precondition)")
    else:
        dtype_label = "f32 (3xtf32 factors, inverse/eigen and precondition)"
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "iter_per_s": 1000.0 / ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype_label,
            "data": "synthetic (randn images, random labels, torch.manual_seed(0) random-init weights)",
            "config": {"workload": f"{args.model} DP-KFAC 2nd-order update, batch {batch}/GPU, "
                                   f"inv_type={args.inv_type}, gamma={args.gamma}, xi={args.xi}, F=K=1",
                       "model": args.model, "global_batch": batch * world, "parallelism": f"dp{world}",
                       "assignment": args.assignment, "algorithm": args.algorithm, "im2col": args.im2col,
                       "comm_overlap": (f"bucketed reduce-scatter from the backward hooks, {args.bucket_mb} MB buckets"
                                        if args.comm_overlap else False),
                       "all_gather": ("none (one rank)" if world == 1 else
                                      "NVLink peer-copy kernel" if getattr(getattr(kf, "xchg", None), "_peer_ptrs", None)
                                      is not None else "NCCL"),
                       "memory_format": "channels_last" if mf is torch.channels_last else "contiguous",
                       "l2": "inputs (layer captures, >1.4 GB) larger than L2; no flush"},
            "overlap": overlap, "ms_per_step_serialized": ms_serial,
            "stages_ms": stages, "stage_roofline": stage_roofline, "roofline": roofline,
            "cpu_baseline": cpu_baseline, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks.summary(),
        }
        emit(line)
    kf.remove_hooks()


_JSON_OUT = None


def emit(line):
    """The one JSON result line, on the process's original stdout."""
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    # Keep stdout JSON-only: libraries (NCCL's version banner at communicator
    # init, cuSOLVER/cuBLAS warnings) write to fd 1 directly, so fd 1 is pointed
    # at stderr and the result line goes to a private copy of the original fd.
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
