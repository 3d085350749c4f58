"""Golden MPD-KFAC (KAISA COMM-OPT / MEM-OPT comparator) runs from the REFERENCE
(kfaclab distsim.mpd_kfac_step, distsim.py:341-420):

    python tests/golden/make_mpd_golden.py   ->  mlp_mpd.npz
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
RUNS = [(2, "co", "inverse"), (2, "mo", "inverse"), (4, "co", "eigen"), (2, "mo", "eigen"), (1, "co", "inverse")]


def main():
    sys.path.insert(0, REF)
    from kfaclab import distsim, kfac, model
    spec = model.NetworkSpec((20, 16, 12, 5), activation="relu", loss_kind="softmax_cross_entropy",
                             bias_mode="homogeneous")
    rng = np.random.default_rng(91)
    batches = [(rng.standard_normal((20, 16)), rng.integers(0, 5, size=16)) for _ in range(4)]
    out = {}
    for bi, (x, y) in enumerate(batches):
        out[f"batch/{bi}/x"], out[f"batch/{bi}/y"] = x, y
    for workers, var, inv in RUNS:
        h = kfac.KfacHyper(gamma=0.05, xi=0.9, inv_type=inv, f_freq=1, k_freq=2)
        cl = distsim.build_cluster(spec, f"mpd_kfac_{var}", workers, seed=5)
        losses = []
        for t, (x, y) in enumerate(batches):
            r = distsim.mpd_kfac_step(cl, distsim.shard_batch(model.Batch(x, y), workers), h, 0.1, 0.9, t, var)
            losses.append(r.loss)
        key = f"run/{workers}/{var}/{inv}"
        out[key + "/losses"] = np.array(losses)
        for i, layer in enumerate(cl.workers[0].replica.layers):
            out[key + f"/w{i}"] = layer.weight
    np.savez_compressed(os.path.join(HERE, "mlp_mpd.npz"), **out)
    print("wrote mlp_mpd.npz")


if __name__ == "__main__":
    main()
