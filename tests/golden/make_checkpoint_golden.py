"""Golden KFACLAB v1 checkpoints written by the REFERENCE (kfaclab trainer.save_checkpoint).

    python tests/golden/make_checkpoint_golden.py

A 2-worker DP-KFAC cluster of a small MLP (inverse and eigen modes) is stepped
twice by distsim.dp_kfac_step and saved; the files pin our encoder/decoder
byte for byte (tests/test_checkpoint.py).
"""
import os
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    from kfaclab import distsim, kfac, model, trainer
    spec = model.NetworkSpec((6, 5, 3), "tanh", "softmax_cross_entropy", "homogeneous")
    rng = np.random.default_rng(4)
    x = rng.standard_normal((6, 8))
    y = rng.integers(0, 3, size=8)
    for inv in ("inverse", "eigen"):
        cl = distsim.build_cluster(spec, "dp_kfac", 2, seed=9)
        h = kfac.KfacHyper(gamma=0.05, xi=0.9, inv_type=inv, f_freq=1, k_freq=1)
        shards = distsim.shard_batch(model.Batch(x, y), 2)
        for t in range(2):
            distsim.dp_kfac_step(cl, shards, h, 0.1, 0.9, t)
        trainer.save_checkpoint(Path(HERE) / f"kfaclab_ckpt_{inv}.bin", cl, iteration=2, epoch=0)
        print("wrote", inv)


if __name__ == "__main__":
    main()
