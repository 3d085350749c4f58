"""Golden balanced partitions (DPKFAC assignment="balanced" = partition.step_time_partition)
for ResNet-50 (B=32), DenseNet-201 (B=16) and Inception-v4 (B=16) at P = 2/4/8, each
validated by the REFERENCE's own checker (kfaclab distsim.validate_partition,
distsim.py:93-101 -- the explicit-assignment hook of build_cluster, distsim.py:140-147).

    python tests/golden/make_partition_golden.py      (build container: needs /root/reference)
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import bench_models as BM  # noqa: E402
from kfaclab import distsim  # noqa: E402  (the reference)
from paper_2206_15143_b200.partition import partition_report, round_robin_partition, step_time_partition  # noqa: E402

out = {}
for model in ("resnet50", "densenet201", "inception_v4"):
    ctor, batch, shape, _ = BM.WORKLOADS[model]
    layers = [[a, o, m] for _, a, o, m, _ in BM.layer_geometry(ctor(), shape, batch)]
    out[model] = {"layers": layers, "partitions": {}}
    for P in (2, 4, 8):
        a = step_time_partition([tuple(x) for x in layers], P)
        distsim.validate_partition(a, len(layers))  # raises on an invalid partition
        out[model]["partitions"][str(P)] = {
            "assignment": [list(p) for p in a],
            "report": partition_report(layers, a),
            "round_robin_report": partition_report(layers, round_robin_partition(len(layers), P))}
with open(os.path.join(HERE, "balanced_partitions.json"), "w") as f:
    json.dump(out, f)
print({m: {P: round(v["report"]["padding"], 4) for P, v in d["partitions"].items()} for m, d in out.items()})
