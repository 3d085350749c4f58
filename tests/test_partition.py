"""Layer -> GPU assignment: bit-exact reference round robin + the LPT balancer."""

import json
import os

import pytest

from conftest import GOLDEN
from paper_2206_15143_b200 import ArgumentError
from paper_2206_15143_b200.partition import (assign_layers_round_robin, balanced_partition, imbalance, layer_cost,
                                             round_robin_partition, validate_partition)


def test_round_robin_bit_exact_against_reference_golden():
    with open(os.path.join(GOLDEN, "partitions.json")) as f:
        table = json.load(f)
    for key, parts in table.items():
        L, P = map(int, key.split("x"))
        got = round_robin_partition(L, P)
        assert [list(p) for p in got] == parts, key
        assert got == assign_layers_round_robin(L, P)


def test_known_answers():
    # reference test_distsim.py:40-57
    assert round_robin_partition(4, 4) == ((0,), (1,), (2,), (3,))
    assert round_robin_partition(5, 2) == ((0, 2, 4), (1, 3))
    assert round_robin_partition(7, 1) == (tuple(range(7)),)
    parts = round_robin_partition(3, 8)
    assert len(parts) == 8 and max(map(len, parts)) - min(map(len, parts)) <= 1
    validate_partition(parts, 3)


def test_validate_partition_rejects_overlap_and_gap():
    with pytest.raises(ArgumentError):
        validate_partition(((0, 1), (1,)), 2)
    with pytest.raises(ArgumentError):
        validate_partition(((0,), ()), 2)
    with pytest.raises(ArgumentError):
        round_robin_partition(3, 0)


def _resnet50_costs():
    with open(os.path.join(GOLDEN, "resnet50_manifest.json")) as f:
        dims = json.load(f)["dims"]
    # M = B*H*W per layer at B=32, derived from the stage of each layer
    ms = [401408] + [100352] * 11 + [25088] * 13 + [6272] * 19 + [1568] * 9 + [32]
    ms[11] = 100352  # layer2.0.conv1 runs at 56x56
    ms[24] = 25088   # layer3.0.conv1 runs at 28x28
    ms[43] = 6272    # layer4.0.conv1 runs at 14x14
    return [layer_cost(a, b, m) for (a, b), m in zip(dims, ms)]


def test_balanced_is_deterministic_valid_and_better_than_round_robin():
    costs = _resnet50_costs()
    for P in (2, 4, 8):
        a = balanced_partition(costs, P)
        assert a == balanced_partition(list(costs), P)
        validate_partition(a, len(costs))
        assert all(list(p) == sorted(p) for p in a)
        assert imbalance(costs, a) <= imbalance(costs, round_robin_partition(len(costs), P))
    assert imbalance(costs, balanced_partition(costs, 8)) < 1.1


def test_balanced_tie_break_by_index_then_rank():
    assert balanced_partition([1.0, 1.0, 1.0, 1.0], 2) == ((0, 2), (1, 3))
    assert balanced_partition([5.0], 3) == ((0,), (), ())


def test_step_time_partition_matches_golden_and_removes_padding():
    """DPKFAC assignment="balanced": bit-exact against the committed golden
    partitions (validated by the reference's distsim.validate_partition when they
    were generated, tests/golden/make_partition_golden.py); owner-major padding
    <= 5% at P = 2/4/8 and an estimated step no slower than round robin."""
    from paper_2206_15143_b200.partition import partition_report, step_time_partition
    with open(os.path.join(GOLDEN, "balanced_partitions.json")) as f:
        gold = json.load(f)
    for model in ("resnet50", "inception_v4"):  # densenet201: same code path, slower to recompute
        layers = [tuple(x) for x in gold[model]["layers"]]
        for P, g in gold[model]["partitions"].items():
            a = step_time_partition(layers, int(P))
            assert [list(p) for p in a] == g["assignment"], (model, P)
            validate_partition(a, len(layers))
            rep = partition_report(layers, a)
            assert rep["padding"] <= 0.05
            assert rep["est_ms"] <= g["round_robin_report"]["est_ms"] + 1e-9
    for model in gold:
        for P, g in gold[model]["partitions"].items():
            validate_partition(tuple(tuple(p) for p in g["assignment"]), len(gold[model]["layers"]))
            assert g["report"]["padding"] <= 0.05
