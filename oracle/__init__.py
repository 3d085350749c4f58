"""CPU oracle for the DP-KFAC second-order update -- TEST INFRASTRUCTURE ONLY.

This package restates, in numpy float64, the reference algorithm of
``kfaclab`` 0.1.0 (``/root/reference/pkg/src/kfaclab``) for exactly the hot path
this repository accelerates: factor construction, running average, pi-split
damped Cholesky inverses, eigendecomposition, preconditioning, the per-layer
step, the round-robin layer partition, and (for the 3-layer MLP config) the
whole simulated ``dp_kfac_step``.

Who may import it: ``tests/``, ``__graft_entry__.smoke()`` (as the checker) and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm).  The
product package ``paper_2206_15143_b200`` never imports, links or executes
anything in here; its CUDA path fails loudly when the extension is missing.

Parity pin: every function here is checked against golden vectors produced by
the reference implementation itself (``tests/golden/make_golden.py`` imports
kfaclab from /root/reference in the build container and writes
``tests/golden/*.npz``); see ``tests/test_oracle_golden.py``.
"""
