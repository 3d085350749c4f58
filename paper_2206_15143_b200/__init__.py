"""paper_2206_15143_b200 -- B200-native DP-KFAC second-order update.

Public surface:
  * ``DPKFAC``                      -- the drop-in optimizer-side preconditioner (dpkfac.py)
  * ``kfac``                        -- functional mirror of kfaclab kfac.py / numerics.py on CUDA tensors
  * ``partition``                   -- reference round-robin partition + the LPT balancer
  * ``errors``                      -- reference exception classes
  * ``checkpoint``                  -- per-rank factor-state checkpoints in the reference KFACLAB\0 v1 layout
The arithmetic lives in ``libdpkfac.so`` (csrc/, sm_100a); see include/dpkfac.h.
"""

from . import errors, partition
from .errors import ArgumentError, DataFormatError, KfacLabError, NumericError, OrderingError, ShapeError
from .kfac import EigenPair, FactorState, KfacHyper
from .partition import balanced_partition, round_robin_partition, validate_partition

__version__ = "0.1.0"


def __getattr__(name):
    # torch-dependent modules load lazily so `import paper_2206_15143_b200` stays cheap
    if name == "DPKFAC":
        from .dpkfac import DPKFAC
        return DPKFAC
    if name in ("kfac", "ops", "dpkfac", "checkpoint"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
