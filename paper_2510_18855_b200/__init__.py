"""B200-native (sm_100a) IcePop policy-gradient objective -- drop-in for the hot path of
arXiv 2510.18855's RL trainer as restated by the reference (mismatchlab).

* ``paper_2510_18855_b200.loss``       tensor API + torch custom op (bf16 tcgen05 / fp64 SIMT)
* ``paper_2510_18855_b200.objective``  drop-in ``objective_and_grad`` / ``LossBreakdown``
* ``paper_2510_18855_b200.distributed`` token sharding + NCCL reductions
* ``include/icepop.h``                 the C ABI of ``libicepop_b200.so``
"""

from .errors import ConfigError, NumericError, TickCapError

__version__ = "0.1.0"

__all__ = ["ConfigError", "NumericError", "TickCapError", "__version__"]
