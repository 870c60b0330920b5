"""B200-native tile tensors (arXiv 2011.01805) -- the data-parallel hot path.

Host API mirrors the reference's ``namespace tiletensor``; all slot arithmetic
runs in hand-written sm_100a kernels behind the C-ABI in
``include/tiletensor_b200.h``.  See DESIGN.md.
"""
from .tiletensor import *  # noqa: F401,F403
from .tiletensor import __all__ as _tt_all
from . import nn  # noqa: F401  (inc/nn.hpp mirror)

__all__ = list(_tt_all)
