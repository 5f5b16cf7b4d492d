"""B200-native DiscoMatch dual-solver hot path.

Drop-in for the reference package ``prodmatch``'s dual solver
(qn.solve / dual / kernels, /root/reference/pkg/src/prodmatch): the same
Python API over hand-written sm_100a CUDA kernels behind the C-ABI in
include/discomatch_b200.h.  Modules mirror the reference's names:
``ilp``, ``splitting``, ``kernels``, ``dual``, ``qn``, ``primal``,
``config``, ``errors``; ``product_space`` builds the shape-matching ILP.
"""

from .config import MODE_HYBRID, MODE_MMA_ONLY, SolveConfig
from .errors import (EmptyFeasibleSet, EmptyHistory, InfeasibleAfterFixing, NativeLibraryError,
                     ProdmatchError, SplitAtTerminalLayer, UnsupportedInstance)
from .ilp import Bdd, IlpInstance, LinearRow, build_equality_bdd, make_row
from . import bdd  # noqa: E402  (attaches the reference's per-diagram Bdd methods)

__version__ = "0.1.0"

__all__ = ["Bdd", "IlpInstance", "LinearRow", "make_row", "build_equality_bdd", "SolveConfig",
           "MODE_HYBRID", "MODE_MMA_ONLY", "ProdmatchError", "EmptyFeasibleSet", "EmptyHistory",
           "InfeasibleAfterFixing", "SplitAtTerminalLayer", "NativeLibraryError", "UnsupportedInstance"]
