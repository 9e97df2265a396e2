"""B200-native RouterWise setup-search inner loop (arxiv 2604.10907).

The hot path — select_setup -> optimize_beta -> optimize_fractions -> solve_dual ->
eval_dual — runs as one persistent sm_100a kernel per sweep (csrc/rw_solver.cuh) behind
the C-ABI in include/rw_b200.h.  `routeplan` mirrors the reference C++ API on top of it.
"""
from . import _abi
from .routeplan import *  # noqa: F401,F403
from .routeplan import Engine, engine, reduce_records, select_setup  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
