"""B200-native CCD hot path of arXiv 1208.0945 (BSCCS MAP fitting).

`bsccs` mirrors the reference engine/solver API; `datagen` builds synthetic
case series; the arithmetic lives in _lib/libbsccs_b200.so (sm_100a).
"""
from . import bsccs, datagen  # noqa: F401
from .bsccs import (  # noqa: F401
    ConvergenceError, Dataset, FitResult, InputError, InternalError, NumericError, PriorKind, PriorSpec,
    SolverConfig, build_dataset, fit,
)
