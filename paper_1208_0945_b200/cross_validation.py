"""Prior-variance cross-validation on the device (cross_validation.hpp).

Mirrors the reference's CVConfig / CVCell / CVResult / grid_search_cv /
kfold_split / predictive_log_likelihood.  The fold loop runs in the native
library (drivers.cpp): each fold's training and held-out datasets are built
on the device (``engine="subset"``, the reference's route) or the folds run
as one batched weighted fit (``engine="batched"``).

Multi-GPU: pass ``group`` (a torch.distributed process group, any backend);
every rank must hold the same dataset on its own device.  Folds are dealt to
ranks in contiguous ranges, the cells are all-gathered and every rank runs
the same selection -- folds are independent (cross_validation.hpp:146-176),
so no collective sits on the fit path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import bsccs as B
from ._native import bsccs_cv_cell, bsccs_cv_config, bsccs_cv_result, lib

ENGINES = {"subset": 0, "batched": 1}


def default_variance_grid() -> List[float]:
    """cross_validation.hpp:19-27: 13 points log-uniform on [0.001, 10]."""
    out = (C.c_double * 13)()
    lib().bsccs_default_variance_grid(out)
    return list(out)


@dataclass
class CVConfig:
    """cross_validation.hpp:29-41 (defaults identical), plus the engine."""
    folds: int = 10
    variance_grid: List[float] = field(default_factory=default_variance_grid)
    prior_kind: B.PriorKind = B.PriorKind.laplace
    variance_is_laplace_scale: bool = False
    seed: int = 0
    solver: B.SolverConfig = field(default_factory=B.SolverConfig)
    warm_start: bool = True
    engine: str = "subset"
    batch: int = 0

    def _c(self) -> bsccs_cv_config:
        if self.engine not in ENGINES:
            raise B.InputError(f"cross-validation: unknown engine {self.engine!r}")
        c = bsccs_cv_config()
        c.folds = int(self.folds)
        c.prior_kind = int(self.prior_kind)
        c.variance_is_laplace_scale = int(bool(self.variance_is_laplace_scale))
        c.warm_start = int(bool(self.warm_start))
        c.seed = int(self.seed) & 0xFFFFFFFFFFFFFFFF
        c.solver = self.solver._c()
        c.engine = ENGINES[self.engine]
        c.batch = int(self.batch)
        return c


@dataclass
class CVCell:
    """cross_validation.hpp:43-48."""
    predictive_ll: float = float("-inf")
    cycles: int = 0
    converged: bool = False
    valid: bool = False


@dataclass
class CVResult:
    """cross_validation.hpp:50-57, plus device instrumentation."""
    variance_grid: List[float]
    cells: List[List[CVCell]]  # [grid point][fold]
    mean_predictive_ll: List[float]
    selected_index: int = -1
    selected_variance: float = 0.0
    total_cycles: int = 0
    device_seconds: float = 0.0
    fits: int = 0
    coordinates_visited: int = 0


kfold_split = B.kfold_split


def predictive_log_likelihood(beta, heldout) -> float:
    """cross_validation.hpp:89-93: init_state on the held-out data at beta,
    then log_likelihood (device)."""
    st = B.init_state(heldout, beta)
    try:
        return B.log_likelihood(heldout, st)
    finally:
        st.close()


def _grid(cfg: CVConfig) -> np.ndarray:
    return np.ascontiguousarray(cfg.variance_grid, dtype=np.float64)


def _cells_to_py(arr, points: int, folds: int) -> List[List[CVCell]]:
    return [[CVCell(arr[g * folds + f].predictive_ll, arr[g * folds + f].cycles, bool(arr[g * folds + f].converged),
                    bool(arr[g * folds + f].valid)) for f in range(folds)] for g in range(points)]


def grid_search_cv(ds, cfg: Optional[CVConfig] = None, pool=None, group=None) -> CVResult:
    """cross_validation.hpp:100-215 on the device.  `pool` is accepted for
    signature parity (the device runs one fit at a time at full width)."""
    cfg = cfg or CVConfig()
    dds = B._dev(ds)
    grid = _grid(cfg)
    P = grid.size
    c = cfg._c()
    res = bsccs_cv_result()
    folds = max(int(cfg.folds), 1)
    cells = (bsccs_cv_cell * (max(P, 1) * folds))()
    mean = np.full(max(P, 1), np.nan)
    if group is None:
        grid_out = np.zeros(max(P, 1))
        B._check(lib().bsccs_grid_search_cv(dds.handle, C.byref(c), B._ptr(grid), P, B._ptr(grid_out), cells,
                                            B._ptr(mean), C.byref(res)))
        sorted_grid = grid_out[:P]
    else:
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        f0, f1 = folds * rank // world, folds * (rank + 1) // world
        B._check(lib().bsccs_cv_run_folds(dds.handle, C.byref(c), B._ptr(grid), P, f0, f1, cells, C.byref(res)))
        mine = {(g, f): bytes(cells[g * folds + f]) for g in range(P) for f in range(f0, f1)}
        stats = (res.device_seconds, res.fits, res.coordinates_visited)
        gathered = [None] * world
        dist.all_gather_object(gathered, (mine, stats), group=group)
        tot = [0.0, 0, 0]
        for part, st in gathered:
            for (g, f), raw in part.items():
                C.memmove(C.byref(cells, (g * folds + f) * C.sizeof(bsccs_cv_cell)), raw, len(raw))
            tot = [a + b for a, b in zip(tot, st)]
        sorted_grid = np.sort(grid)
        B._check(lib().bsccs_cv_select(B._ptr(sorted_grid), P, folds, cells, B._ptr(mean), C.byref(res)))
        res.device_seconds, res.fits, res.coordinates_visited = tot[0], int(tot[1]), int(tot[2])
    return CVResult(list(sorted_grid), _cells_to_py(cells, P, folds), list(mean[:P]), res.selected_index,
                    res.selected_variance, res.total_cycles, res.device_seconds, res.fits, res.coordinates_visited)
