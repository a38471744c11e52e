"""Bootstrap uncertainty on the device (bootstrap.hpp).

Mirrors the reference's BootstrapConfig / BootstrapResult / resample /
run_bootstrap / report_ranked_intervals.  Replicate r resamples subjects
from Rng(seed, r + 1) (bootstrap.hpp:103-106) and is refitted in the native
library (drivers.cpp): materialised on the device and fitted by the
single-fit kernel (``engine="subset"``) or run R at a time as weighted fits
of the parent dataset (``engine="batched"``).

Multi-GPU: pass ``group`` (torch.distributed); replicates are dealt to ranks
in contiguous ranges (each is a pure function of (seed, r)), the estimates
are all-gathered and every rank computes the same summary.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import bsccs as B
from ._native import bsccs_bootstrap_config, bsccs_bootstrap_result, lib

ENGINES = {"subset": 0, "batched": 1}

resample = B.resample


@dataclass
class BootstrapConfig:
    """bootstrap.hpp:17-28 (defaults identical), plus the engine."""
    replicates: int = 200
    level: float = 0.95
    seed: int = 0
    prior: B.PriorSpec = field(default_factory=B.PriorSpec)
    solver: B.SolverConfig = field(default_factory=B.SolverConfig)
    warm_start: bool = True
    engine: str = "subset"
    batch: int = 0

    def _c(self) -> bsccs_bootstrap_config:
        if self.engine not in ENGINES:
            raise B.InputError(f"bootstrap: unknown engine {self.engine!r}")
        c = bsccs_bootstrap_config()
        c.replicates = int(self.replicates)
        c.warm_start = int(bool(self.warm_start))
        c.level = float(self.level)
        c.seed = int(self.seed) & 0xFFFFFFFFFFFFFFFF
        c.prior = self.prior._c()
        c.solver = self.solver._c()
        c.engine = ENGINES[self.engine]
        c.batch = int(self.batch)
        return c


@dataclass
class BootstrapResult:
    """bootstrap.hpp:30-41, plus device instrumentation."""
    beta_full: np.ndarray
    full_converged: bool
    lower: np.ndarray
    upper: np.ndarray
    p_hat: np.ndarray
    replicates: int = 0
    used: int = 0
    non_converged: int = 0
    device_seconds: float = 0.0
    total_cycles: int = 0
    coordinates_visited: int = 0


def run_bootstrap(ds, cfg: Optional[BootstrapConfig] = None, pool=None, group=None) -> BootstrapResult:
    """bootstrap.hpp:79-158 on the device."""
    cfg = cfg or BootstrapConfig()
    dds = B._dev(ds)
    J = dds.num_drugs
    c = cfg._c()
    res = bsccs_bootstrap_result()
    beta_full, lower, upper, p_hat = (np.zeros(J) for _ in range(4))
    if group is None:
        B._check(lib().bsccs_run_bootstrap(dds.handle, C.byref(c), B._ptr(beta_full), B._ptr(lower), B._ptr(upper),
                                           B._ptr(p_hat), C.byref(res)))
    else:
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        full = B.fit(dds, cfg.prior, cfg.solver)  # identical on every rank (deterministic)
        beta_full = full.beta_map
        R = int(cfg.replicates)
        r0, r1 = R * rank // world, R * (rank + 1) // world
        est = np.zeros((max(r1 - r0, 1), J))
        conv = np.zeros(max(r1 - r0, 1), np.int32)
        part = bsccs_bootstrap_result()
        if r1 > r0:
            B._check(lib().bsccs_bootstrap_replicates(dds.handle, C.byref(c),
                                                      B._ptr(beta_full) if cfg.warm_start else None, r0, r1,
                                                      B._ptr(est), B._ptr(conv), C.byref(part)))
        gathered = [None] * world
        dist.all_gather_object(gathered, (r0, r1, est[:r1 - r0], conv[:r1 - r0],
                                          (part.device_seconds, part.total_cycles, part.coordinates_visited)),
                               group=group)
        all_est = np.zeros((R, J))
        all_conv = np.zeros(R, np.int32)
        tot = [full.device_seconds, full.cycles_run, full.coordinates_visited]
        for a, b, e, cv, st in gathered:
            all_est[a:b] = e
            all_conv[a:b] = cv
            tot = [x + y for x, y in zip(tot, st)]
        B._check(lib().bsccs_bootstrap_summarize(J, R, float(cfg.level), B._ptr(all_est), B._ptr(all_conv),
                                                 B._ptr(lower), B._ptr(upper), B._ptr(p_hat), C.byref(res)))
        res.full_converged = int(full.converged)
        res.device_seconds, res.total_cycles, res.coordinates_visited = tot[0], int(tot[1]), int(tot[2])
    return BootstrapResult(beta_full, bool(res.full_converged), lower, upper, p_hat, res.replicates, res.used,
                           res.non_converged, res.device_seconds, res.total_cycles, res.coordinates_visited)


@dataclass
class RankedDrug:
    """bootstrap.hpp:160-166."""
    drug_id: str
    beta: float = 0.0
    lower: float = 0.0
    upper: float = 0.0
    p_hat: float = 0.0


def report_ranked_intervals(ds, result: BootstrapResult, min_p_hat: float = 0.5) -> List[RankedDrug]:
    """bootstrap.hpp:168-193: drugs kept in more than min_p_hat of the
    replicates, strongest full-data estimate first, label as tie-break."""
    labels = getattr(ds, "drug_ids", None) or []
    rows = []
    for j in range(len(result.p_hat)):
        if result.p_hat[j] > min_p_hat:
            rows.append(RankedDrug(labels[j] if labels else f"drug_{j}", float(result.beta_full[j]),
                                   float(result.lower[j]), float(result.upper[j]), float(result.p_hat[j])))
    rows.sort(key=lambda r: (-r.beta, r.drug_id))
    return rows
