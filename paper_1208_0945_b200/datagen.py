"""Synthetic SCCS data through the native generators (csrc/datagen.cpp).

simulate():   the reference generative model simulate() (simulate.hpp:50-137)
              -- the config-1 oracle case.
fast_sccs():  the fast generator of SURVEY §8(d) for the 1M / 10M configs
              (uniform or Zipf drug prevalence).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List

import numpy as np

from ._native import lib
from .bsccs import Dataset, _check

# SURVEY §8(d) shapes
ORACLE_SEED = 12080945
FAST_SEED = 20261017


@dataclass
class SimConfig:
    """simulate.hpp:19-31."""
    subjects: int = 1000
    drugs: int = 4
    min_eras: int = 2
    max_eras: int = 6
    min_era_length: int = 10
    max_era_length: int = 60
    prevalence: List[float] = field(default_factory=list)
    true_beta: List[float] = field(default_factory=list)
    baseline_log_rate_mean: float = -5.0
    baseline_log_rate_sd: float = 0.5
    seed: int = 0


def _take(h) -> Dataset:
    try:
        sz = (C.c_int64 * 4)()
        _check(lib().bsccs_host_dataset_sizes(h, sz))
        N, K, J, nnz = list(sz)
        ptrs = [C.c_void_p() for _ in range(8)]
        _check(lib().bsccs_host_dataset_arrays(h, *[C.byref(p) for p in ptrs]))

        def arr(p, n, dt):
            if n == 0:
                return np.zeros(0, dtype=dt)
            buf = (C.c_char * (n * np.dtype(dt).itemsize)).from_address(p.value)
            return np.frombuffer(buf, dtype=dt).copy()

        a = [arr(ptrs[0], N + 1, np.int32), arr(ptrs[1], N, np.int32), arr(ptrs[2], K, np.int32),
             arr(ptrs[3], K, np.int32), arr(ptrs[4], J + 1, np.int64), arr(ptrs[5], nnz, np.int32),
             arr(ptrs[6], nnz, np.int32), arr(ptrs[7], J, np.int64)]
        return Dataset(*a)
    finally:
        lib().bsccs_host_dataset_destroy(h)


def simulate(cfg: SimConfig) -> Dataset:
    prev = np.ascontiguousarray(cfg.prevalence, dtype=np.float64)
    tb = np.ascontiguousarray(cfg.true_beta, dtype=np.float64)
    if prev.size != cfg.drugs:
        from .bsccs import InputError
        raise InputError("simulate: prevalence must list one value per drug")
    if tb.size != cfg.drugs:
        from .bsccs import InputError
        raise InputError("simulate: true_beta must list one value per drug")
    h = C.c_void_p()
    _check(lib().bsccs_synth_simulate(cfg.subjects, cfg.drugs, cfg.min_eras, cfg.max_eras, cfg.min_era_length,
                                      cfg.max_era_length, prev.ctypes.data_as(C.c_void_p),
                                      tb.ctypes.data_as(C.c_void_p), cfg.baseline_log_rate_mean,
                                      cfg.baseline_log_rate_sd, cfg.seed & 0xFFFFFFFFFFFFFFFF, C.byref(h)))
    return _take(h)


def oracle_case_config() -> SimConfig:
    """Config 1 of BASELINE.json: 10,300 attempts x 100 drugs."""
    drugs = 100
    tb = [0.0] * drugs
    for i in range(10):
        tb[10 * i] = 0.7 if i % 2 == 0 else -0.5
    return SimConfig(subjects=10300, drugs=drugs, min_eras=10, max_eras=20, min_era_length=10, max_era_length=60,
                     prevalence=[0.02] * drugs, true_beta=tb, baseline_log_rate_mean=-5.0,
                     baseline_log_rate_sd=0.5, seed=ORACLE_SEED)


def fast_sccs(attempts: int, drugs: int, lambda_x: float = 3.0, zipf: bool = False, seed: int = FAST_SEED,
              threads: int = 0) -> Dataset:
    h = C.c_void_p()
    _check(lib().bsccs_synth_fast(int(attempts), int(drugs), float(lambda_x), int(bool(zipf)),
                                  seed & 0xFFFFFFFFFFFFFFFF, int(threads), C.byref(h)))
    return _take(h)


# named workloads of BASELINE.json configs
def config_dataset(name: str, zipf: bool = False) -> Dataset:
    if name == "oracle":
        return simulate(oracle_case_config())
    if name == "10k":
        return fast_sccs(10_300, 100, 2.0, zipf)
    if name == "1M":
        return fast_sccs(1_030_000, 1500, 3.0, zipf)
    if name == "10M":
        return fast_sccs(10_300_000, 4000, 3.0, zipf)
    raise ValueError(f"unknown workload {name}")
