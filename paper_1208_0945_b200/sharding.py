"""Patient (row) sharding of a case series across GPUs / CTA groups.

SURVEY §8(e): subjects are the independent strata and a subject's eras are
contiguous (dataset.hpp:45-48), so a contiguous subject range with its eras
and, per column, the contiguous pair sub-range of those subjects forms a
self-contained shard.  Every shard keeps the GLOBAL y_dot_x (gradient,
engine.hpp:294) and the global column counts (skip rule, solver.hpp:119-121);
the per-coordinate (sum n*w, sum n*w(1-w)) partials of all shards are
all-reduced inside the sweep kernel, so every shard takes the identical step.

Host pieces here are pure numpy (tested on CPU, incl. a gloo world-size-2
run); device binding goes through bsccs_dataset_create_shard /
bsccs_group_create_local / bsccs_group_fit.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from ._native import bsccs_fit_result, lib
from .bsccs import Dataset, DeviceDataset, FitResult, InputError, PriorSpec, SolverConfig, _check, _ptr


@dataclass
class Shard:
    """One shard: its own Dataset (subjects / eras renumbered from 0) plus
    the global per-column vectors every shard must share."""
    dataset: Dataset
    subject_begin: int
    subject_end: int
    era_begin: int
    y_dot_x_global: np.ndarray
    col_nnz_global: np.ndarray


def balanced_subject_bounds(ds: Dataset, nshards: int) -> np.ndarray:
    """Contiguous subject ranges balanced on (eras + pairs) per subject --
    the same weight the device uses to split a shard across its CTAs."""
    if nshards < 1:
        raise InputError("sharding: need at least one shard")
    N = ds.num_subjects
    off = ds.subject_offsets.astype(np.int64)
    row_cnt = np.bincount(ds.rows, minlength=ds.num_eras).astype(np.int64)
    row_cum = np.concatenate([[0], np.cumsum(row_cnt)])
    w = (off[1:] - off[:-1]) + (row_cum[off[1:]] - row_cum[off[:-1]])
    excl = np.concatenate([[0], np.cumsum(w)])
    total = int(excl[-1])
    bounds = np.empty(nshards + 1, dtype=np.int64)
    for c in range(nshards + 1):
        target = -(-total * c // nshards)  # ceil
        bounds[c] = N if c == nshards else int(np.searchsorted(excl[:-1], target, side="left"))
    bounds[0] = 0
    return bounds


def shard_dataset(ds: Dataset, nshards: int, only: Optional[int] = None) -> List[Shard]:
    """Split `ds` into `nshards` contiguous patient shards (all of them, or
    just shard `only`, as one rank of a multi-process fit needs).  A column's
    pairs are in ascending row -- hence subject -- order, so each shard's
    part of a column is one contiguous range, found by binary search."""
    bounds = balanced_subject_bounds(ds, nshards)
    J = ds.num_drugs
    cp = ds.col_ptr.astype(np.int64)
    col_nnz = np.diff(cp)
    out = []
    for r in (range(nshards) if only is None else [int(only)]):
        s0, s1 = int(bounds[r]), int(bounds[r + 1])
        e0, e1 = int(ds.subject_offsets[s0]), int(ds.subject_offsets[s1])
        lo = np.empty(J, np.int64)
        hi = np.empty(J, np.int64)
        for j in range(J):
            seg = ds.subjects[cp[j]:cp[j + 1]]
            lo[j] = cp[j] + np.searchsorted(seg, s0, side="left")
            hi[j] = cp[j] + np.searchsorted(seg, s1, side="left")
        cnt = hi - lo
        take = np.concatenate([np.arange(a, b, dtype=np.int64) for a, b in zip(lo, hi)]) if cnt.sum() else \
            np.zeros(0, np.int64)
        rows = ds.rows[take] - e0
        subs = ds.subjects[take] - s0
        col_ptr = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
        ev = ds.event_counts[ds.rows[take]].astype(np.int64)
        ydx = np.add.reduceat(ev, np.minimum(col_ptr[:-1], ev.size - 1)) if ev.size else np.zeros(J, np.int64)
        ydx = np.where(cnt > 0, ydx, 0).astype(np.int64)
        sub_ds = Dataset(ds.subject_offsets[s0:s1 + 1] - e0, ds.events_per_subject[s0:s1],
                         ds.era_lengths[e0:e1], ds.event_counts[e0:e1], col_ptr, rows, subs, y_dot_x=ydx)
        out.append(Shard(sub_ds, s0, s1, e0, ds.y_dot_x.copy(), col_nnz.copy()))
    return out


def merge_shards(shards: Sequence[Shard]) -> Dataset:
    """Inverse of shard_dataset (test helper): reassemble the global CSC."""
    J = shards[0].dataset.num_drugs
    offs, nps, lens, ys = [np.zeros(1, dtype=np.int64)], [], [], []
    rows_c = [[] for _ in range(J)]
    subs_c = [[] for _ in range(J)]
    for sh in shards:
        d = sh.dataset
        offs.append(d.subject_offsets[1:].astype(np.int64) + sh.era_begin)
        nps.append(d.events_per_subject)
        lens.append(d.era_lengths)
        ys.append(d.event_counts)
        for j in range(J):
            r, s = d.column(j)
            rows_c[j].append(r + sh.era_begin)
            subs_c[j].append(s + sh.subject_begin)
    col_ptr = np.concatenate([[0], np.cumsum([sum(len(x) for x in rows_c[j]) for j in range(J)])])
    rows = np.concatenate([np.concatenate(rc) for rc in rows_c])
    subs = np.concatenate([np.concatenate(sc) for sc in subs_c])
    return Dataset(np.concatenate(offs), np.concatenate(nps), np.concatenate(lens), np.concatenate(ys), col_ptr,
                   rows, subs, shards[0].y_dot_x_global)


def split_ctas(total_ctas: int, nshards: int) -> List[int]:
    base, extra = divmod(total_ctas, nshards)
    return [base + (1 if r < extra else 0) for r in range(nshards)]


class LocalGroup:
    """All shards on one device, one cooperative launch per cycle: the
    single-GPU execution of the cross-shard exchange protocol."""

    def __init__(self, shards: Sequence[Shard], device: int = 0, ctas_per_shard: Sequence[int] = None,
                 virtual_ranks: bool = False):
        if ctas_per_shard is None:
            from .bsccs import device_info
            ctas_per_shard = split_ctas(device_info(device)["ctas"], len(shards))
        self.shards = list(shards)
        self.devs = [DeviceDataset(sh.dataset, device, int(cc), (sh.y_dot_x_global, sh.col_nnz_global))
                     for sh, cc in zip(shards, ctas_per_shard)]
        arr = (C.c_void_p * len(self.devs))(*[d.handle for d in self.devs])
        h = C.c_void_p()
        create = lib().bsccs_group_create_virtual if virtual_ranks else lib().bsccs_group_create_local
        _check(create(arr, len(self.devs), C.byref(h)))
        self.handle = h

    def fit(self, prior: PriorSpec, cfg: SolverConfig = None, init_beta=None) -> FitResult:
        cfg = cfg or SolverConfig()
        J = self.shards[0].dataset.num_drugs
        b = None if init_beta is None else np.ascontiguousarray(init_beta, dtype=np.float64)
        beta = np.empty(J, dtype=np.float64)
        res = bsccs_fit_result()
        p, c = prior._c(), cfg._c()
        _check(lib().bsccs_group_fit(self.handle, C.byref(p), C.byref(c), _ptr(b), _ptr(beta), C.byref(res)))
        return FitResult(beta, res.log_posterior, res.cycles_run, bool(res.converged), res.final_criterion,
                         res.coordinates_visited, res.coordinates_moved, res.dense_refreshes, res.device_seconds,
                         res.sweep_seconds, res.algorithmic_bytes, res.kernel_launches)

    def close(self):
        if self.handle:
            _check(lib().bsccs_group_destroy(self.handle))
            self.handle = None
        for d in self.devs:
            d.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class RankGroup:
    """One rank of a multi-process patient-sharded fit (one GPU per process,
    launched by torchrun).  Ranks trade the CUDA IPC handle of their
    exchange area through torch.distributed; afterwards the per-coordinate
    partials travel as `red.add` into every peer's area over NVLink, inside
    the sweep kernel -- no host collective on the per-coordinate path.  The
    per-fit log-likelihood is summed exactly through the same words."""

    def __init__(self, shard: Shard, device: int, ctas: int = 0, upload_subjects: bool = True):
        import torch.distributed as dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.dds = DeviceDataset(shard.dataset, device, ctas, (shard.y_dot_x_global, shard.col_nnz_global),
                                 upload_subjects=upload_subjects)
        self.J = shard.dataset.num_drugs
        all_ctas = [None] * self.world
        dist.all_gather_object(all_ctas, self.dds.ctas)
        h = C.c_void_p()
        arr = (C.c_int32 * self.world)(*all_ctas)
        _check(lib().bsccs_group_create_rank(self.dds.handle, self.rank, self.world, arr, C.byref(h)))
        self.handle = h
        blob = (C.c_uint8 * 64)()
        _check(lib().bsccs_group_ipc_handle(h, blob))
        blobs = [None] * self.world
        dist.all_gather_object(blobs, bytes(blob))
        allb = (C.c_uint8 * (64 * self.world)).from_buffer_copy(b"".join(blobs))
        _check(lib().bsccs_group_open_peers(h, allb))
        dist.barrier()  # every exchange area zeroed and mapped before any add

    def fit(self, prior: PriorSpec, cfg: SolverConfig = None, init_beta=None) -> FitResult:
        cfg = cfg or SolverConfig()
        b = None if init_beta is None else np.ascontiguousarray(init_beta, dtype=np.float64)
        beta = np.empty(self.J, dtype=np.float64)
        res = bsccs_fit_result()
        p, c = prior._c(), cfg._c()
        _check(lib().bsccs_group_fit(self.handle, C.byref(p), C.byref(c), _ptr(b), _ptr(beta), C.byref(res)))
        return FitResult(beta, res.log_posterior, res.cycles_run, bool(res.converged), res.final_criterion,
                         res.coordinates_visited, res.coordinates_moved, res.dense_refreshes, res.device_seconds,
                         res.sweep_seconds, res.algorithmic_bytes, res.kernel_launches)

    def close(self):
        import torch.distributed as dist
        if self.handle:
            dist.barrier()  # nobody still adds into our area
            _check(lib().bsccs_group_destroy(self.handle))
            self.handle = None
        self.dds.close()
