"""Python mirror of the reference `bsccs` engine/solver API over the C ABI.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/bsccs/): Dataset / build_dataset /
subset_dataset (dataset.hpp), init_state / dense_recompute /
fused_grad_hess / sparse_delta_update / log_likelihood (engine.hpp),
PriorSpec / log_density / penalized_step (prior.hpp), SolverConfig /
SolverState / run_cycle / fit / FitResult (solver.hpp), and the four
exception types (common.hpp:10-35).  All arithmetic runs in
libbsccs_b200.so (device kernels for the engine, the same C++ as the
kernels for the prior); this module only marshals arrays.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native
from ._native import bsccs_fit_result, bsccs_prior, bsccs_solver_config, lib

# ---------------------------------------------------------------- errors


class InputError(RuntimeError):
    """bsccs::input_error (common.hpp:11-14)."""


class NumericError(RuntimeError):
    """bsccs::numeric_error (common.hpp:18-21)."""


class ConvergenceError(RuntimeError):
    """bsccs::convergence_error (common.hpp:26-29)."""


class InternalError(RuntimeError):
    """bsccs::internal_error (common.hpp:32-35)."""


class CudaError(RuntimeError):
    """CUDA runtime failure (no reference analogue)."""


_STATUS = {1: InputError, 2: NumericError, 3: InternalError, 4: ConvergenceError, 5: CudaError}


def _check(rc: int) -> None:
    if rc:
        raise _STATUS.get(rc, InternalError)(lib().bsccs_last_error().decode(errors="replace"))


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------- prior / config


class PriorKind(enum.IntEnum):
    none = 0
    normal = 1
    laplace = 2


class ConvergenceMode(enum.IntEnum):
    raw_sum = 0
    normalized = 1


class Precision(enum.IntEnum):
    Single = 0
    Double = 1


class UpdatePath(enum.IntEnum):
    sparse = 0
    dense = 1


@dataclass
class PriorSpec:
    """prior.hpp:17-25."""
    kind: PriorKind = PriorKind.none
    variance: float = 1.0
    variance_is_laplace_scale: bool = False

    def laplace_scale(self) -> float:
        return self.variance if self.variance_is_laplace_scale else float(np.sqrt(self.variance / 2.0))

    def _c(self) -> bsccs_prior:
        return bsccs_prior(int(self.kind), int(bool(self.variance_is_laplace_scale)), float(self.variance))


def normal_prior(variance: float) -> PriorSpec:
    return PriorSpec(PriorKind.normal, variance)


def laplace_prior(variance: float) -> PriorSpec:
    return PriorSpec(PriorKind.laplace, variance)


@dataclass
class SolverConfig:
    """solver.hpp:21-46 (defaults identical)."""
    epsilon: float = 0.0005
    max_cycles: int = 1000
    trust_init: float = 1.0
    convergence: ConvergenceMode = ConvergenceMode.raw_sum
    precision: Precision = Precision.Double
    path: UpdatePath = UpdatePath.sparse
    partitions: int = 1
    dense_refresh_interval: int = 50
    random_cycle: bool = False
    cycle_seed: int = 0
    min_parallel_nnz: int = 4096

    def _c(self) -> bsccs_solver_config:
        c = bsccs_solver_config()
        c.epsilon = self.epsilon
        c.max_cycles = self.max_cycles
        c.convergence = int(self.convergence)
        c.trust_init = self.trust_init
        c.precision = int(self.precision)
        c.path = int(self.path)
        c.partitions = self.partitions
        c.dense_refresh_interval = self.dense_refresh_interval
        c.random_cycle = int(bool(self.random_cycle))
        c.cycle_seed = self.cycle_seed & 0xFFFFFFFFFFFFFFFF
        c.min_parallel_nnz = self.min_parallel_nnz
        return c


@dataclass
class FitResult:
    """solver.hpp:66-72, plus device instrumentation."""
    beta_map: np.ndarray
    log_posterior: float = float("-inf")
    cycles_run: int = 0
    converged: bool = False
    final_criterion: float = float("inf")
    coordinates_visited: int = 0
    coordinates_moved: int = 0
    dense_refreshes: int = 0
    device_seconds: float = 0.0
    sweep_seconds: float = 0.0
    algorithmic_bytes: float = 0.0
    kernel_launches: int = 0


@dataclass
class GradHess:
    """engine.hpp:49-52."""
    gradient: float = 0.0
    hessian: float = 0.0


def penalized_step(prior: PriorSpec, beta_j: float, g: float, h: float) -> float:
    """prior.hpp:72-122 -- evaluated by the same C++ the sweep kernel runs."""
    out = C.c_double()
    p = prior._c()
    _check(lib().bsccs_penalized_step(C.byref(p), float(beta_j), float(g), float(h), C.byref(out)))
    return out.value


def log_density(prior: PriorSpec, beta: Sequence[float]) -> float:
    """prior.hpp:36-61."""
    b = np.ascontiguousarray(beta, dtype=np.float64)
    out = C.c_double()
    p = prior._c()
    _check(lib().bsccs_log_density(C.byref(p), _ptr(b), int(b.size), C.byref(out)))
    return out.value


def validate_prior(prior: PriorSpec) -> None:
    """prior.hpp:27-32."""
    if prior.kind != PriorKind.none and not (prior.variance > 0.0 and np.isfinite(prior.variance)):
        raise InputError("prior variance must be positive and finite")


# ---------------------------------------------------------------- RNG


class Rng:
    """xoshiro256** seeded through splitmix64 (rng.hpp:30-124): the stream
    behind SolverState::order_rng (solver.hpp:81) for shuffled cycles."""

    M64 = 0xFFFFFFFFFFFFFFFF

    def __init__(self, seed: int, stream: int = 0):
        a, b = seed & self.M64, (~stream) & self.M64
        s = []
        for _ in range(4):
            a, za = self._sm(a)
            b, zb = self._sm(b)
            s.append(za ^ zb)
        if not any(s):
            s[0] = 0x9E3779B97F4A7C15
        self.s = s

    @classmethod
    def _sm(cls, state):
        state = (state + 0x9E3779B97F4A7C15) & cls.M64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & cls.M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & cls.M64
        return state, z ^ (z >> 31)

    @classmethod
    def _rotl(cls, x, k):
        return ((x << k) | (x >> (64 - k))) & cls.M64

    def next(self) -> int:
        s = self.s
        out = (self._rotl((s[1] * 5) & self.M64, 7) * 9) & self.M64
        t = (s[1] << 17) & self.M64
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = self._rotl(s[3], 45)
        return out

    def uniform(self) -> float:
        return float(self.next() >> 11) * 2.0 ** -53

    def below(self, n: int) -> int:
        if n <= 0:
            raise InternalError("Rng::below requires n > 0")
        while True:
            x = self.next()
            r = x % n
            if not (x - r > ((0 - n) & self.M64)):
                return r

    def uniform_int(self, lo: int, hi: int) -> int:
        return lo + self.below(hi - lo + 1)


# ---------------------------------------------------------------- dataset


@dataclass
class Era:
    """dataset.hpp:20-27."""
    length_days: int = 0
    event_count: int = 0
    exposures: Sequence[int] = field(default_factory=list)


@dataclass
class SubjectRecord:
    """dataset.hpp:29-34."""
    subject_id: str
    eras: Sequence[Era]


class Dataset:
    """Host form of bsccs::Dataset (dataset.hpp:53-68), flat CSC.

    Column j's pairs are [col_ptr[j], col_ptr[j+1]) of `rows` / `subjects`
    (SparseColumn::rows / ::subjects concatenated)."""

    def __init__(self, subject_offsets, events_per_subject, era_lengths, event_counts, col_ptr, rows, subjects,
                 y_dot_x=None, drug_ids=None):
        self.subject_offsets = np.ascontiguousarray(subject_offsets, dtype=np.int32)
        self.events_per_subject = np.ascontiguousarray(events_per_subject, dtype=np.int32)
        self.era_lengths = np.ascontiguousarray(era_lengths, dtype=np.int32)
        self.event_counts = np.ascontiguousarray(event_counts, dtype=np.int32)
        self.col_ptr = np.ascontiguousarray(col_ptr, dtype=np.int64)
        self.rows = np.ascontiguousarray(rows, dtype=np.int32)
        self.subjects = np.ascontiguousarray(subjects, dtype=np.int32)
        if y_dot_x is None:
            pair_col = np.repeat(np.arange(self.num_drugs), np.diff(self.col_ptr))
            y_dot_x = np.bincount(pair_col, weights=self.event_counts[self.rows],
                                  minlength=self.num_drugs).astype(np.int64)
        self.y_dot_x = np.ascontiguousarray(y_dot_x, dtype=np.int64)
        self.drug_ids = list(drug_ids) if drug_ids else []
        self._device = {}

    num_subjects = property(lambda s: int(s.subject_offsets.size - 1))
    num_eras = property(lambda s: int(s.era_lengths.size))
    num_drugs = property(lambda s: int(s.col_ptr.size - 1))
    nnz = property(lambda s: int(s.rows.size))
    max_column_nnz = property(lambda s: int(np.diff(s.col_ptr).max(initial=0)))

    def column(self, j: int):
        a, b = self.col_ptr[j], self.col_ptr[j + 1]
        return self.rows[a:b], self.subjects[a:b]

    def arrays(self):
        return (self.subject_offsets, self.events_per_subject, self.era_lengths, self.event_counts, self.col_ptr,
                self.rows, self.subjects, self.y_dot_x)

    def on_device(self, device: int = 0, ctas: int = 0) -> "DeviceDataset":
        key = (device, ctas)
        if key not in self._device:
            self._device[key] = DeviceDataset(self, device, ctas)
        return self._device[key]

    def __eq__(self, other):
        return isinstance(other, Dataset) and all(np.array_equal(a, b) for a, b in zip(self.arrays(), other.arrays()))


def build_dataset(records: Sequence[SubjectRecord], num_drugs: int, drug_ids=None) -> Dataset:
    """dataset.hpp:74-152: validate eras, drop zero-event subjects, CSC with
    ascending rows per column, y_dot_x."""
    if num_drugs < 1:
        raise InputError("build_dataset: need at least one drug")
    if drug_ids and len(drug_ids) != num_drugs:
        raise InputError("build_dataset: drug label count does not match drug count")
    offsets, nps, lens, ys = [0], [], [], []
    cols = [[] for _ in range(num_drugs)]
    csub = [[] for _ in range(num_drugs)]
    row = 0
    nsub = 0
    for rec in records:
        total = 0
        for era in rec.eras:
            if era.length_days <= 0:
                raise InputError(f"subject '{rec.subject_id}': era length must be positive")
            if era.event_count < 0:
                raise InputError(f"subject '{rec.subject_id}': negative event count")
            prev = -1
            for j in era.exposures:
                if j < 0 or j >= num_drugs:
                    raise InputError(f"subject '{rec.subject_id}': exposure index {j} out of range")
                if j <= prev:
                    raise InputError(f"subject '{rec.subject_id}': exposure indices must be strictly ascending")
                prev = j
            total += era.event_count
        if total == 0:
            continue
        for era in rec.eras:
            lens.append(era.length_days)
            ys.append(era.event_count)
            for j in era.exposures:
                cols[j].append(row)
                csub[j].append(nsub)
            row += 1
        offsets.append(row)
        nps.append(total)
        nsub += 1
    if nsub == 0:
        raise InputError("build_dataset: no subjects with events remain after exclusion")
    col_ptr = np.zeros(num_drugs + 1, dtype=np.int64)
    col_ptr[1:] = np.cumsum([len(c) for c in cols])
    rows = np.array([r for c in cols for r in c], dtype=np.int32)
    subs = np.array([s for c in csub for s in c], dtype=np.int32)
    return Dataset(offsets, nps, lens, ys, col_ptr, rows, subs, None, drug_ids)


def subset_dataset(ds: Dataset, subject_indices: Sequence[int]) -> Dataset:
    """dataset.hpp:157-217: rebuild over the selection in the given order;
    repeated indices become independent copies; columns keep ascending rows."""
    sel = np.asarray(subject_indices, dtype=np.int64)
    if sel.size == 0:
        raise InputError("subset_dataset: empty subject selection")
    if (sel < 0).any() or (sel >= ds.num_subjects).any():
        raise InputError("subset_dataset: subject index out of range")
    off = ds.subject_offsets.astype(np.int64)
    cnt = off[sel + 1] - off[sel]
    new_start = np.concatenate([[0], np.cumsum(cnt)])
    src = np.repeat(off[sel] - new_start[:-1], cnt) + np.arange(new_start[-1])  # source era of each output era
    out_sub = np.repeat(np.arange(sel.size), cnt)
    J = ds.num_drugs
    pair_col = np.repeat(np.arange(J), np.diff(ds.col_ptr))
    o = np.argsort(ds.rows, kind="stable")  # by row, then column ascending
    col_by_row = pair_col[o]
    row_ptr = np.searchsorted(ds.rows[o], np.arange(ds.num_eras + 1))
    n_per = row_ptr[src + 1] - row_ptr[src]
    excl = np.concatenate([[0], np.cumsum(n_per)])[:-1]
    pos = np.repeat(row_ptr[src] - excl, n_per) + np.arange(int(n_per.sum()))
    new_row = np.repeat(np.arange(src.size), n_per)
    col = col_by_row[pos]
    order = np.lexsort((new_row, col))
    new_row, col = new_row[order], col[order]
    col_ptr = np.concatenate([[0], np.cumsum(np.bincount(col, minlength=J))])
    ydx = np.bincount(col, weights=ds.event_counts[src[new_row]], minlength=J).astype(np.int64)
    return Dataset(new_start, ds.events_per_subject[sel], ds.era_lengths[src], ds.event_counts[src], col_ptr,
                   new_row, out_sub[new_row], ydx, ds.drug_ids)


def kfold_split(ds, folds: int, seed: int) -> List[np.ndarray]:
    """cross_validation.hpp:58-80: seeded Fisher-Yates over subject ids,
    dealt round-robin into `folds` lists (the reference's order)."""
    n = ds.num_subjects
    out = np.empty(n, dtype=np.int32)
    sizes = np.empty(max(int(folds), 0), dtype=np.int32)
    _check(lib().bsccs_kfold_split(n, int(folds), int(seed) & (2**64 - 1), _ptr(out), _ptr(sizes)))
    return np.split(out, np.cumsum(sizes)[:-1])


def resample(ds, seed: int, stream: int = 0) -> np.ndarray:
    """bootstrap.hpp:43-52 with the generator Rng(seed, stream)."""
    n = ds.num_subjects
    out = np.empty(n, dtype=np.int32)
    _check(lib().bsccs_resample(n, int(seed) & (2**64 - 1), int(stream) & (2**64 - 1), _ptr(out)))
    return out


def read_long_format(path: str, dictionary: Optional[Sequence[str]] = None, device: int = 0, ctas: int = 0,
                     threads: int = 0) -> "DeviceDataset":
    """io.hpp:88-174 + dataset.hpp:74-152: the era-level long format parsed
    by native host threads and laid out as CSC on the device."""
    h = C.c_void_p()
    d = None
    n = 0
    if dictionary:
        d = (C.c_char_p * len(dictionary))(*[x.encode() for x in dictionary])
        n = len(dictionary)
    _check(lib().bsccs_dataset_read_long_format(str(path).encode(), d, n, device, ctas, threads, C.byref(h)))
    return DeviceDataset(None, device, ctas, handle=h)


def write_long_format(path: str, records: Sequence[SubjectRecord], drug_ids: Sequence[str]) -> None:
    """io.hpp:176-196: one era per line, subject, length, events, labels."""
    with open(path, "w") as out:
        for rec in records:
            for era in rec.eras:
                out.write(f"{rec.subject_id}\t{era.length_days}\t{era.event_count}\t"
                          + " ".join(drug_ids[j] for j in era.exposures) + "\n")


# ---------------------------------------------------------------- device


class DeviceDataset:
    """Device-resident dataset handle (bsccs_dataset_create)."""

    def __init__(self, ds: Optional[Dataset], device: int = 0, ctas: int = 0, shard_globals=None, handle=None,
                 upload_subjects: bool = True):
        """upload_subjects=False passes NULL for the per-pair subjects: the
        device derives them from the rows (each era's owner) instead of
        copying them, and their agreement with the rows is then not checked."""
        self.host = ds
        self.device = device
        if handle is not None:  # built on the device (subset)
            self.handle = handle
            self._sizes = None
            return
        h = C.c_void_p()
        a = [_ptr(x) for x in ds.arrays()]
        if not upload_subjects:
            a[6] = None
        if shard_globals is None:
            _check(lib().bsccs_dataset_create(ds.num_subjects, ds.num_eras, ds.num_drugs, ds.nnz,
                                              *a, device, ctas, C.byref(h)))
        else:
            ydx, cnnz = (np.ascontiguousarray(x, dtype=np.int64) for x in shard_globals)
            _check(lib().bsccs_dataset_create_shard(ds.num_subjects, ds.num_eras, ds.num_drugs, ds.nnz,
                                                    *a[:7], _ptr(ydx), _ptr(cnnz), device, ctas,
                                                    C.byref(h)))
        self.handle = h
        self._sizes = None
        if ds.drug_ids:
            labels = (C.c_char_p * len(ds.drug_ids))(*[x.encode() for x in ds.drug_ids])
            _check(lib().bsccs_dataset_set_drug_ids(h, labels, len(ds.drug_ids)))

    def info(self):
        out = (C.c_int64 * 6)()
        _check(lib().bsccs_dataset_info(self.handle, out))
        return dict(zip(["N", "K", "J", "nnz", "ctas", "device_bytes"], list(out)))

    @property
    def ctas(self) -> int:
        return self.info()["ctas"]

    def _size(self, k):
        if self._sizes is None:
            self._sizes = self.info()
        return int(self._sizes[k])

    num_subjects = property(lambda s: s._size("N"))
    num_eras = property(lambda s: s._size("K"))
    num_drugs = property(lambda s: s._size("J"))
    nnz = property(lambda s: s._size("nnz"))

    @property
    def drug_ids(self) -> List[str]:
        """Dataset::drug_ids (dataset.hpp:66) held with the device copy."""
        need = C.c_int64()
        _check(lib().bsccs_dataset_drug_ids(self.handle, None, 0, C.byref(need)))
        buf = C.create_string_buffer(max(int(need.value), 1))
        _check(lib().bsccs_dataset_drug_ids(self.handle, buf, len(buf), None))
        txt = buf.value.decode()
        return txt.split("\n") if txt else []

    def subset(self, subject_indices: Sequence[int], ctas: int = 0) -> "DeviceDataset":
        """subset_dataset (dataset.hpp:157-217) built on the device."""
        sel = np.ascontiguousarray(subject_indices, dtype=np.int32)
        h = C.c_void_p()
        _check(lib().bsccs_dataset_subset(self.handle, _ptr(sel), sel.size, ctas, C.byref(h)))
        return DeviceDataset(None, self.device, ctas, handle=h)

    def to_host(self) -> Dataset:
        """Flat CSC arrays copied back from the device."""
        n = self.info()
        N, K, J, nnz = n["N"], n["K"], n["J"], n["nnz"]
        arr = [np.empty(N + 1, np.int32), np.empty(N, np.int32), np.empty(K, np.int32), np.empty(K, np.int32),
               np.empty(J + 1, np.int64), np.empty(nnz, np.int32), np.empty(nnz, np.int32), np.empty(J, np.int64)]
        _check(lib().bsccs_dataset_export(self.handle, *[_ptr(a) for a in arr]))
        return Dataset(*arr, drug_ids=self.drug_ids)

    def close(self):
        if self.handle:
            _check(lib().bsccs_dataset_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _dev(ds) -> DeviceDataset:
    if isinstance(ds, DeviceDataset):
        return ds
    if isinstance(ds, Dataset):
        return ds.on_device()
    raise InputError("expected a Dataset or DeviceDataset")


class EngineState:
    """EngineState<double> (engine.hpp:36-45) held on the device."""

    def __init__(self, dds: DeviceDataset, handle):
        self.dds = dds
        self.handle = handle

    def _get(self, which):
        ds = self.dds
        n = {"beta": ds.num_drugs, "xbeta": ds.num_eras, "l_exp_xbeta": ds.num_eras,
             "denominators": ds.num_subjects}[which]
        out = np.empty(n, dtype=np.float64)
        args = [None] * 4
        args[["beta", "xbeta", "l_exp_xbeta", "denominators"].index(which)] = _ptr(out)
        _check(lib().bsccs_state_get(self.handle, *args))
        return out

    beta = property(lambda s: s._get("beta"))
    xbeta = property(lambda s: s._get("xbeta"))
    l_exp_xbeta = property(lambda s: s._get("l_exp_xbeta"))
    denominators = property(lambda s: s._get("denominators"))

    def copy(self) -> "EngineState":
        h = C.c_void_p()
        _check(lib().bsccs_state_clone(self.handle, C.byref(h)))
        return EngineState(self.dds, h)

    def close(self):
        if self.handle:
            _check(lib().bsccs_state_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def init_state(ds, beta: Optional[Sequence[float]] = None) -> EngineState:
    """engine.hpp:137-166."""
    dds = _dev(ds)
    b = None
    if beta is not None and len(beta) > 0:
        b = np.ascontiguousarray(beta, dtype=np.float64)
        if b.size != dds.num_drugs:
            raise InputError("init_state: coefficient count does not match drug count")
    h = C.c_void_p()
    _check(lib().bsccs_state_create(dds.handle, _ptr(b), C.byref(h)))
    return EngineState(dds, h)


def dense_recompute(ds, state: EngineState, beta: Optional[Sequence[float]] = None) -> None:
    """engine.hpp:170-200."""
    b = None
    if beta is not None:
        b = np.ascontiguousarray(beta, dtype=np.float64)
        if b.size != state.dds.num_drugs:
            raise InputError("dense_recompute: coefficient count does not match state")
    _check(lib().bsccs_dense_recompute(state.handle, _ptr(b)))


def fused_grad_hess(ds, state: EngineState, j: int) -> GradHess:
    """engine.hpp:285-298."""
    g, h = C.c_double(), C.c_double()
    _check(lib().bsccs_grad_hess(state.handle, int(j), C.byref(g), C.byref(h)))
    return GradHess(g.value, h.value)


def parallel_fused_grad_hess(ds, state: EngineState, j: int, partitions: int = 1, pool=None,
                             min_chunk: int = 4096) -> GradHess:
    """engine.hpp:305-361.  The device reduction is always partitioned (one
    subject-aligned slice per CTA, fixed-order combine), so `partitions` only
    keeps the reference's validation."""
    if partitions < 1:
        raise InputError("parallel_fused_grad_hess: partitions must be >= 1")
    return fused_grad_hess(ds, state, j)


def sparse_delta_update(ds, state: EngineState, j: int, delta: float) -> None:
    """engine.hpp:205-231."""
    _check(lib().bsccs_sparse_update(state.handle, int(j), float(delta)))


def log_likelihood(ds, state: EngineState) -> float:
    """engine.hpp:404-425."""
    out = C.c_double()
    _check(lib().bsccs_log_likelihood(state.handle, C.byref(out)))
    return out.value


# ---------------------------------------------------------------- solver


def validate_config(cfg: SolverConfig) -> None:
    """solver.hpp:48-64."""
    if not (cfg.epsilon > 0.0) or not np.isfinite(cfg.epsilon):
        raise InputError("solver: epsilon must be positive and finite")
    if cfg.max_cycles < 1:
        raise InputError("solver: max_cycles must be at least 1")
    if not (cfg.trust_init > 0.0) or not np.isfinite(cfg.trust_init):
        raise InputError("solver: trust region width must be positive and finite")
    if cfg.partitions < 1:
        raise InputError("solver: partitions must be at least 1")
    if cfg.dense_refresh_interval < 1:
        raise InputError("solver: dense refresh interval must be at least 1")


class SolverState:
    """solver.hpp:76-93: trust radii, visit order, cycle count, order RNG."""

    def __init__(self, ds, cfg: SolverConfig):
        J = _dev(ds).num_drugs
        self.trust = np.full(J, cfg.trust_init, dtype=np.float64)
        self.order = np.arange(J, dtype=np.int32)
        self.order_rng = Rng(cfg.cycle_seed)
        self.cycle = 0


def run_cycle(ds, state: EngineState, solver: SolverState, prior: PriorSpec, cfg: SolverConfig,
              pool=None) -> float:
    """solver.hpp:101-166 as one persistent-kernel sweep."""
    if cfg.random_cycle:
        order = solver.order
        for j in range(order.size, 1, -1):
            r = solver.order_rng.below(j)
            order[j - 1], order[r] = order[r], order[j - 1]
    crit = C.c_double()
    p, c = prior._c(), cfg._c()
    order = solver.order if cfg.random_cycle else None
    _check(lib().bsccs_run_cycle(state.handle, C.byref(p), C.byref(c), _ptr(order), _ptr(solver.trust),
                                 C.byref(crit)))
    solver.cycle += 1
    return crit.value


def fit(ds, prior: PriorSpec, cfg: Optional[SolverConfig] = None, init_beta: Optional[Sequence[float]] = None,
        pool=None) -> FitResult:
    """solver.hpp:206-220 on the device (dataset uploaded once and cached)."""
    cfg = cfg or SolverConfig()
    dds = _dev(ds)
    J = dds.num_drugs
    b = None
    if init_beta is not None and len(init_beta) > 0:
        b = np.ascontiguousarray(init_beta, dtype=np.float64)
        if b.size != J:
            raise InputError("init_state: coefficient count does not match drug count")
    beta = np.empty(J, dtype=np.float64)
    res = bsccs_fit_result()
    p, c = prior._c(), cfg._c()
    _check(lib().bsccs_fit(dds.handle, C.byref(p), C.byref(c), _ptr(b), _ptr(beta), C.byref(res)))
    return FitResult(beta, res.log_posterior, res.cycles_run, bool(res.converged), res.final_criterion,
                     res.coordinates_visited, res.coordinates_moved, res.dense_refreshes, res.device_seconds,
                     res.sweep_seconds, res.algorithmic_bytes, res.kernel_launches)


def fit_batch(ds, priors: Sequence[PriorSpec], weights=None, init_betas=None,
              cfg: Optional[SolverConfig] = None):
    """R <= 16 fits in one batched launch per cycle (bsccs_fit_batch): fit r
    weights subject i by weights[r][i] (its multiplicity in a selection; 0
    leaves it out).  Returns (list of FitResult, list of per-fit status) --
    a failed fit carries its exception class instead of stopping the batch."""
    cfg = cfg or SolverConfig()
    dds = _dev(ds)
    R, J, N = len(priors), dds.num_drugs, dds.num_subjects
    pr = (bsccs_prior * max(R, 1))(*[p._c() for p in priors])
    w = None if weights is None else np.ascontiguousarray(weights, dtype=np.int32).reshape(R, N)
    b0 = None if init_betas is None else np.ascontiguousarray(init_betas, dtype=np.float64).reshape(R, J)
    beta = np.zeros((max(R, 1), J))
    res = (bsccs_fit_result * max(R, 1))()
    st = np.zeros(max(R, 1), dtype=np.int32)
    c = cfg._c()
    _check(lib().bsccs_fit_batch(dds.handle, R, pr, _ptr(w), _ptr(b0), C.byref(c), _ptr(beta), res, _ptr(st)))
    out = []
    for r in range(R):
        x = res[r]
        out.append(FitResult(beta[r].copy(), x.log_posterior, x.cycles_run, bool(x.converged), x.final_criterion,
                             x.coordinates_visited, x.coordinates_moved, x.dense_refreshes, x.device_seconds,
                             x.sweep_seconds, x.algorithmic_bytes, x.kernel_launches))
    return out, [None if s == 0 else _STATUS.get(int(s), InternalError) for s in st[:R]]


def launch_count() -> int:
    return int(lib().bsccs_launch_count())


def device_info(device: int = 0):
    sms, ctas = C.c_int32(), C.c_int32()
    _check(lib().bsccs_device_info(device, C.byref(sms), C.byref(ctas)))
    return {"sm_count": sms.value, "ctas": ctas.value}
