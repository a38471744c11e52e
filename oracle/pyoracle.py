"""TEST INFRASTRUCTURE ONLY -- ctypes access to the parity checkers.

  Port  : oracle/build/liboracle.so   (C restatement, ccd_oracle.c)
  Ref   : oracle/_ref/libbsccs_ref.so (the reference headers themselves,
          compiled by oracle/Makefile from /root/reference/proj/include)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module.  The product path (paper_1208_0945_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_LIB = HERE / "build" / "liboracle.so"
REF_LIB = HERE / "_ref" / "libbsccs_ref.so"

i32, i64, f64, u64 = C.c_int32, C.c_int64, C.c_double, C.c_uint64
VP = C.c_void_p


def _p(a):
    return None if a is None else a.ctypes.data_as(VP)


class OrDataset(C.Structure):
    _fields_ = [("N", i32), ("K", i32), ("J", i32), ("nnz", i64)] + [(n, VP) for n in (
        "subject_offsets", "events_per_subject", "era_lengths", "event_counts", "col_ptr", "rows", "subjects",
        "y_dot_x")]


class OrState(C.Structure):
    _fields_ = [("beta", VP), ("xbeta", VP), ("l_exp_xbeta", VP), ("denominators", VP)]


class OrPrior(C.Structure):
    _fields_ = [("kind", i32), ("variance_is_laplace_scale", i32), ("variance", f64)]


class OrConfig(C.Structure):
    _fields_ = [("epsilon", f64), ("max_cycles", i32), ("normalized", i32), ("trust_init", f64),
                ("dense_refresh_interval", i32), ("random_cycle", i32), ("cycle_seed", u64)]


class OrResult(C.Structure):
    _fields_ = [("log_posterior", f64), ("final_criterion", f64), ("cycles_run", i32), ("converged", i32),
                ("coordinates_visited", i64)]


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def available_ref() -> bool:
    return REF_LIB.exists()


# ---------------------------------------------------------------- C port

class Port:
    """The plain-C restatement (parity checker, bit-for-bit with the reference)."""

    def __init__(self):
        if not PORT_LIB.exists():
            raise ImportError(f"{PORT_LIB} missing: run `make -C oracle oracle`")
        self.lib = C.CDLL(str(PORT_LIB))
        self.lib.or_last_error.restype = C.c_char_p

    def _chk(self, rc):
        if rc:
            raise OracleError(rc, self.lib.or_last_error().decode())

    @staticmethod
    def _ds(ds):
        keep = ds.arrays()
        d = OrDataset(ds.num_subjects, ds.num_eras, ds.num_drugs, ds.nnz, *[_p(a) for a in keep])
        return d, keep

    def new_state(self, ds):
        arrs = dict(beta=np.zeros(ds.num_drugs), xbeta=np.zeros(ds.num_eras), l_exp_xbeta=np.zeros(ds.num_eras),
                    denominators=np.zeros(ds.num_subjects))
        st = OrState(*[_p(arrs[k]) for k in ("beta", "xbeta", "l_exp_xbeta", "denominators")])
        return st, arrs

    def init_state(self, ds, beta=None):
        d, keep = self._ds(ds)
        st, arrs = self.new_state(ds)
        b = None if beta is None else np.ascontiguousarray(beta, dtype=np.float64)
        self._chk(self.lib.or_init_state(C.byref(d), _p(b), C.byref(st)))
        return arrs

    def _st(self, arrs):
        return OrState(*[_p(arrs[k]) for k in ("beta", "xbeta", "l_exp_xbeta", "denominators")])

    def grad_hess(self, ds, arrs, j):
        d, keep = self._ds(ds)
        st = self._st(arrs)
        g, h = f64(), f64()
        self._chk(self.lib.or_grad_hess(C.byref(d), C.byref(st), i32(j), C.byref(g), C.byref(h)))
        return g.value, h.value

    def sparse_update(self, ds, arrs, j, delta):
        d, keep = self._ds(ds)
        st = self._st(arrs)
        self._chk(self.lib.or_sparse_update(C.byref(d), C.byref(st), i32(j), f64(delta)))

    def dense_recompute(self, ds, arrs):
        d, keep = self._ds(ds)
        st = self._st(arrs)
        self._chk(self.lib.or_dense_recompute(C.byref(d), C.byref(st)))

    def log_likelihood(self, ds, arrs):
        d, keep = self._ds(ds)
        st = self._st(arrs)
        out = f64()
        self._chk(self.lib.or_log_likelihood(C.byref(d), C.byref(st), C.byref(out)))
        return out.value

    def penalized_step(self, prior, beta_j, g, h):
        p = OrPrior(int(prior.kind), int(prior.variance_is_laplace_scale), float(prior.variance))
        out = f64()
        self._chk(self.lib.or_penalized_step(C.byref(p), f64(beta_j), f64(g), f64(h), C.byref(out)))
        return out.value

    def fit(self, ds, prior, cfg, init_beta=None):
        d, keep = self._ds(ds)
        p = OrPrior(int(prior.kind), int(prior.variance_is_laplace_scale), float(prior.variance))
        c = OrConfig(cfg.epsilon, cfg.max_cycles, int(cfg.convergence), cfg.trust_init, cfg.dense_refresh_interval,
                     int(cfg.random_cycle), cfg.cycle_seed)
        beta = np.zeros(ds.num_drugs)
        b = None if init_beta is None else np.ascontiguousarray(init_beta, dtype=np.float64)
        r = OrResult()
        self._chk(self.lib.or_fit(C.byref(d), C.byref(p), C.byref(c), _p(b), _p(beta), C.byref(r)))
        return dict(beta=beta, log_posterior=r.log_posterior, cycles_run=r.cycles_run, converged=bool(r.converged),
                    final_criterion=r.final_criterion, coordinates_visited=r.coordinates_visited)


# ---------------------------------------------------------------- reference

class _CPrior(C.Structure):
    _fields_ = [("kind", i32), ("variance_is_laplace_scale", i32), ("variance", f64)]


class _CCfg(C.Structure):
    _fields_ = [("epsilon", f64), ("max_cycles", i32), ("convergence", i32), ("trust_init", f64),
                ("precision", i32), ("path", i32), ("partitions", i32), ("dense_refresh_interval", i32),
                ("random_cycle", i32), ("reserved0", i32), ("cycle_seed", u64), ("min_parallel_nnz", u64)]


class _CRes(C.Structure):
    _fields_ = [("log_posterior", f64), ("final_criterion", f64), ("cycles_run", i32), ("converged", i32),
                ("coordinates_visited", i64), ("coordinates_moved", i64), ("dense_refreshes", i64),
                ("device_seconds", f64), ("sweep_seconds", f64), ("algorithmic_bytes", f64),
                ("kernel_launches", i64)]


def _cprior(prior):
    return _CPrior(int(prior.kind), int(prior.variance_is_laplace_scale), float(prior.variance))


def _ccfg(cfg):
    return _CCfg(cfg.epsilon, cfg.max_cycles, int(cfg.convergence), cfg.trust_init, int(cfg.precision),
                 int(cfg.path), cfg.partitions, cfg.dense_refresh_interval, int(cfg.random_cycle), 0,
                 cfg.cycle_seed, cfg.min_parallel_nnz)


class Reference:
    """The reference itself (bsccs headers compiled untouched)."""

    def __init__(self):
        if not REF_LIB.exists():
            raise ImportError(f"{REF_LIB} missing: run `make -C oracle ref` where /root/reference exists")
        self.lib = C.CDLL(str(REF_LIB))
        self.lib.ref_last_error.restype = C.c_char_p
        self.lib.ref_dataset_nnz.restype = i64

    def _chk(self, rc):
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def dataset(self, ds):
        h = VP()
        a = ds.arrays()
        self._chk(self.lib.ref_dataset_create(i32(ds.num_subjects), i32(ds.num_eras), i32(ds.num_drugs),
                                              i64(ds.nnz), *[_p(x) for x in a], C.byref(h)))
        return RefDataset(self, h)

    def simulate(self, cfg):
        prev = np.ascontiguousarray(cfg.prevalence, dtype=np.float64)
        tb = np.ascontiguousarray(cfg.true_beta, dtype=np.float64)
        h = VP()
        self._chk(self.lib.ref_simulate(i32(cfg.subjects), i32(cfg.drugs), i32(cfg.min_eras), i32(cfg.max_eras),
                                        i32(cfg.min_era_length), i32(cfg.max_era_length), _p(prev), _p(tb),
                                        f64(cfg.baseline_log_rate_mean), f64(cfg.baseline_log_rate_sd),
                                        u64(cfg.seed), C.byref(h)))
        return RefDataset(self, h)

    def read_long_format(self, path, dictionary=None):
        """reference read_long_format + build_dataset -> (RefDataset, labels)"""
        d = None
        n = 0
        if dictionary:
            d = (C.c_char_p * len(dictionary))(*[x.encode() for x in dictionary])
            n = len(dictionary)
        h = VP()
        buf = C.create_string_buffer(1 << 20)
        self._chk(self.lib.ref_read_long_format(str(path).encode(), d, i32(n), C.byref(h), buf, i64(len(buf))))
        txt = buf.value.decode()
        return RefDataset(self, h), (txt.split("\n") if txt else [])

    def fast_sccs(self, attempts, drugs, lambda_x=3.0, zipf=False, seed=20261017, threads=None):
        """SURVEY §8(d) fast generator on the reference's own Rng (ref_shim.cpp):
        the same arrays as the product generator, without loading it."""
        h = VP()
        self._chk(self.lib.ref_fast_sccs(i64(int(attempts)), i32(int(drugs)), f64(lambda_x), i32(int(bool(zipf))),
                                         u64(int(seed) & 0xFFFFFFFFFFFFFFFF), i32(threads or host_cores()),
                                         C.byref(h)))
        return RefDataset(self, h)

    def penalized_step(self, prior, beta_j, g, h):
        out = f64()
        p = _cprior(prior)
        self._chk(self.lib.ref_penalized_step(C.byref(p), f64(beta_j), f64(g), f64(h), C.byref(out)))
        return out.value

    def log_density(self, prior, beta):
        b = np.ascontiguousarray(beta, dtype=np.float64)
        out = f64()
        p = _cprior(prior)
        self._chk(self.lib.ref_log_density(C.byref(p), _p(b), i32(b.size), C.byref(out)))
        return out.value


class RefDataset:
    def __init__(self, ref, h):
        self.ref, self.h = ref, h

    def __del__(self):
        try:
            self.ref.lib.ref_dataset_destroy(self.h)
        except Exception:
            pass

    def to_host(self):
        from paper_1208_0945_b200.bsccs import Dataset
        return Dataset(*self.arrays())

    def subset(self, idx):
        sel = np.ascontiguousarray(idx, dtype=np.int32)
        h = VP()
        self.ref._chk(self.ref.lib.ref_subset(self.h, _p(sel), i64(sel.size), C.byref(h)))
        return RefDataset(self.ref, h)

    def columns(self, cols):
        """column sample: same subjects and eras, only `cols` (ref_dataset_columns)"""
        c = np.ascontiguousarray(cols, dtype=np.int32)
        h = VP()
        self.ref._chk(self.ref.lib.ref_dataset_columns(self.h, _p(c), i32(c.size), C.byref(h)))
        return RefDataset(self.ref, h)

    def arrays(self):
        """flat CSC arrays (numpy), in Dataset.arrays() order"""
        sz = (i64 * 4)()
        self.ref.lib.ref_dataset_sizes(self.h, sz)
        N, K, J, nnz = list(sz)
        a = [np.zeros(N + 1, np.int32), np.zeros(N, np.int32), np.zeros(K, np.int32), np.zeros(K, np.int32),
             np.zeros(J + 1, np.int64), np.zeros(nnz, np.int32), np.zeros(nnz, np.int32), np.zeros(J, np.int64)]
        self.ref.lib.ref_dataset_flatten(self.h, *[_p(x) for x in a])
        return a

    def bootstrap_replicate(self, seed, r, prior, cfg, init_beta=None):
        """run_bootstrap's replicate r (bootstrap.hpp:103-112): beta and fit summary"""
        J = self._J()
        beta = np.zeros(J)
        b = None if init_beta is None else np.ascontiguousarray(init_beta, dtype=np.float64)
        res = _CRes()
        p, c = _cprior(prior), _ccfg(cfg)
        self.ref._chk(self.ref.lib.ref_bootstrap_replicate(self.h, u64(seed), i32(r), C.byref(p), C.byref(c), _p(b),
                                                           _p(beta), C.byref(res)))
        return dict(beta=beta, log_posterior=res.log_posterior, cycles_run=res.cycles_run,
                    converged=bool(res.converged), final_criterion=res.final_criterion)

    def kfold_split(self, folds, seed):
        n = self.sizes()["N"]
        out = np.zeros(n, np.int32)
        sizes = np.zeros(folds, np.int32)
        self.ref._chk(self.ref.lib.ref_kfold_split(self.h, i32(folds), u64(seed), _p(out), _p(sizes)))
        return np.split(out, np.cumsum(sizes)[:-1])

    def resample(self, seed, stream):
        out = np.zeros(self.sizes()["N"], np.int32)
        self.ref._chk(self.ref.lib.ref_resample(self.h, u64(seed), u64(stream), _p(out)))
        return out

    def predictive_ll(self, beta):
        b = np.ascontiguousarray(beta, dtype=np.float64)
        out = f64()
        self.ref._chk(self.ref.lib.ref_predictive_ll(self.h, _p(b), C.byref(out)))
        return out.value

    def grid_search_cv(self, folds, grid, prior_kind, seed, cfg, warm_start=True, scale=False, threads=1):
        g = np.ascontiguousarray(grid, dtype=np.float64)
        P = g.size
        grid_out, mean = np.zeros(P), np.zeros(P)
        cell_ll = np.zeros(P * folds)
        cell_int = np.zeros(3 * P * folds, np.int32)
        sel, selv, tot = i32(), f64(), i64()
        c = _ccfg(cfg)
        self.ref._chk(self.ref.lib.ref_grid_search_cv(
            self.h, i32(folds), i32(int(prior_kind)), i32(int(scale)), i32(int(warm_start)), u64(seed),
            C.byref(c), _p(g), i32(P), i32(threads), _p(grid_out), _p(cell_ll), _p(cell_int), _p(mean),
            C.byref(sel), C.byref(selv), C.byref(tot)))
        ci = cell_int.reshape(P, folds, 3)
        return dict(variance_grid=grid_out, predictive_ll=cell_ll.reshape(P, folds), cycles=ci[..., 0],
                    converged=ci[..., 1], valid=ci[..., 2], mean_predictive_ll=mean, selected_index=sel.value,
                    selected_variance=selv.value, total_cycles=tot.value)

    def run_bootstrap(self, replicates, level, seed, prior, cfg, warm_start=True, threads=1):
        J = self._J()
        a = [np.zeros(J) for _ in range(4)]
        ints = np.zeros(3, np.int32)
        p, c = _cprior(prior), _ccfg(cfg)
        self.ref._chk(self.ref.lib.ref_run_bootstrap(
            self.h, i32(replicates), f64(level), u64(seed), C.byref(p), C.byref(c), i32(int(warm_start)),
            i32(threads), *[_p(x) for x in a], _p(ints)))
        return dict(beta_full=a[0], lower=a[1], upper=a[2], p_hat=a[3], used=int(ints[0]),
                    non_converged=int(ints[1]), full_converged=bool(ints[2]))

    def fit(self, prior, cfg, init_beta=None, threads=1):
        J = self._J()
        beta = np.zeros(J)
        b = None if init_beta is None else np.ascontiguousarray(init_beta, dtype=np.float64)
        r = _CRes()
        sec = f64()
        p, c = _cprior(prior), _ccfg(cfg)
        self.ref._chk(self.ref.lib.ref_fit(self.h, C.byref(p), C.byref(c), _p(b), i32(threads), _p(beta),
                                           C.byref(r), C.byref(sec)))
        return dict(beta=beta, log_posterior=r.log_posterior, cycles_run=r.cycles_run, converged=bool(r.converged),
                    final_criterion=r.final_criterion, seconds=sec.value)

    def _J(self):
        sz = (i64 * 4)()
        self.ref.lib.ref_dataset_sizes(self.h, sz)
        return int(sz[2])

    def sizes(self):
        sz = (i64 * 4)()
        self.ref.lib.ref_dataset_sizes(self.h, sz)
        return dict(zip(("N", "K", "J", "nnz"), list(sz)))

    def state(self, beta=None, cfg=None):
        return RefState(self, beta, cfg)


class RefState:
    def __init__(self, rds, beta=None, cfg=None):
        self.rds = rds
        lib = rds.ref.lib
        b = None if beta is None else np.ascontiguousarray(beta, dtype=np.float64)
        h = VP()
        c = _ccfg(cfg) if cfg is not None else None
        rds.ref._chk(lib.ref_state_create(rds.h, _p(b), C.byref(c) if c is not None else None, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            self.rds.ref.lib.ref_state_destroy(self.h)
        except Exception:
            pass

    def set_threads(self, threads):
        self.rds.ref.lib.ref_state_set_threads(self.h, i32(threads))

    def grad_hess(self, j, partitions=1):
        g, h = f64(), f64()
        self.rds.ref._chk(self.rds.ref.lib.ref_grad_hess(self.rds.h, self.h, i32(j), i32(partitions), C.byref(g),
                                                         C.byref(h)))
        return g.value, h.value

    def sparse_update(self, j, delta):
        self.rds.ref._chk(self.rds.ref.lib.ref_sparse_update(self.rds.h, self.h, i32(j), f64(delta)))

    def dense_recompute(self, beta=None):
        b = None if beta is None else np.ascontiguousarray(beta, dtype=np.float64)
        self.rds.ref._chk(self.rds.ref.lib.ref_dense_recompute(self.rds.h, self.h, _p(b)))

    def log_likelihood(self):
        out = f64()
        self.rds.ref._chk(self.rds.ref.lib.ref_log_likelihood(self.rds.h, self.h, C.byref(out)))
        return out.value

    def get(self):
        s = self.rds.sizes()
        a = [np.zeros(s["J"]), np.zeros(s["K"]), np.zeros(s["K"]), np.zeros(s["N"])]
        self.rds.ref.lib.ref_state_get(self.h, *[_p(x) for x in a])
        return dict(zip(("beta", "xbeta", "l_exp_xbeta", "denominators"), a))

    def run_cycle(self, prior, cfg):
        crit = f64()
        s = self.rds.sizes()
        trust = np.zeros(s["J"])
        p, c = _cprior(prior), _ccfg(cfg)
        self.rds.ref._chk(self.rds.ref.lib.ref_run_cycle(self.rds.h, self.h, C.byref(p), C.byref(c), C.byref(crit),
                                                         _p(trust)))
        return crit.value, trust


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def timed(fn, *a, **k):
    t0 = time.perf_counter()
    out = fn(*a, **k)
    return out, time.perf_counter() - t0
