"""ctypes binding of include/bsccs_b200.h (libbsccs_b200.so, built in-tree).

There is no fallback: if the library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

LIB_PATH = Path(os.environ.get("BSCCS_B200_LIB", Path(__file__).resolve().parent / "_lib" / "libbsccs_b200.so"))

i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double
P = C.POINTER


class bsccs_prior(C.Structure):
    _fields_ = [("kind", i32), ("variance_is_laplace_scale", i32), ("variance", f64)]


class bsccs_solver_config(C.Structure):
    _fields_ = [
        ("epsilon", f64), ("max_cycles", i32), ("convergence", i32), ("trust_init", f64),
        ("precision", i32), ("path", i32), ("partitions", i32), ("dense_refresh_interval", i32),
        ("random_cycle", i32), ("reserved0", i32), ("cycle_seed", u64), ("min_parallel_nnz", u64),
    ]


class bsccs_fit_result(C.Structure):
    _fields_ = [
        ("log_posterior", f64), ("final_criterion", f64), ("cycles_run", i32), ("converged", i32),
        ("coordinates_visited", i64), ("coordinates_moved", i64), ("dense_refreshes", i64),
        ("device_seconds", f64), ("sweep_seconds", f64), ("algorithmic_bytes", f64), ("kernel_launches", i64),
    ]


class bsccs_cv_config(C.Structure):
    _fields_ = [("folds", i32), ("prior_kind", i32), ("variance_is_laplace_scale", i32), ("warm_start", i32),
                ("seed", u64), ("solver", bsccs_solver_config), ("engine", i32), ("batch", i32)]


class bsccs_cv_cell(C.Structure):
    _fields_ = [("predictive_ll", f64), ("cycles", i32), ("converged", i32), ("valid", i32), ("reserved", i32)]


class bsccs_cv_result(C.Structure):
    _fields_ = [("selected_index", i32), ("points", i32), ("selected_variance", f64), ("total_cycles", i64),
                ("device_seconds", f64), ("fits", i64), ("coordinates_visited", i64)]


class bsccs_bootstrap_config(C.Structure):
    _fields_ = [("replicates", i32), ("warm_start", i32), ("level", f64), ("seed", u64), ("prior", bsccs_prior),
                ("solver", bsccs_solver_config), ("engine", i32), ("batch", i32)]


class bsccs_bootstrap_result(C.Structure):
    _fields_ = [("replicates", i32), ("used", i32), ("non_converged", i32), ("full_converged", i32),
                ("device_seconds", f64), ("total_cycles", i64), ("coordinates_visited", i64)]


# (name, restype, argtypes); restype int = bsccs_status
_SIGS = [
    ("bsccs_abi_version", i32, []),
    ("bsccs_last_error", C.c_char_p, []),
    ("bsccs_device_info", C.c_int, [i32, P(i32), P(i32)]),
    ("bsccs_launch_count", i64, []),
    ("bsccs_debug_set_sweep_flags", None, [i32]),
    ("bsccs_debug_set_sweep", None, [i32, C.c_double]),
    ("bsccs_debug_last_sweep", i32, []),
    ("bsccs_debug_last_rcd_shape", i32, []),
    ("bsccs_debug_trace", i32, [i32, i32, C.c_void_p, i64]),
    ("bsccs_debug_exchange_sum", i32, [i32, C.c_void_p, i32, C.POINTER(C.c_double), C.POINTER(C.c_int32)]),
    ("bsccs_dataset_create", C.c_int, [i32, i32, i32, i64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, i32, i32,
                                        P(C.c_void_p)]),
    ("bsccs_dataset_create_shard", C.c_int, [i32, i32, i32, i64, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_void_p, i32, i32, P(C.c_void_p)]),
    ("bsccs_dataset_destroy", C.c_int, [C.c_void_p]),
    ("bsccs_dataset_info", C.c_int, [C.c_void_p, P(i64)]),
    ("bsccs_dataset_subset", C.c_int, [C.c_void_p, C.c_void_p, i64, i32, P(C.c_void_p)]),
    ("bsccs_dataset_read_long_format", C.c_int, [C.c_char_p, C.c_void_p, i32, i32, i32, i32, P(C.c_void_p)]),
    ("bsccs_dataset_set_drug_ids", C.c_int, [C.c_void_p, C.c_void_p, i32]),
    ("bsccs_dataset_drug_ids", C.c_int, [C.c_void_p, C.c_char_p, i64, P(i64)]),
    ("bsccs_dataset_export", C.c_int, [C.c_void_p] + [C.c_void_p] * 8),
    ("bsccs_kfold_split", C.c_int, [i32, i32, u64, C.c_void_p, C.c_void_p]),
    ("bsccs_resample", C.c_int, [i32, u64, u64, C.c_void_p]),
    ("bsccs_state_create", C.c_int, [C.c_void_p, C.c_void_p, P(C.c_void_p)]),
    ("bsccs_state_clone", C.c_int, [C.c_void_p, P(C.c_void_p)]),
    ("bsccs_state_destroy", C.c_int, [C.c_void_p]),
    ("bsccs_dense_recompute", C.c_int, [C.c_void_p, C.c_void_p]),
    ("bsccs_grad_hess", C.c_int, [C.c_void_p, i32, P(f64), P(f64)]),
    ("bsccs_sparse_update", C.c_int, [C.c_void_p, i32, f64]),
    ("bsccs_log_likelihood", C.c_int, [C.c_void_p, P(f64)]),
    ("bsccs_state_get", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("bsccs_penalized_step", C.c_int, [P(bsccs_prior), f64, f64, f64, P(f64)]),
    ("bsccs_log_density", C.c_int, [P(bsccs_prior), C.c_void_p, i32, P(f64)]),
    ("bsccs_run_cycle", C.c_int, [C.c_void_p, P(bsccs_prior), P(bsccs_solver_config), C.c_void_p,
                                   C.c_void_p, P(f64)]),
    ("bsccs_fit", C.c_int, [C.c_void_p, P(bsccs_prior), P(bsccs_solver_config), C.c_void_p, C.c_void_p,
                             P(bsccs_fit_result)]),
    ("bsccs_solver_config_default", None, [P(bsccs_solver_config)]),
    ("bsccs_fit_batch", C.c_int, [C.c_void_p, i32, P(bsccs_prior), C.c_void_p, C.c_void_p, P(bsccs_solver_config),
                                   C.c_void_p, P(bsccs_fit_result), C.c_void_p]),
    ("bsccs_cv_config_default", None, [P(bsccs_cv_config)]),
    ("bsccs_default_variance_grid", None, [C.c_void_p]),
    ("bsccs_grid_search_cv", C.c_int, [C.c_void_p, P(bsccs_cv_config), C.c_void_p, i32, C.c_void_p,
                                        C.c_void_p, C.c_void_p, P(bsccs_cv_result)]),
    ("bsccs_cv_run_folds", C.c_int, [C.c_void_p, P(bsccs_cv_config), C.c_void_p, i32, i32, i32, C.c_void_p,
                                      P(bsccs_cv_result)]),
    ("bsccs_cv_select", C.c_int, [C.c_void_p, i32, i32, C.c_void_p, C.c_void_p, P(bsccs_cv_result)]),
    ("bsccs_bootstrap_config_default", None, [P(bsccs_bootstrap_config)]),
    ("bsccs_run_bootstrap", C.c_int, [C.c_void_p, P(bsccs_bootstrap_config), C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p, P(bsccs_bootstrap_result)]),
    ("bsccs_bootstrap_replicates", C.c_int, [C.c_void_p, P(bsccs_bootstrap_config), C.c_void_p, i32, i32,
                                              C.c_void_p, C.c_void_p, P(bsccs_bootstrap_result)]),
    ("bsccs_bootstrap_summarize", C.c_int, [i32, i32, f64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                             C.c_void_p, P(bsccs_bootstrap_result)]),
    ("bsccs_group_slot_bytes", i64, [i32]),
    ("bsccs_group_create_local", C.c_int, [P(C.c_void_p), i32, P(C.c_void_p)]),
    ("bsccs_group_create_virtual", C.c_int, [P(C.c_void_p), i32, P(C.c_void_p)]),
    ("bsccs_group_create_rank", C.c_int, [C.c_void_p, i32, i32, C.c_void_p, P(C.c_void_p)]),
    ("bsccs_group_ipc_handle", C.c_int, [C.c_void_p, C.c_void_p]),
    ("bsccs_group_open_peers", C.c_int, [C.c_void_p, C.c_void_p]),
    ("bsccs_group_destroy", C.c_int, [C.c_void_p]),
    ("bsccs_group_fit", C.c_int, [C.c_void_p, P(bsccs_prior), P(bsccs_solver_config), C.c_void_p,
                                   C.c_void_p, P(bsccs_fit_result)]),
    ("bsccs_synth_simulate", C.c_int, [i32, i32, i32, i32, i32, i32, C.c_void_p, C.c_void_p, f64, f64, u64,
                                        P(C.c_void_p)]),
    ("bsccs_synth_fast", C.c_int, [i64, i32, f64, i32, u64, i32, P(C.c_void_p)]),
    ("bsccs_host_dataset_sizes", C.c_int, [C.c_void_p, P(i64)]),
    ("bsccs_host_dataset_arrays", C.c_int, [C.c_void_p] + [P(C.c_void_p)] * 8),
    ("bsccs_host_dataset_destroy", C.c_int, [C.c_void_p]),
]

EXPORTED = [name for name, _, _ in _SIGS]

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1208_0945_b200.build` "
                "(there is no CPU fallback)")
        dll = C.CDLL(str(LIB_PATH))
        for name, res, args in _SIGS:
            fn = getattr(dll, name)
            fn.restype = res
            fn.argtypes = args
        _lib = dll
    return _lib
