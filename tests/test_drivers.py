"""The many-fit callers of fit(): device subset_dataset, kfold_split,
resample, grid_search_cv and run_bootstrap, against the reference built from
its untouched headers (oracle/_ref) and the committed golden fixtures
(tests/golden/drivers_oracle_case.json, tests/golden/make_golden.py).

Parity bar (north star): beta / interval ends within 1e-6 relative (1e-9
absolute near zero), log-likelihoods within 1e-8 relative, identical cycle
counts, identical selections and p_hat."""
import ctypes as C

import numpy as np
import pytest

from conftest import load_golden
from helpers import ds_from_json
from paper_1208_0945_b200 import bootstrap as BT
from paper_1208_0945_b200 import bsccs as B
from paper_1208_0945_b200 import cross_validation as CV
from paper_1208_0945_b200 import datagen
from paper_1208_0945_b200._native import bsccs_bootstrap_result, bsccs_cv_cell, bsccs_cv_result, lib

BETA_REL, ZERO_ABS, LL_REL = 1e-6, 1e-9, 1e-8


@pytest.fixture(scope="module")
def oracle_ds():
    return datagen.simulate(datagen.oracle_case_config())


@pytest.fixture(scope="module")
def golden():
    return load_golden("drivers_oracle_case.json")


def close(a, b, rel=BETA_REL, zabs=ZERO_ABS):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.all(np.abs(a - b) <= np.maximum(rel * np.maximum(np.abs(a), np.abs(b)), zabs))


# ------------------------------------------------------------------ host only


def test_kfold_split_matches_reference(oracle_ds, ref):
    rds = ref.dataset(oracle_ds)
    for folds, seed in [(2, 0), (8, 17), (10, 12080945)]:
        ours = B.kfold_split(oracle_ds, folds, seed)
        theirs = rds.kfold_split(folds, seed)
        assert len(ours) == len(theirs) == folds
        for a, b in zip(ours, theirs):
            assert np.array_equal(a, b)


def test_kfold_split_errors(oracle_ds):
    with pytest.raises(B.InputError):
        B.kfold_split(oracle_ds, 1, 0)
    tiny = B.Dataset([0, 1], [1], [3], [1], [0, 0], [], [])
    with pytest.raises(B.InputError):
        B.kfold_split(tiny, 2, 0)


def test_resample_matches_reference(oracle_ds, ref):
    rds = ref.dataset(oracle_ds)
    for seed, stream in [(77, 1), (77, 2), (0, 0), (2**63 + 5, 9)]:
        assert np.array_equal(B.resample(oracle_ds, seed, stream), rds.resample(seed, stream))


def test_resample_golden(oracle_ds, golden):
    r = B.resample(oracle_ds, golden["bootstrap"]["seed"], 1)
    assert r[:32].tolist() == golden["resample_77_1_head"]


def _summ(est, conv, level):
    J = est.shape[1]
    lo, up, ph = np.zeros(J), np.zeros(J), np.zeros(J)
    res = bsccs_bootstrap_result()
    B._check(lib().bsccs_bootstrap_summarize(J, est.shape[0], level, B._ptr(np.ascontiguousarray(est)),
                                             B._ptr(np.ascontiguousarray(conv, dtype=np.int32)), B._ptr(lo),
                                             B._ptr(up), B._ptr(ph), C.byref(res)))
    return lo, up, ph, res


def _percentile(sorted_vals, q):
    """bootstrap.hpp:55-68 restated"""
    m = len(sorted_vals)
    if m == 1:
        return sorted_vals[0]
    pos = q * (m - 1)
    lo = int(pos)
    if lo + 1 >= m:
        return sorted_vals[m - 1]
    frac = pos - lo
    return sorted_vals[lo] + frac * (sorted_vals[lo + 1] - sorted_vals[lo])


def test_bootstrap_summary_restated():
    rng = np.random.default_rng(3)
    est = rng.normal(size=(37, 5))
    est[rng.random(est.shape) < 0.3] = 0.0
    conv = (rng.random(37) < 0.8).astype(np.int32)
    lo, up, ph, res = _summ(est, conv, 0.9)
    assert res.used == conv.sum() and res.non_converged == 37 - conv.sum()
    for j in range(5):
        col = sorted(est[conv == 1, j])
        assert lo[j] == _percentile(col, (1 - 0.9) / 2)
        assert up[j] == _percentile(col, 1 - (1 - 0.9) / 2)
        assert ph[j] == np.count_nonzero(col) / len(col)
    # one used replicate: both ends are its value (bootstrap.hpp:57-59)
    lo, up, _, _ = _summ(est[:2], np.array([0, 1], np.int32), 0.95)
    assert np.array_equal(lo, est[1]) and np.array_equal(up, est[1])
    with pytest.raises(B.ConvergenceError):
        _summ(est[:2], np.array([0, 0], np.int32), 0.95)


def _select(grid, cells_ll, valid):
    P, F = cells_ll.shape
    cells = (bsccs_cv_cell * (P * F))()
    for g in range(P):
        for f in range(F):
            cells[g * F + f].predictive_ll = cells_ll[g, f]
            cells[g * F + f].valid = int(valid[g, f])
            cells[g * F + f].cycles = 3
    mean = np.zeros(P)
    res = bsccs_cv_result()
    B._check(lib().bsccs_cv_select(B._ptr(np.asarray(grid, float)), P, F, cells, B._ptr(mean), C.byref(res)))
    return res, mean


def test_cv_selection_rules():
    grid = [0.01, 0.1, 1.0]
    ll = np.array([[-5.0, -5.0], [-4.0, -4.0], [-4.0, -4.0]])
    res, mean = _select(grid, ll, np.ones_like(ll))
    assert res.selected_index == 1 and res.selected_variance == 0.1  # ties go to the smaller variance
    assert res.total_cycles == 3 * 6
    valid = np.ones_like(ll)
    valid[1, 0] = 0
    res, mean = _select(grid, ll, valid)
    assert res.selected_index == 2 and np.isnan(mean[1])
    with pytest.raises(B.ConvergenceError):
        _select(grid, ll, np.zeros_like(ll))


def test_default_grid_matches_reference_formula():
    g = CV.default_variance_grid()
    lo, hi = np.log(0.001), np.log(10.0)
    assert g == [float(np.exp(lo + (hi - lo) * i / 12.0)) for i in range(13)]


# ------------------------------------------------------------------ device


@pytest.mark.gpu
def test_device_subset_bit_exact(oracle_ds, ref):
    rds = ref.dataset(oracle_ds)
    dds = oracle_ds.on_device()
    sels = [B.resample(oracle_ds, 77, 1), B.kfold_split(oracle_ds, 8, 17)[3],
            np.array([5, 5, 5, 0, oracle_ds.num_subjects - 1], np.int32), np.arange(oracle_ds.num_subjects)]
    for sel in sels:
        mine = dds.subset(sel).to_host()
        theirs = rds.subset(sel).to_host()
        for a, b in zip(mine.arrays(), theirs.arrays()):
            assert np.array_equal(a, b)


@pytest.mark.gpu
def test_device_subset_errors(oracle_ds):
    dds = oracle_ds.on_device()
    with pytest.raises(B.InputError):
        dds.subset(np.array([], np.int32))
    with pytest.raises(B.InputError):
        dds.subset(np.array([0, oracle_ds.num_subjects], np.int32))
    with pytest.raises(B.InputError):
        dds.subset(np.array([-1], np.int32))


@pytest.mark.gpu
def test_subset_fit_matches_reference(oracle_ds, ref):
    """a fit on a device-built bootstrap dataset vs the reference fit on its own subset"""
    sel = B.resample(oracle_ds, 77, 3)
    sub = oracle_ds.on_device().subset(sel)
    r = B.fit(sub, B.normal_prior(0.1))
    t = ref.dataset(oracle_ds).subset(sel).fit(B.normal_prior(0.1), B.SolverConfig())
    assert r.cycles_run == t["cycles_run"]
    assert close(r.beta_map, t["beta"])
    assert abs(r.log_posterior - t["log_posterior"]) <= LL_REL * abs(t["log_posterior"])


def _cv_cfg(g, engine):
    c = g["cv"]
    return CV.CVConfig(folds=c["folds"], variance_grid=c["grid"], prior_kind=B.PriorKind[c["prior"]], seed=c["seed"],
                       warm_start=c["warm_start"], engine=engine)


def _check_cv(res, exp):
    assert np.array_equal(res.variance_grid, exp["variance_grid"])
    assert res.selected_index == exp["selected_index"]
    assert res.selected_variance == exp["selected_variance"]
    assert res.total_cycles == exp["total_cycles"]
    P, F = len(res.cells), len(res.cells[0])
    for g in range(P):
        for f in range(F):
            cell = res.cells[g][f]
            assert cell.valid == bool(exp["valid"][g][f])
            assert cell.cycles == exp["cycles"][g][f], (g, f)
            e = float(exp["predictive_ll"][g][f])
            assert abs(cell.predictive_ll - e) <= LL_REL * abs(e), (g, f, cell.predictive_ll, e)
    for a, b in zip(res.mean_predictive_ll, exp["mean_predictive_ll"]):
        assert abs(a - float(b)) <= LL_REL * abs(float(b))


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["subset", "batched"])
def test_grid_search_cv_matches_reference(oracle_ds, golden, engine):
    res = CV.grid_search_cv(oracle_ds, _cv_cfg(golden, engine))
    _check_cv(res, golden["cv"]["expected"])


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["subset", "batched"])
def test_grid_search_cv_live_reference_cold(oracle_ds, ref, engine):
    """cold starts, normal prior, 3 folds -- against the live reference"""
    cfg = CV.CVConfig(folds=3, variance_grid=[0.5, 0.02, 0.1], prior_kind=B.PriorKind.normal, seed=5,
                      warm_start=False, engine=engine)
    res = CV.grid_search_cv(oracle_ds, cfg)
    exp = ref.dataset(oracle_ds).grid_search_cv(3, [0.5, 0.02, 0.1], B.PriorKind.normal, 5, B.SolverConfig(),
                                                warm_start=False)
    exp = {k: (v.tolist() if hasattr(v, "tolist") else v) for k, v in exp.items()}
    _check_cv(res, exp)


def _boot_cfg(g, engine):
    b = g["bootstrap"]
    return BT.BootstrapConfig(replicates=b["replicates"], level=b["level"], seed=b["seed"],
                              prior=B.PriorSpec(B.PriorKind[b["prior"]], b["variance"]), warm_start=b["warm_start"],
                              engine=engine)


def _check_boot(res, exp):
    assert res.used == exp["used"] and res.non_converged == exp["non_converged"]
    assert res.full_converged == exp["full_converged"]
    assert close(res.beta_full, [float(x) for x in exp["beta_full"]])
    assert close(res.lower, [float(x) for x in exp["lower"]])
    assert close(res.upper, [float(x) for x in exp["upper"]])
    assert np.array_equal(res.p_hat, [float(x) for x in exp["p_hat"]])


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["subset", "batched"])
def test_run_bootstrap_matches_reference(oracle_ds, golden, engine):
    res = BT.run_bootstrap(oracle_ds, _boot_cfg(golden, engine))
    _check_boot(res, golden["bootstrap"]["expected"])


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["subset", "batched"])
def test_run_bootstrap_laplace_live_reference(oracle_ds, ref, engine):
    """laplace prior (zeros and p_hat < 1), cold starts, 6 replicates"""
    prior = B.laplace_prior(0.05)
    cfg = BT.BootstrapConfig(replicates=6, level=0.8, seed=123, prior=prior, warm_start=False, engine=engine)
    res = BT.run_bootstrap(oracle_ds, cfg)
    exp = ref.dataset(oracle_ds).run_bootstrap(6, 0.8, 123, prior, B.SolverConfig(), warm_start=False)
    _check_boot(res, exp)
    assert res.p_hat.min() < 1.0


@pytest.mark.gpu
def test_driver_input_errors(oracle_ds):
    with pytest.raises(B.InputError):
        CV.grid_search_cv(oracle_ds, CV.CVConfig(variance_grid=[]))
    with pytest.raises(B.InputError):
        CV.grid_search_cv(oracle_ds, CV.CVConfig(variance_grid=[0.1, 0.1]))
    with pytest.raises(B.InputError):
        CV.grid_search_cv(oracle_ds, CV.CVConfig(variance_grid=[-1.0]))
    with pytest.raises(B.InputError):
        BT.run_bootstrap(oracle_ds, BT.BootstrapConfig(replicates=0))
    with pytest.raises(B.InputError):
        BT.run_bootstrap(oracle_ds, BT.BootstrapConfig(level=1.0))


@pytest.mark.gpu
def test_fit_batch_matches_reference_fits(oracle_ds, ref):
    """one batched launch, five fits of different selections / priors /
    starts, each against the reference fit on the materialised selection"""
    rds = ref.dataset(oracle_ds)
    N = oracle_ds.num_subjects
    res_idx = B.resample(oracle_ds, 77, 4)
    held = np.sort(B.kfold_split(oracle_ds, 5, 9)[2])
    rest = np.setdiff1d(np.arange(N), held).astype(np.int32)
    w = np.ones((5, N), np.int32)
    w[1] = np.bincount(res_idx, minlength=N)
    w[2] = 0
    w[2][rest] = 1
    w[4] = np.bincount(res_idx, minlength=N)
    priors = [B.normal_prior(0.1), B.normal_prior(0.1), B.laplace_prior(0.1), B.laplace_prior(1.0),
              B.laplace_prior(0.05)]
    start = rds.fit(B.normal_prior(0.1), B.SolverConfig())["beta"]
    init = np.zeros((5, oracle_ds.num_drugs))
    init[4] = start
    fits, status = B.fit_batch(oracle_ds, priors, w, init)
    sel = [None, res_idx, rest, None, res_idx]
    for r in range(5):
        assert status[r] is None
        src = rds if sel[r] is None else rds.subset(sel[r])
        t = src.fit(priors[r], B.SolverConfig(), init_beta=init[r] if r == 4 else None)
        assert fits[r].cycles_run == t["cycles_run"], r
        assert fits[r].converged == t["converged"]
        assert close(fits[r].beta_map, t["beta"]), r
        assert abs(fits[r].log_posterior - t["log_posterior"]) <= LL_REL * abs(t["log_posterior"]), r


@pytest.mark.gpu
def test_fit_batch_sixteen_and_errors(oracle_ds, ref):
    """a full 16-fit block; a diverging fit (no prior, x'beta past 700) fails
    alone with the reference's error class while the others finish"""
    rds = ref.dataset(oracle_ds)
    N = oracle_ds.num_subjects
    w = np.stack([np.bincount(B.resample(oracle_ds, 5, r + 1), minlength=N) for r in range(16)]).astype(np.int32)
    priors = [B.normal_prior(0.1)] * 16
    fits, status = B.fit_batch(oracle_ds, priors, w)
    for r in (0, 7, 15):
        t = rds.subset(B.resample(oracle_ds, 5, r + 1)).fit(priors[r], B.SolverConfig())
        assert fits[r].cycles_run == t["cycles_run"]
        assert close(fits[r].beta_map, t["beta"])
    # a start with |x'beta| > 700 fails alone (init_state's overflow guard,
    # engine.hpp:56-74 -> numeric_error) while its batch mates finish
    init = np.zeros((3, oracle_ds.num_drugs))
    init[1, :] = 701.0
    fits, status = B.fit_batch(oracle_ds, [B.normal_prior(0.1)] * 3, None, init)
    with pytest.raises(Exception) as ei:
        rds.fit(B.normal_prior(0.1), B.SolverConfig(), init_beta=init[1])
    assert getattr(ei.value, "code", None) == 2  # BSCCS_NUMERIC_ERROR <- bsccs::numeric_error
    assert status[1] is B.NumericError
    assert status[0] is None and status[2] is None
    t = rds.fit(B.normal_prior(0.1), B.SolverConfig())
    for r in (0, 2):
        assert fits[r].cycles_run == t["cycles_run"] and close(fits[r].beta_map, t["beta"])


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["subset", "batched"])
def test_cv_shuffled_order_normalized_criterion(oracle_ds, ref, engine):
    """random_cycle (a fresh Fisher-Yates order every cycle, solver.hpp:109-114)
    and the normalized criterion through both engines, against the reference"""
    solver = B.SolverConfig(random_cycle=True, cycle_seed=31, convergence=B.ConvergenceMode.normalized,
                            epsilon=1e-6)
    cfg = CV.CVConfig(folds=3, variance_grid=[0.05, 0.5], prior_kind=B.PriorKind.laplace, seed=2, solver=solver,
                      engine=engine)
    res = CV.grid_search_cv(oracle_ds, cfg)
    exp = ref.dataset(oracle_ds).grid_search_cv(3, [0.05, 0.5], B.PriorKind.laplace, 2, solver)
    exp = {k: (v.tolist() if hasattr(v, "tolist") else v) for k, v in exp.items()}
    _check_cv(res, exp)


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["subset", "batched"])
def test_bootstrap_dense_route(oracle_ds, ref, engine):
    """UpdatePath::dense replicates (the batched request takes the
    materialised route) against the reference"""
    solver = B.SolverConfig(path=B.UpdatePath.dense)
    prior = B.normal_prior(0.1)
    res = BT.run_bootstrap(oracle_ds, BT.BootstrapConfig(replicates=3, seed=4, prior=prior, solver=solver,
                                                         engine=engine))
    exp = ref.dataset(oracle_ds).run_bootstrap(3, 0.95, 4, prior, solver)
    _check_boot(res, exp)
    with pytest.raises(B.InputError):
        B.fit_batch(oracle_ds, [prior], None, None, solver)


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["subset", "batched"])
def test_bootstrap_cycle_cap_and_refresh(oracle_ds, ref, engine):
    """a cycle cap that stops some replicates short (counted as non-converged,
    excluded from the summaries, bootstrap.hpp:118-127) and a dense refresh
    every 2 cycles (solver.hpp:187-189), cold starts"""
    solver = B.SolverConfig(max_cycles=7, dense_refresh_interval=2, epsilon=3e-4)  # 2 of 9 converge
    prior = B.laplace_prior(0.2)
    cfg = BT.BootstrapConfig(replicates=9, seed=11, prior=prior, solver=solver, warm_start=False, engine=engine)
    exp = ref.dataset(oracle_ds).run_bootstrap(9, 0.95, 11, prior, solver, warm_start=False)
    if exp["used"] == 0:
        with pytest.raises(B.ConvergenceError):
            BT.run_bootstrap(oracle_ds, cfg)
        return
    res = BT.run_bootstrap(oracle_ds, cfg)
    _check_boot(res, exp)
    assert res.non_converged == exp["non_converged"]
