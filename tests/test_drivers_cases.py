"""The reference's own unit tests of its many-fit callers, restated for the
device drivers (both engines): test_cv.cpp:58-200 and
test_bootstrap.cpp:39-215.  Scenarios and configurations are the
reference's; where the reference asserts exact equality the device is held
to the north-star parity bar (1e-6 on coefficients, 1e-8 on likelihoods)
against the reference run on the same inputs, and to bitwise equality with
itself (determinism)."""
import numpy as np
import pytest

from paper_1208_0945_b200 import bootstrap as BT
from paper_1208_0945_b200 import bsccs as B
from paper_1208_0945_b200 import cross_validation as CV
from paper_1208_0945_b200 import datagen

ENGINES = ["subset", "batched"]


def cv_scenario():
    """test_cv.cpp:36-46"""
    return datagen.simulate(datagen.SimConfig(subjects=150, drugs=4, prevalence=[0.3] * 4,
                                              true_beta=[1.0, 0.0, -0.8, 0.5], baseline_log_rate_mean=-4.0,
                                              seed=91))


def scenario_config(engine, **kw):
    """test_cv.cpp:48-56"""
    c = CV.CVConfig(folds=5, variance_grid=[0.01, 0.05, 0.25, 1.0, 5.0], seed=17,
                    solver=B.SolverConfig(epsilon=1e-8, max_cycles=5000), engine=engine)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def boot_scenario():
    """test_bootstrap.cpp:14-23"""
    return datagen.simulate(datagen.SimConfig(subjects=80, drugs=3, prevalence=[0.35] * 3,
                                              true_beta=[1.2, 0.0, -0.6], baseline_log_rate_mean=-4.0, seed=57))


def base_config(engine, **kw):
    """test_bootstrap.cpp:25-34"""
    c = BT.BootstrapConfig(replicates=12, seed=29, prior=B.laplace_prior(0.5),
                           solver=B.SolverConfig(epsilon=1e-6, max_cycles=2000), engine=engine)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


@pytest.mark.gpu
def test_held_out_likelihood_hand_values():
    """test_cv.cpp:91-96: one subject, the exposed day carries the event"""
    toy = B.build_dataset([B.SubjectRecord("s1", [B.Era(1, 0, []), B.Era(1, 1, [0])])], 1)
    assert CV.predictive_log_likelihood([0.0], toy) == pytest.approx(-np.log(2.0), rel=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ENGINES)
def test_one_point_grid(engine):
    """test_cv.cpp:109-122"""
    r = CV.grid_search_cv(cv_scenario(), scenario_config(engine, variance_grid=[0.3]))
    assert r.selected_index == 0 and r.selected_variance == 0.3
    assert len(r.cells) == 1 and len(r.cells[0]) == 5
    assert all(c.valid and c.converged for c in r.cells[0])


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ENGINES)
def test_warm_starts_fewer_cycles_same_choice(engine, ref):
    """test_cv.cpp:124-139, and both runs against the reference"""
    ds = cv_scenario()
    warm = CV.grid_search_cv(ds, scenario_config(engine))
    cold = CV.grid_search_cv(ds, scenario_config(engine, warm_start=False))
    assert warm.selected_variance == cold.selected_variance
    assert warm.total_cycles < cold.total_cycles
    assert np.all(np.abs(np.array(warm.mean_predictive_ll) - np.array(cold.mean_predictive_ll)) < 1e-6)
    rds = ref.dataset(ds)
    sc = scenario_config(engine)
    for res, w in ((warm, True), (cold, False)):
        exp = rds.grid_search_cv(5, sc.variance_grid, B.PriorKind.laplace, 17, sc.solver, warm_start=w)
        assert res.selected_index == exp["selected_index"]
        assert res.total_cycles == exp["total_cycles"]
        for a, b in zip(res.mean_predictive_ll, exp["mean_predictive_ll"]):
            assert abs(a - b) <= 1e-8 * abs(b)


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ENGINES)
def test_search_is_deterministic(engine):
    """test_cv.cpp:141-156: reruns give identical numbers"""
    ds = cv_scenario()
    a = CV.grid_search_cv(ds, scenario_config(engine))
    b = CV.grid_search_cv(ds, scenario_config(engine))
    assert a.selected_variance == b.selected_variance
    assert a.mean_predictive_ll == b.mean_predictive_ll
    assert a.total_cycles == b.total_cycles


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ENGINES)
def test_grid_validated_before_fitting(engine):
    """test_cv.cpp:158-170"""
    ds = cv_scenario()
    for grid in ([], [0.5, 0.5], [0.5, -1.0]):
        with pytest.raises(B.InputError):
            CV.grid_search_cv(ds, scenario_config(engine, variance_grid=grid))
    with pytest.raises(B.InputError):
        CV.grid_search_cv(ds, scenario_config(engine, folds=1))


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ENGINES)
def test_grid_points_failing_everywhere(engine, ref):
    """test_cv.cpp:172-200: fifty drugs that each diverge on a dedicated
    subject plus three subjects exposed to all of them -- every cell of the
    only grid point fails (overflow in training or in the held-out
    evaluation), so there is nothing to select"""
    drugs = 50
    recs = [B.SubjectRecord(f"solo{j}", [B.Era(1, 1, [j]), B.Era(1, 0, [])]) for j in range(drugs)]
    recs += [B.SubjectRecord(f"combo{m}", [B.Era(1, 1, list(range(drugs))), B.Era(1, 0, [])]) for m in range(3)]
    ds = B.build_dataset(recs, drugs)
    cfg = CV.CVConfig(folds=2, variance_grid=[1.0], prior_kind=B.PriorKind.none,
                      solver=B.SolverConfig(max_cycles=5000), engine=engine)
    import pyoracle
    with pytest.raises(pyoracle.OracleError) as ei:
        ref.dataset(ds).grid_search_cv(2, [1.0], B.PriorKind.none, 0, cfg.solver)
    assert ei.value.code == 4  # convergence_error
    with pytest.raises(B.ConvergenceError):
        CV.grid_search_cv(ds, cfg)


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ENGINES)
def test_bootstrap_pipeline_and_reruns(engine, ref):
    """test_bootstrap.cpp:58-126: the documented pipeline (against the
    reference's), interval sanity, and identical reruns"""
    ds = boot_scenario()
    cfg = base_config(engine)
    a = BT.run_bootstrap(ds, cfg)
    b = BT.run_bootstrap(ds, cfg)
    assert np.array_equal(a.lower, b.lower) and np.array_equal(a.upper, b.upper)
    assert np.array_equal(a.p_hat, b.p_hat) and a.used == b.used
    exp = ref.dataset(ds).run_bootstrap(12, 0.95, 29, cfg.prior, cfg.solver)
    assert a.used == exp["used"] and a.non_converged == exp["non_converged"] and a.replicates == 12
    for x, y in ((a.beta_full, exp["beta_full"]), (a.lower, exp["lower"]), (a.upper, exp["upper"])):
        assert np.all(np.abs(x - y) <= np.maximum(1e-6 * np.abs(y), 1e-9))
    assert np.array_equal(a.p_hat, exp["p_hat"])
    assert np.all(a.lower <= a.upper)


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ENGINES)
def test_single_replicate_collapses(engine):
    """test_bootstrap.cpp:140-150"""
    r = BT.run_bootstrap(boot_scenario(), base_config(engine, replicates=1))
    assert r.used == 1
    assert np.array_equal(r.lower, r.upper)
    assert np.all((r.p_hat == 0.0) | (r.p_hat == 1.0))


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ENGINES)
def test_never_exposed_drug_pins_to_zero(engine):
    """test_bootstrap.cpp:152-165: a column no era references"""
    ds = boot_scenario()
    wide = B.Dataset(ds.subject_offsets, ds.events_per_subject, ds.era_lengths, ds.event_counts,
                     np.append(ds.col_ptr, ds.col_ptr[-1]), ds.rows, ds.subjects, None,
                     ["d000", "d001", "d002", "ghost"])
    r = BT.run_bootstrap(wide, base_config(engine, replicates=6))
    assert r.beta_full[3] == 0.0 and r.lower[3] == 0.0 and r.upper[3] == 0.0 and r.p_hat[3] == 0.0


def test_ranked_report():
    """test_bootstrap.cpp:167-195 (host logic)"""
    ds = B.build_dataset([B.SubjectRecord("s", [B.Era(1, 1, [0, 1, 2, 3]), B.Era(1, 0, [])])], 4,
                         ["w", "x", "y", "z"])
    res = BT.BootstrapResult(np.array([0.5, -0.2, 0.5, 0.9]), True, np.array([0.1, -0.5, 0.2, 0.4]),
                             np.array([0.8, 0.1, 0.9, 1.5]), np.array([0.8, 0.4, 0.9, 1.0]), 10, 10, 0)
    rows = BT.report_ranked_intervals(ds, res, 0.5)
    assert [r.drug_id for r in rows] == ["z", "w", "y"]
    assert (rows[1].beta, rows[1].lower, rows[1].upper, rows[1].p_hat) == (0.5, 0.1, 0.8, 0.8)
    assert len(BT.report_ranked_intervals(ds, res, 0.0)) == 4
    assert BT.report_ranked_intervals(ds, res, 1.0) == []
    assert len(BT.report_ranked_intervals(ds, res, 0.8)) == 2


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ENGINES)
def test_impossible_configs_and_universal_failure(engine):
    """test_bootstrap.cpp:197-215"""
    ds = boot_scenario()
    for kw in (dict(replicates=0), dict(level=1.0), dict(level=0.0)):
        with pytest.raises(B.InputError):
            BT.run_bootstrap(ds, base_config(engine, **kw))
    with pytest.raises(B.ConvergenceError):
        BT.run_bootstrap(ds, base_config(engine, solver=B.SolverConfig(epsilon=1e-12, max_cycles=1)))
