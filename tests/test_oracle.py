"""The parity checker itself: the C restatement (oracle/ccd_oracle.c) is
pinned bit-for-bit against the reference's golden outputs (tests/golden,
generated from the untouched reference headers) and, where the reference
build is present, against the reference directly."""
import numpy as np
import pytest

from conftest import load_golden
from helpers import ds_from_json, fa, prior_from, random_beta, random_dataset, toy_dataset
from paper_1208_0945_b200 import bsccs as B
from paper_1208_0945_b200 import datagen


def test_toy_kats(port):
    # test_engine.cpp:28-64
    ds = toy_dataset()
    st = port.init_state(ds)
    assert list(st["xbeta"]) == [0.0, 0.0]
    assert list(st["l_exp_xbeta"]) == [1.0, 1.0]
    assert list(st["denominators"]) == [2.0]
    assert port.log_likelihood(ds, st) == pytest.approx(-0.6931471805599453, rel=1e-12)
    g, h = port.grad_hess(ds, st, 0)
    assert (g, h) == (0.5, -0.25)
    port.sparse_update(ds, st, 0, 1.0)
    assert st["denominators"][0] == pytest.approx(1.0 + np.e, rel=1e-15)


def test_dyadic_exact(port):
    # test_engine.cpp:66-81
    recs = [B.SubjectRecord("a", [B.Era(1, 0, [0]), B.Era(1, 1, [])]),
            B.SubjectRecord("b", [B.Era(1, 0, [0]), B.Era(1, 2, []), B.Era(1, 0, []), B.Era(1, 0, [])])]
    ds = B.build_dataset(recs, 1)
    st = port.init_state(ds)
    assert port.grad_hess(ds, st, 0) == (-1.0, -0.625)


def test_step_kats(port):
    # test_prior.cpp:88-96
    assert port.penalized_step(B.PriorSpec(), 0.0, 0.5, -0.25) == 2.0
    assert port.penalized_step(B.laplace_prior(2.0), 0.0, 0.5, -0.25) == 0.0
    assert port.penalized_step(B.normal_prior(1.0), 1.0, 0.0, -1.0) == pytest.approx(-0.5, rel=1e-15)


def test_oracle_case_golden(port):
    g = load_golden("oracle_case.json")
    ds = datagen.simulate(datagen.oracle_case_config())
    for fit in g["fits"]:
        r = port.fit(ds, prior_from(fit["prior"]), B.SolverConfig())
        assert r["cycles_run"] == fit["cycles_run"]
        assert r["log_posterior"] == float(fit["log_posterior"])
        assert np.array_equal(r["beta"], fa(fit["beta"]))


def test_engine_cases_golden(port):
    for case in load_golden("engine_cases.json"):
        ds = ds_from_json(case["dataset"])
        st = port.init_state(ds, fa(case["beta"]))
        assert np.array_equal(st["xbeta"], fa(case["xbeta"]))
        assert np.array_equal(st["l_exp_xbeta"], fa(case["l_exp_xbeta"]))
        assert np.array_equal(st["denominators"], fa(case["denominators"]))
        for j, (g, h) in enumerate(case["grad_hess"]):
            assert port.grad_hess(ds, st, j) == (float(g), float(h))
        assert port.log_likelihood(ds, st) == float(case["log_likelihood"])
        for j, d in case["updates"]:
            port.sparse_update(ds, st, j, float(d))
        for k in ("beta", "xbeta", "l_exp_xbeta", "denominators"):
            assert np.array_equal(st[k], fa(case["after"][k])), k


def test_small_suite_golden(port):
    cases = load_golden("small_suite.json")
    assert len(cases) == 100
    for c in cases[:40]:
        s = c["sim"]
        cfg = datagen.SimConfig(subjects=s["subjects"], drugs=s["drugs"], min_eras=1, max_eras=6, min_era_length=5,
                                max_era_length=30, prevalence=[float(s["prevalence"])] * s["drugs"],
                                true_beta=fa(s["true_beta"]).tolist(), baseline_log_rate_mean=-3.0,
                                baseline_log_rate_sd=0.4, seed=s["seed"])
        ds = datagen.simulate(cfg)
        scfg = B.SolverConfig(epsilon=1e-8, max_cycles=10000)
        for fit in c["fits"]:
            r = port.fit(ds, prior_from(fit["prior"]), scfg)
            assert r["cycles_run"] == fit["cycles_run"]
            assert np.array_equal(r["beta"], fa(fit["beta"]))


def test_port_equals_reference_random(port, ref):
    rng = B.Rng(777)
    for trial in range(15):
        J = rng.uniform_int(1, 7)
        ds = random_dataset(rng, J, rng.uniform_int(3, 50))
        rds = ref.dataset(ds)
        for prior in (B.normal_prior(0.5), B.laplace_prior(0.3), B.PriorSpec()):
            cfg = B.SolverConfig(max_cycles=50)
            try:
                a = rds.fit(prior, cfg)
            except Exception as e:  # the port must fail the same way
                with pytest.raises(Exception):
                    port.fit(ds, prior, cfg)
                continue
            b = port.fit(ds, prior, cfg)
            assert a["cycles_run"] == b["cycles_run"]
            assert np.array_equal(a["beta"], b["beta"])
            assert a["log_posterior"] == b["log_posterior"]


def test_random_cycle_port_equals_reference(port, ref):
    rng = B.Rng(127)
    ds = random_dataset(rng, 5, 40)
    cfg = B.SolverConfig(epsilon=1e-8, max_cycles=5000, random_cycle=True, cycle_seed=22)
    a = ref.dataset(ds).fit(B.normal_prior(0.6), cfg)
    b = port.fit(ds, B.normal_prior(0.6), cfg)
    assert a["cycles_run"] == b["cycles_run"] and np.array_equal(a["beta"], b["beta"])
