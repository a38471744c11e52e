"""Device engine vs the reference (test_engine.cpp restated, plus the
golden engine cases generated from the reference).  Tolerances: x'beta is
bit-exact (same per-row addition order); exp-derived values within 4 ulp
(CUDA exp vs glibc exp, both <= 1 ulp); reductions within 1e-12 relative
(the reference's own bound for re-partitioned sums, test_engine.cpp:103-125)."""
import numpy as np
import pytest

from conftest import load_golden
from helpers import ds_from_json, fa, random_beta, random_dataset, rel_gap, toy_dataset
from paper_1208_0945_b200 import bsccs as B

pytestmark = pytest.mark.gpu

ULP4 = 4 * np.finfo(np.float64).eps


def close(a, b, rtol):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.all(np.abs(a - b) <= rtol * np.maximum(1.0, np.maximum(np.abs(a), np.abs(b))))


def test_toy_state_at_zero():
    ds = toy_dataset()
    st = B.init_state(ds)
    assert list(st.beta) == [0.0]
    assert list(st.xbeta) == [0.0, 0.0]
    assert list(st.l_exp_xbeta) == [1.0, 1.0]
    assert list(st.denominators) == [2.0]
    assert B.log_likelihood(ds, st) == pytest.approx(-0.6931471805599453, rel=1e-12)


def test_toy_gradient_and_curvature():
    ds = toy_dataset()
    st = B.init_state(ds)
    gh = B.fused_grad_hess(ds, st, 0)
    assert gh.gradient == pytest.approx(0.5, abs=1e-15)
    assert gh.hessian == pytest.approx(-0.25, abs=1e-15)


def test_unit_sparse_step():
    ds = toy_dataset()
    st = B.init_state(ds)
    B.sparse_delta_update(ds, st, 0, 1.0)
    assert list(st.beta) == [1.0]
    assert list(st.xbeta) == [0.0, 1.0]
    assert st.denominators[0] == pytest.approx(1.0 + np.exp(1.0), rel=1e-15)
    assert B.log_likelihood(ds, st) == pytest.approx(1.0 - np.log(1.0 + np.exp(1.0)), rel=1e-12)
    B.dense_recompute(ds, st, [np.log(2.0)])
    assert B.log_likelihood(ds, st) == pytest.approx(np.log(2.0 / 3.0), rel=1e-12)


def test_two_subject_dyadic_exact():
    recs = [B.SubjectRecord("a", [B.Era(1, 0, [0]), B.Era(1, 1, [])]),
            B.SubjectRecord("b", [B.Era(1, 0, [0]), B.Era(1, 2, []), B.Era(1, 0, []), B.Era(1, 0, [])])]
    ds = B.build_dataset(recs, 1)
    gh = B.fused_grad_hess(ds, B.init_state(ds), 0)
    assert ds.y_dot_x[0] == 0
    assert gh.gradient == -1.0
    assert gh.hessian == -0.625


@pytest.mark.parametrize("b", [-40.0, -60.0, -200.0, -600.0])
def test_tiny_weights_keep_full_precision(ref, b):
    """Hessian terms far below the exchange's 2^-80 resolution (w ~ e^b, a
    coordinate driven towards -inf): the scaled refinement rounds of the
    exchange (xchg.cuh needs_refine) reproduce the reference's (g, h) to
    1e-12 relative -- not h == 0, which would take the reference's h == 0
    branches (prior.hpp:95-98,107-109) where the reference does not"""
    rng = B.Rng(5151)
    ds = random_dataset(rng, 3, 60)
    beta = [b, 0.3, -0.2]
    st = B.init_state(ds, beta)
    rs = ref.dataset(ds).state(beta)
    for j in range(3):
        a = B.fused_grad_hess(ds, st, j)
        g, h = rs.grad_hess(j)
        assert h < 0.0 and a.hessian < 0.0
        assert abs(a.hessian - h) <= 1e-12 * abs(h), (j, a.hessian, h)
        assert abs(a.gradient - g) <= 1e-12 * abs(g) if g != 0.0 else a.gradient == 0.0


def test_weights_in_unit_interval_and_no_negative_zero(port):
    rng = B.Rng(31)
    for trial in range(30):
        J = rng.uniform_int(1, 8)
        ds = random_dataset(rng, J, 40)
        beta = random_beta(rng, J, 1.0)
        st = B.init_state(ds, beta)
        ost = port.init_state(ds, beta)
        for j in range(J):
            a = B.fused_grad_hess(ds, st, j)
            assert a.hessian <= 0.0
            if a.hessian == 0.0:
                assert not np.signbit(a.hessian)
            g, h = port.grad_hess(ds, ost, j)
            assert rel_gap(a.gradient, g) < 1e-12
            assert rel_gap(a.hessian, h) < 1e-12


def test_incremental_drift_bounded():
    rng = B.Rng(47)
    ds = random_dataset(rng, 5, 80)
    st = B.init_state(ds)
    for _ in range(1000):
        B.sparse_delta_update(ds, st, rng.uniform_int(0, 4), -0.05 + 0.1 * rng.uniform())
    fresh = st.copy()
    B.dense_recompute(ds, fresh)
    assert np.array_equal(fresh.beta, st.beta)
    assert close(st.xbeta, fresh.xbeta, 1e-9)
    assert close(st.l_exp_xbeta, fresh.l_exp_xbeta, 1e-9)
    assert close(st.denominators, fresh.denominators, 1e-9)


def test_zero_step_noop_and_nonfinite_rejected():
    ds = toy_dataset()
    st = B.init_state(ds)
    before = (st.beta, st.xbeta, st.l_exp_xbeta, st.denominators)
    B.sparse_delta_update(ds, st, 0, 0.0)
    after = (st.beta, st.xbeta, st.l_exp_xbeta, st.denominators)
    assert all(np.array_equal(a, b) for a, b in zip(before, after))
    with pytest.raises(B.NumericError):
        B.sparse_delta_update(ds, st, 0, float("nan"))
    with pytest.raises(B.NumericError):
        B.sparse_delta_update(ds, st, 0, float("inf"))


def test_overflow_guard():
    ds = toy_dataset()
    with pytest.raises(B.NumericError):
        B.init_state(ds, [701.0])
    st = B.init_state(ds, [699.0])
    with pytest.raises(B.NumericError):
        B.sparse_delta_update(ds, st, 0, 5.0)


def test_covering_drug_exactly_uninformative():
    recs = [B.SubjectRecord("a", [B.Era(3, 1, [0]), B.Era(2, 0, [0, 1])]),
            B.SubjectRecord("b", [B.Era(5, 2, [0]), B.Era(1, 1, [0])])]
    ds = B.build_dataset(recs, 2)
    rng = B.Rng(59)
    for _ in range(5):
        st = B.init_state(ds, random_beta(rng, 2, 1.0))
        gh = B.fused_grad_hess(ds, st, 0)
        assert gh.gradient == 0.0 and gh.hessian == 0.0 and not np.signbit(gh.hessian)


def test_log_likelihood_additive_over_subjects():
    rng = B.Rng(61)
    ds = random_dataset(rng, 3, 30)
    twice = B.subset_dataset(ds, list(range(ds.num_subjects)) * 2)
    beta = random_beta(rng, 3, 0.7)
    a = B.log_likelihood(ds, B.init_state(ds, beta))
    b = B.log_likelihood(twice, B.init_state(twice, beta))
    assert rel_gap(2.0 * a, b) < 1e-12


def test_golden_engine_cases():
    for case in load_golden("engine_cases.json"):
        ds = ds_from_json(case["dataset"])
        st = B.init_state(ds, fa(case["beta"]))
        assert np.array_equal(st.xbeta, fa(case["xbeta"]))  # same add order: bit-exact
        assert close(st.l_exp_xbeta, fa(case["l_exp_xbeta"]), ULP4)
        assert close(st.denominators, fa(case["denominators"]), ULP4 * 8)
        for j, (g, h) in enumerate(case["grad_hess"]):
            gh = B.fused_grad_hess(ds, st, j)
            assert rel_gap(gh.gradient, float(g)) < 1e-12
            assert rel_gap(gh.hessian, float(h)) < 1e-12
        assert rel_gap(B.log_likelihood(ds, st), float(case["log_likelihood"])) < 1e-12
        for j, d in case["updates"]:
            B.sparse_delta_update(ds, st, j, float(d))
        assert np.array_equal(st.beta, fa(case["after"]["beta"]))
        assert close(st.xbeta, fa(case["after"]["xbeta"]), 1e-15)
        assert close(st.l_exp_xbeta, fa(case["after"]["l_exp_xbeta"]), 1e-14)
        assert close(st.denominators, fa(case["after"]["denominators"]), 1e-13)
        assert rel_gap(B.log_likelihood(ds, st), float(case["ll_after"])) < 1e-12


def test_slices_cover_many_ctas():
    """A dataset with more subjects than CTAs, forcing every CTA to own a
    slice and runs to cross register-cached tiles."""
    rng = B.Rng(5)
    ds = random_dataset(rng, 3, 3000, exposure_prob=0.8)
    beta = random_beta(rng, 3, 0.8)
    st = B.init_state(ds, beta)
    import pyoracle
    port = pyoracle.Port()
    ost = port.init_state(ds, beta)
    for j in range(3):
        a = B.fused_grad_hess(ds, st, j)
        g, h = port.grad_hess(ds, ost, j)
        assert rel_gap(a.gradient, g) < 1e-12 and rel_gap(a.hessian, h) < 1e-12
    for j, d in [(0, 0.3), (2, -0.2), (1, 0.11)]:
        B.sparse_delta_update(ds, st, j, d)
        port.sparse_update(ds, ost, j, d)
    assert close(st.denominators, ost["denominators"], 1e-13)
    assert close(st.xbeta, ost["xbeta"], 0.0)


@pytest.mark.parametrize("ctas", [1, 2, 3])
def test_streamed_slices_beyond_register_tiles(ctas):
    """Few CTAs, so every column's slice is far larger than the register
    tiles: the chunked streamed path, with runs crossing chunk edges and the
    tile/stream boundary, in the tier-1 ops and in whole sweeps, against the
    oracle (the skewed-column case of SURVEY §8(d))."""
    import pyoracle
    rng = B.Rng(77 + ctas)
    ds = random_dataset(rng, 4, 2500, exposure_prob=0.85)
    beta = random_beta(rng, 4, 0.6)
    dds = B.DeviceDataset(ds, 0, ctas)
    assert max(np.diff(ds.col_ptr)) > 1200 * ctas  # beyond the register tiles of every CTA
    st = B.init_state(dds, beta)
    port = pyoracle.Port()
    ost = port.init_state(ds, beta)
    for j in range(4):
        a = B.fused_grad_hess(dds, st, j)
        g, h = port.grad_hess(ds, ost, j)
        assert rel_gap(a.gradient, g) < 1e-12 and rel_gap(a.hessian, h) < 1e-12
    for j, d in [(0, 0.3), (2, -0.2), (1, 0.11), (3, 0.05)]:
        B.sparse_delta_update(dds, st, j, d)
        port.sparse_update(ds, ost, j, d)
    assert close(st.denominators, ost["denominators"], 1e-12)
    assert close(st.xbeta, ost["xbeta"], 0.0)
    for prior in (B.laplace_prior(0.1), B.normal_prior(1.0)):
        res = B.fit(dds, prior)
        exp = port.fit(ds, prior, B.SolverConfig())
        assert res.cycles_run == exp["cycles_run"]
        assert np.all(np.abs(res.beta_map - exp["beta"]) <= np.maximum(1e-8 * np.abs(exp["beta"]), 1e-11))
        assert rel_gap(res.log_posterior, exp["log_posterior"]) < 1e-10


def test_streamed_sweep_without_subject_tile():
    """One CTA owning ~25k subjects: too many for the shared-memory subject
    tile, so the sweep runs the instantiation with subject records in HBM and
    the streamed path (k_ccd<0,1>), against the oracle."""
    import pyoracle
    from paper_1208_0945_b200 import datagen
    ds = datagen.fast_sccs(26_000, 6, 3.0)
    assert ds.num_subjects > 20_000
    dds = B.DeviceDataset(ds, 0, 1)
    port = pyoracle.Port()
    for prior in (B.laplace_prior(0.1), B.normal_prior(0.5)):
        res = B.fit(dds, prior)
        exp = port.fit(ds, prior, B.SolverConfig())
        assert res.cycles_run == exp["cycles_run"]
        assert np.all(np.abs(res.beta_map - exp["beta"]) <= np.maximum(1e-8 * np.abs(exp["beta"]), 1e-11))
        assert rel_gap(res.log_posterior, exp["log_posterior"]) < 1e-10


def test_speculative_sweep_without_subject_tile():
    """Eight CTAs owning ~12k subjects each (too many for the shared-memory
    subject tile) with slices inside the register tiles: the speculative
    sweep with the touched-subject bitmaps (k_ccd<0,0>), against the oracle."""
    import pyoracle
    from paper_1208_0945_b200 import datagen
    ds = datagen.fast_sccs(100_000, 200, 0.5)
    dds = B.DeviceDataset(ds, 0, 8)
    assert max(np.diff(ds.col_ptr)) < 8 * 900  # slices fit the register tiles
    port = pyoracle.Port()
    for prior in (B.laplace_prior(0.1), B.normal_prior(0.5)):
        res = B.fit(dds, prior)
        exp = port.fit(ds, prior, B.SolverConfig())
        assert res.cycles_run == exp["cycles_run"]
        assert np.all(np.abs(res.beta_map - exp["beta"]) <= np.maximum(1e-8 * np.abs(exp["beta"]), 1e-11))
        assert rel_gap(res.log_posterior, exp["log_posterior"]) < 1e-10


@pytest.mark.parametrize("corrupt,message", [
    ("row_out_of_range", "invalid pair"),
    ("foreign_subject", "invalid pair"),
    ("rows_not_ascending", "invalid pair"),
    ("era_length_zero", "era length must be positive"),
    ("subject_without_eras", "every subject needs at least one era"),
])
def test_device_build_validation(corrupt, message):
    """build_dataset's invariants (dataset.hpp:135-175) checked by the device
    build (k_validate_small, k_pair_meta) on a dataset large enough for many
    build blocks, each corruption planted mid-array."""
    from paper_1208_0945_b200 import datagen
    ds = datagen.fast_sccs(20_000, 30, 3.0)
    a = [x.copy() for x in ds.arrays()]
    off, eps, lens, cnts, cptr, rows, subs, ydx = a
    p = int(cptr[17]) + 5  # inside column 17
    if corrupt == "row_out_of_range":
        rows[p] = lens.size
    elif corrupt == "foreign_subject":
        subs[p] = (subs[p] + 7) % (off.size - 1)
    elif corrupt == "rows_not_ascending":
        rows[p], rows[p + 1] = rows[p + 1], rows[p]
        subs[p], subs[p + 1] = subs[p + 1], subs[p]
    elif corrupt == "era_length_zero":
        lens[lens.size // 2] = 0
    elif corrupt == "subject_without_eras":
        i = (off.size - 1) // 2
        off[i + 1] = off[i]
    bad = B.Dataset(off, eps, lens, cnts, cptr, rows, subs, ydx)
    with pytest.raises(B.InputError, match=message):
        B.DeviceDataset(bad, 0)


@pytest.mark.parametrize("corrupt,message", [
    ("row_out_of_range", "invalid pair"),
    ("rows_not_ascending", "invalid pair"),
    ("subject_without_eras", "every subject needs at least one era"),
])
def test_device_build_validation_derived_subjects(corrupt, message):
    """subjects = NULL (derived on the device from the rows): the same
    invariants are still rejected, nothing is read out of range"""
    from paper_1208_0945_b200 import datagen
    ds = datagen.fast_sccs(20_000, 30, 3.0)
    a = [x.copy() for x in ds.arrays()]
    off, eps, lens, cnts, cptr, rows, subs, ydx = a
    p = int(cptr[17]) + 5
    if corrupt == "row_out_of_range":
        rows[p] = lens.size
    elif corrupt == "rows_not_ascending":
        rows[p], rows[p + 1] = rows[p + 1], rows[p]
    elif corrupt == "subject_without_eras":
        i = (off.size - 1) // 2
        off[i + 1] = off[i]
    bad = B.Dataset(off, eps, lens, cnts, cptr, rows, subs, ydx)
    with pytest.raises(B.InputError, match=message):
        B.DeviceDataset(bad, 0, upload_subjects=False)


def test_derived_subjects_same_fit():
    """a dataset created without its per-pair subjects (derived on the
    device) fits bit for bit like the one created with them"""
    from paper_1208_0945_b200 import datagen
    ds = datagen.fast_sccs(60_000, 80, 3.0)
    prior, cfg = B.laplace_prior(0.2), B.SolverConfig(epsilon=1e-8)
    a = B.DeviceDataset(ds, 0)
    b = B.DeviceDataset(ds, 0, upload_subjects=False)
    assert a.info() == b.info()
    ra, rb = B.fit(a, prior, cfg), B.fit(b, prior, cfg)
    assert ra.cycles_run == rb.cycles_run
    assert np.array_equal(ra.beta_map, rb.beta_map)
    assert ra.log_posterior == rb.log_posterior
    a.close()
    b.close()


def test_three_tile_sweep_with_subject_tile():
    """Mean slices of ~500 pairs per CTA (beyond the one-tile kernel's 352,
    inside the three-tile kernel's 1,056) with the subject tile: the
    t3::k_ccd<1,0> instantiation, against the oracle."""
    import pyoracle
    rng = B.Rng(31)
    ds = random_dataset(rng, 8, 4000, exposure_prob=0.3)
    dds = B.DeviceDataset(ds, 0, 8)
    nnz_col = np.diff(ds.col_ptr)
    assert nnz_col.mean() / 8 > 300 and nnz_col.max() / 8 < 900
    port = pyoracle.Port()
    for prior in (B.laplace_prior(0.1), B.normal_prior(0.5)):
        res = B.fit(dds, prior)
        exp = port.fit(ds, prior, B.SolverConfig())
        assert res.cycles_run == exp["cycles_run"]
        assert np.all(np.abs(res.beta_map - exp["beta"]) <= np.maximum(1e-8 * np.abs(exp["beta"]), 1e-11))
        assert rel_gap(res.log_posterior, exp["log_posterior"]) < 1e-10
