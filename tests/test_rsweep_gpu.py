"""The resident-beta sweep k_rcd (csrc/rsweep.cuh) against the reference and
against the per-era sweep k_ccd, on the paths specific to it:

* pair records whose era carries more than 8 / more than 16 other drugs
  (the padded overflow lists);
* the hand-over to k_ccd when a step leaves the range where products of
  exp(beta) cannot over/underflow (a test hook lowers the bound);
* the state it leaves behind (x'beta rebuilt from beta, the compact
  denominators) as the single-coordinate ops and state_get see it;
* dense refresh every cycle, shuffled order, multi-shard launches.

Parity bar as everywhere (north star): beta 1e-6 relative (1e-9 absolute for
reference zeros), log-posterior 1e-8 relative, identical cycle count.
"""
import numpy as np
import pytest

from helpers import random_dataset
from paper_1208_0945_b200 import _native
from paper_1208_0945_b200 import bsccs as B
from paper_1208_0945_b200 import sharding

pytestmark = pytest.mark.gpu

K_CCD, K_RCD, BOTH = 1, 2, 3


def set_sweep(kind=0, beta_limit=0.0):
    _native.lib().bsccs_debug_set_sweep(kind, beta_limit)


def last_sweep():
    return _native.lib().bsccs_debug_last_sweep()


@pytest.fixture(autouse=True)
def _automatic_sweep():
    set_sweep(0, 0.0)
    yield
    set_sweep(0, 0.0)


def assert_parity(res, o):
    ref = np.asarray(o["beta"], float)
    assert res.cycles_run == o["cycles_run"]
    zero = ref == 0.0
    assert np.all(np.abs(res.beta_map[zero]) <= 1e-9)
    assert np.all(np.abs(res.beta_map[~zero] - ref[~zero]) <= 1e-6 * np.abs(ref[~zero]))
    assert abs(res.log_posterior - o["log_posterior"]) <= 1e-8 * abs(o["log_posterior"])


def wide_dataset(rng, num_drugs, num_subjects, lo, hi):
    """eras carrying lo..hi drugs each (more than 8 / 16 other drugs: the
    records' overflow lists)"""
    recs = []
    for s in range(num_subjects):
        eras = []
        for _ in range(rng.uniform_int(1, 4)):
            m = rng.uniform_int(lo, hi)
            drugs = sorted({rng.uniform_int(0, num_drugs - 1) for _ in range(m)})
            eras.append(B.Era(rng.uniform_int(1, 30), rng.uniform_int(0, 2), drugs))
        recs.append(B.SubjectRecord(f"s{s}", eras))
    return B.build_dataset(recs, num_drugs)


def test_random_problems_match_reference(port):
    rng = B.Rng(907)
    for trial in range(8):
        J = rng.uniform_int(2, 30)
        ds = random_dataset(rng, J, rng.uniform_int(20, 120))
        for prior in (B.normal_prior(1.0), B.laplace_prior(0.5)):
            cfg = B.SolverConfig(epsilon=1e-9, max_cycles=10000)
            res = B.fit(ds, prior, cfg)
            assert last_sweep() == K_RCD
            assert_parity(res, port.fit(ds, prior, cfg))


@pytest.mark.parametrize("lo,hi", [(6, 14), (15, 26)])
def test_wide_eras_overflow_lists(port, lo, hi):
    rng = B.Rng(911 + lo)
    ds = wide_dataset(rng, 40, 150, lo, hi)
    for prior in (B.normal_prior(0.5), B.laplace_prior(0.2)):
        cfg = B.SolverConfig(epsilon=1e-8)
        res = B.fit(ds, prior, cfg)
        assert last_sweep() == K_RCD
        assert_parity(res, port.fit(ds, prior, cfg))


def test_same_fit_as_per_era_sweep():
    """k_rcd and k_ccd on the same problem: both within rounding of each
    other (x'beta rebuilt from beta here, carried incrementally there)"""
    rng = B.Rng(919)
    ds = random_dataset(rng, 12, 400)
    prior = B.laplace_prior(0.3)
    cfg = B.SolverConfig(epsilon=1e-10)
    a = B.fit(ds, prior, cfg)
    assert last_sweep() == K_RCD
    set_sweep(K_CCD)
    b = B.fit(ds, prior, cfg)
    assert last_sweep() == K_CCD
    assert a.cycles_run == b.cycles_run
    nz = b.beta_map != 0.0
    assert np.array_equal(a.beta_map == 0.0, b.beta_map == 0.0)
    assert np.all(np.abs(a.beta_map[nz] - b.beta_map[nz]) <= 1e-9 * np.abs(b.beta_map[nz]))
    assert abs(a.log_posterior - b.log_posterior) <= 1e-11 * abs(b.log_posterior)


def test_handover_when_beta_leaves_product_range(port):
    """a lowered |beta| bound makes steps cross it mid-cycle: the sweep stops
    before that step's update and the cycle finishes on k_ccd (criterion
    against the cycle start rebuilt from beta); later cycles stay on k_ccd
    while beta is out of range"""
    rng = B.Rng(929)
    ds = random_dataset(rng, 8, 200)
    prior = B.normal_prior(2.0)
    cfg = B.SolverConfig(epsilon=1e-9)
    set_sweep(0, 0.05)
    st = B.init_state(ds)
    solver = B.SolverState(ds, cfg)
    B.run_cycle(ds, st, solver, prior, cfg)
    assert last_sweep() == BOTH
    res = B.fit(ds, prior, cfg)
    assert_parity(res, port.fit(ds, prior, cfg))


def test_state_after_cycle_matches_reference(ref):
    """after k_rcd cycles the subject blocks are rebuilt on demand: x'beta
    from beta (the reference carries it incrementally: equal to rounding),
    l*exp and the denominators as the sweep left them"""
    rng = B.Rng(937)
    ds = random_dataset(rng, 10, 150)
    prior, cfg = B.laplace_prior(0.4), B.SolverConfig()
    st = B.init_state(ds)
    solver = B.SolverState(ds, cfg)
    rds = ref.dataset(ds)
    rst = rds.state(None, cfg)
    for _ in range(3):
        crit = B.run_cycle(ds, st, solver, prior, cfg)
        rcrit, _ = rst.run_cycle(prior, cfg)
        assert last_sweep() == K_RCD
        assert crit == pytest.approx(rcrit, rel=1e-10, abs=1e-14)
    got = rst.get()
    assert np.allclose(st.beta, got["beta"], rtol=1e-12, atol=1e-15)
    assert np.allclose(st.xbeta, got["xbeta"], rtol=1e-12, atol=1e-14)
    assert np.allclose(st.l_exp_xbeta, got["l_exp_xbeta"], rtol=1e-12, atol=1e-300)
    assert np.allclose(st.denominators, got["denominators"], rtol=1e-12, atol=1e-300)
    # the single-coordinate ops continue from that state on the subject blocks
    g = B.fused_grad_hess(ds, st, 3)
    rg, rh = rst.grad_hess(3)
    assert g.gradient == pytest.approx(rg, rel=1e-10, abs=1e-12)
    assert g.hessian == pytest.approx(rh, rel=1e-10, abs=1e-12)
    # ... and the next sweep picks the denominators up from them
    B.sparse_delta_update(ds, st, 3, 0.125)
    rst.sparse_update(3, 0.125)
    crit = B.run_cycle(ds, st, solver, prior, cfg)
    rcrit, _ = rst.run_cycle(prior, cfg)
    assert crit == pytest.approx(rcrit, rel=1e-9, abs=1e-14)
    assert np.allclose(st.beta, rst.get()["beta"], rtol=1e-10, atol=1e-14)


def test_dense_refresh_every_cycle_and_shuffled_order(port):
    rng = B.Rng(941)
    ds = random_dataset(rng, 9, 180)
    prior = B.normal_prior(0.8)
    for cfg in (B.SolverConfig(epsilon=1e-9, dense_refresh_interval=1),
                B.SolverConfig(epsilon=1e-9, random_cycle=True, cycle_seed=5)):
        res = B.fit(ds, prior, cfg)
        assert last_sweep() == K_RCD
        assert_parity(res, port.fit(ds, prior, cfg))


@pytest.mark.parametrize("shards", [2, 3])
def test_local_group_on_resident_sweep(shards):
    """several shards in one launch, each with its own records, compact
    denominators and shared-memory beta: the same fit as one shard"""
    rng = B.Rng(947 + shards)
    ds = random_dataset(rng, 10, 300)
    prior, cfg = B.laplace_prior(0.3), B.SolverConfig(epsilon=1e-9)
    single = B.fit(ds, prior, cfg)
    grp = sharding.LocalGroup(sharding.shard_dataset(ds, shards), 0)
    res = grp.fit(prior, cfg)
    assert last_sweep() == K_RCD
    grp.close()
    assert res.cycles_run == single.cycles_run
    nz = single.beta_map != 0.0
    assert np.array_equal(res.beta_map == 0.0, ~nz)
    assert np.all(np.abs(res.beta_map[nz] - single.beta_map[nz]) <= 1e-10 * np.abs(single.beta_map[nz]))


@pytest.mark.parametrize("ctas,drugs,subjects,lam,shape", [
    (4, 400, 3000, 3.0, 1 | 16),  # ~60 pairs per slice: one slot x 384 threads, subject tile
    (4, 60, 3000, 3.0, 2 | 16),   # ~560: two slots x 512 threads
    (4, 35, 3000, 3.0, 3 | 16),   # ~960: three slots x 384 threads
    (2, 1500, 50000, 3.0, 2),     # ~25k subjects per CTA: no subject tile (touched-subject bitmaps + lookup)
])
def test_every_shape_matches_reference(port, ctas, drugs, subjects, lam, shape):
    """each k_rcd shape (forced by the CTA count and the drug count) against
    the C oracle, Laplace and Normal"""
    from paper_1208_0945_b200 import datagen
    ds = datagen.fast_sccs(subjects, drugs, lam)
    dds = B.DeviceDataset(ds, 0, ctas)
    for prior in (B.laplace_prior(0.1), B.normal_prior(0.5)):
        cfg = B.SolverConfig(epsilon=1e-7)
        res = B.fit(dds, prior, cfg)
        assert last_sweep() == K_RCD
        assert _native.lib().bsccs_debug_last_rcd_shape() == shape
        assert_parity(res, port.fit(ds, prior, cfg))
    dds.close()


def test_skewed_and_empty_columns(port):
    """Zipf drug prevalence over 3,000 drugs (a few columns hold most pairs,
    many a handful, many none): the build's column lookup (bucket table over
    the column pointers) and the records of tiny columns, with the per-pair
    subjects uploaded or derived on the device, against the C oracle"""
    g = np.random.default_rng(5)
    J = 3000
    recs = []
    for sidx in range(4000):
        eras = []
        for _ in range(int(g.integers(1, 6))):
            drugs = sorted({int(min(J - 1, g.zipf(1.3) - 1)) for _ in range(int(g.integers(0, 5)))})
            eras.append(B.Era(int(g.integers(1, 60)), int(g.integers(0, 3)), drugs))
        recs.append(B.SubjectRecord(f"s{sidx}", eras))
    ds = B.build_dataset(recs, J)
    nnz_col = np.diff(ds.col_ptr)
    assert (nnz_col == 0).sum() > J // 2 and nnz_col.max() > 1000
    cfg = B.SolverConfig(epsilon=1e-7)
    for upload in (True, False):
        dds = B.DeviceDataset(ds, 0, upload_subjects=upload)
        res = B.fit(dds, B.laplace_prior(0.1), cfg)
        assert_parity(res, port.fit(ds, B.laplace_prior(0.1), cfg))
        dds.close()
