"""Configs 4 and 5 at their named size (BASELINE.json: the 1M-patient x 1,500
set), against the reference's own drivers run here on 8 cores
(tests/golden/drivers_1M.json, tests/golden/make_golden.py drivers_1M):

  * config 4 in full: grid_search_cv, 8 folds x 8 variances log-uniform on
    [0.001, 10], Laplace, seed 17, warm chains (cross_validation.hpp:100-215);
  * config 5, a 16-replicate prefix of run_bootstrap (Normal 0.1, seed 77,
    warm; replicate r depends only on (seed, r), so the prefix is an exact
    sub-run of the 200-replicate job, bootstrap.hpp:79-158);
  * the reference's replicate fits r = 0..3 themselves (bootstrap.hpp:103-112)
    against the batched weighted engine (k_bccd) and the materialised
    subset route.

Both engines.  Parity bar: beta / interval ends 1e-6 relative (1e-9 absolute
near zero), log-likelihoods 1e-8 relative, identical cycles, selections and
p_hat."""
import hashlib

import numpy as np
import pytest

from conftest import load_golden
from paper_1208_0945_b200 import bootstrap as BT
from paper_1208_0945_b200 import bsccs as B
from paper_1208_0945_b200 import cross_validation as CV
from paper_1208_0945_b200 import datagen

from test_drivers import BETA_REL, LL_REL, ZERO_ABS, _check_boot, _check_cv, close

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def golden():
    return load_golden("drivers_1M.json")


@pytest.fixture(scope="module")
def ds1m(golden):
    ds = datagen.fast_sccs(golden["attempts"], golden["drugs"], golden["lambda_x"])
    h = hashlib.sha256()
    for a in ds.arrays():
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == golden["digest"]
    return ds


@pytest.fixture(scope="module")
def dds1m(ds1m):
    d = B.DeviceDataset(ds1m, 0)
    yield d
    d.close()


def test_golden_shape(golden):
    assert golden["sizes"] == {"N": 962094, "K": 14530220, "J": 1500, "nnz": 43599559}
    assert len(golden["cv"]["grid"]) == 8 and golden["cv"]["folds"] == 8
    assert golden["bootstrap"]["replicates"] == 16 and len(golden["replicates"]) == 4


@pytest.mark.parametrize("engine", ["batched", "subset"])
def test_config4_grid_search_cv_1M(dds1m, golden, engine):
    c = golden["cv"]
    cfg = CV.CVConfig(folds=c["folds"], variance_grid=c["grid"], prior_kind=B.PriorKind[c["prior"]], seed=c["seed"],
                      warm_start=c["warm_start"], engine=engine)
    _check_cv(CV.grid_search_cv(dds1m, cfg), c["expected"])


@pytest.mark.parametrize("engine", ["batched", "subset"])
def test_config5_bootstrap_prefix_1M(dds1m, golden, engine):
    b = golden["bootstrap"]
    cfg = BT.BootstrapConfig(replicates=b["replicates"], level=b["level"], seed=b["seed"],
                             prior=B.PriorSpec(B.PriorKind[b["prior"]], b["variance"]), warm_start=b["warm_start"],
                             engine=engine)
    _check_boot(BT.run_bootstrap(dds1m, cfg), b["expected"])


def _check_rep(beta, lp, cycles, rep):
    ref = np.array([float(x) for x in rep["beta"]])
    assert cycles == rep["cycles_run"]
    assert close(beta, ref, BETA_REL, ZERO_ABS)
    assert abs(lp - float(rep["log_posterior"])) <= LL_REL * abs(float(rep["log_posterior"]))


def test_config5_replicates_batched_engine(ds1m, dds1m, golden):
    """the reference's replicate estimates r = 0..3 from one batched launch
    per cycle (subject multiplicities as weights), warm from beta_full"""
    beta_full = np.array([float(x) for x in golden["bootstrap"]["expected"]["beta_full"]])
    W = np.stack([np.bincount(B.resample(ds1m, 77, r + 1), minlength=ds1m.num_subjects)
                  for r in range(4)]).astype(np.int32)
    fits, status = B.fit_batch(dds1m, [B.normal_prior(0.1)] * 4, W, np.tile(beta_full, (4, 1)))
    for r, rep in enumerate(golden["replicates"]):
        assert status[r] is None
        _check_rep(fits[r].beta_map, fits[r].log_posterior, fits[r].cycles_run, rep)


def test_config5_replicates_subset_route(ds1m, dds1m, golden):
    """... and from the device subset builder + the single-fit kernel"""
    beta_full = np.array([float(x) for x in golden["bootstrap"]["expected"]["beta_full"]])
    for r, rep in enumerate(golden["replicates"][:2]):
        sub = dds1m.subset(B.resample(ds1m, 77, r + 1))
        f = B.fit(sub, B.normal_prior(0.1), B.SolverConfig(), beta_full)
        sub.close()
        _check_rep(f.beta_map, f.log_posterior, f.cycles_run, rep)
