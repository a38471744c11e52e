"""Patient sharding.

CPU: shard / merge round trips, balanced bounds, and a world-size-2 gloo run
in which each rank owns one shard, computes its (sum n*w, sum n*w(1-w)) and
log-likelihood partials with the C oracle, and all-reduces them -- the
host-side protocol of the multi-GPU sweep -- checked against the unsharded
oracle.  GPU: the same shards bound into one cooperative launch (LocalGroup)
reproduce the single-shard device fit.
"""
import os
import socket

import numpy as np
import pytest

from helpers import random_dataset
from paper_1208_0945_b200 import bsccs as B
from paper_1208_0945_b200 import datagen, sharding


def test_shard_merge_round_trip():
    rng = B.Rng(11)
    for trial in range(6):
        ds = random_dataset(rng, rng.uniform_int(1, 6), rng.uniform_int(5, 80))
        for n in (1, 2, 3, 5):
            shards = sharding.shard_dataset(ds, n)
            assert len(shards) == n
            assert sum(s.dataset.num_subjects for s in shards) == ds.num_subjects
            assert sharding.merge_shards(shards) == ds
            for s in shards:
                assert np.array_equal(s.y_dot_x_global, ds.y_dot_x)
                assert np.array_equal(s.col_nnz_global, np.diff(ds.col_ptr))


def test_balanced_bounds_cover_and_balance():
    ds = datagen.fast_sccs(4000, 40, 3.0)
    b = sharding.balanced_subject_bounds(ds, 4)
    assert b[0] == 0 and b[-1] == ds.num_subjects and np.all(np.diff(b) > 0)
    shards = sharding.shard_dataset(ds, 4)
    work = [s.dataset.num_eras + s.dataset.nnz for s in shards]
    assert max(work) / min(work) < 1.05


def test_sharded_partials_sum_to_global(port):
    ds = datagen.fast_sccs(3000, 30, 3.0)
    beta = np.linspace(-0.4, 0.4, ds.num_drugs)
    full = port.init_state(ds, beta)
    shards = sharding.shard_dataset(ds, 3)
    sts = [port.init_state(s.dataset, beta) for s in shards]
    ll = sum(port.log_likelihood(s.dataset, st) for s, st in zip(shards, sts))
    assert abs(ll - port.log_likelihood(ds, full)) <= 1e-11 * abs(ll)
    for j in range(ds.num_drugs):
        g, h = port.grad_hess(ds, full, j)
        gs = hs = 0.0
        for s, st in zip(shards, sts):
            gl, hl = port.grad_hess(s.dataset, st, j)
            gs += float(s.dataset.y_dot_x[j]) - gl
            hs += -hl
        assert abs((float(ds.y_dot_x[j]) - gs) - g) <= 1e-9 * max(1.0, abs(g))
        assert abs(-hs - h) <= 1e-9 * max(1.0, abs(h))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port_no, q):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "oracle")]
    import torch
    import torch.distributed as dist

    import pyoracle
    from paper_1208_0945_b200 import bsccs as Bw
    from paper_1208_0945_b200 import datagen as dg
    from paper_1208_0945_b200 import sharding as sh

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ds = dg.fast_sccs(2500, 25, 3.0)
        mine = sh.shard_dataset(ds, world)[rank]
        port = pyoracle.Port()
        prior = Bw.normal_prior(0.5)
        J = ds.num_drugs
        beta = np.zeros(J)
        trust = np.ones(J)
        st = port.init_state(mine.dataset, beta)
        # sharded CCD: per coordinate, all-reduce the (gs, hs) partials
        # (the 16-byte exchange of the sweep kernel), identical step everywhere
        for cycle in range(4):
            for j in range(J):
                gl, hl = port.grad_hess(mine.dataset, st, j)
                t = torch.tensor([float(mine.dataset.y_dot_x[j]) - gl, -hl], dtype=torch.float64)
                dist.all_reduce(t)
                g = float(mine.y_dot_x_global[j]) - float(t[0])
                h = 0.0 if float(t[1]) == 0.0 else -float(t[1])
                step = port.penalized_step(prior, beta[j], g, h)
                d = float(np.clip(step, -trust[j], trust[j]))
                if d != 0.0:
                    port.sparse_update(mine.dataset, st, j, d)
                    beta[j] += d
                trust[j] = max(2 * abs(d), trust[j] / 2)
        ll = torch.tensor([port.log_likelihood(mine.dataset, st)], dtype=torch.float64)
        dist.all_reduce(ll)
        # exchange of 64-byte IPC-handle blobs (multi-GPU plumbing)
        blobs = [None] * world
        dist.all_gather_object(blobs, bytes([rank]) * 64)
        if rank == 0:
            full = port.fit(ds, prior, Bw.SolverConfig(max_cycles=4, epsilon=1e-300))
            q.put((beta.tolist(), float(ll[0]), full["beta"].tolist(), [b[0] for b in blobs]))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharded_ccd_matches_unsharded():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port_no, q)) for r in range(2)]
    for p in procs:
        p.start()
    beta, ll, full_beta, blob_ranks = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert blob_ranks == [0, 1]
    np.testing.assert_allclose(beta, full_beta, rtol=1e-9, atol=1e-12)
    assert np.isfinite(ll)


@pytest.mark.gpu
@pytest.mark.parametrize("nshards,virtual", [(2, False), (3, False), (2, True), (4, True)])
def test_local_group_matches_single_fit(nshards, virtual):
    """virtual=True: each shard is a separate 'rank' with its own exchange
    area, every CTA adds into all areas with system-scope adds -- the
    multi-GPU protocol on one device."""
    ds = datagen.config_dataset("10k")
    prior = B.laplace_prior(0.1)
    single = B.fit(ds, prior)
    grp = sharding.LocalGroup(sharding.shard_dataset(ds, nshards), virtual_ranks=virtual)
    res = grp.fit(prior)
    grp.close()
    assert res.cycles_run == single.cycles_run
    nz = single.beta_map != 0
    assert np.all(res.beta_map[~nz] == 0.0)
    assert np.all(np.abs(res.beta_map[nz] - single.beta_map[nz]) <= 1e-9 * np.abs(single.beta_map[nz]))
    assert abs(res.log_posterior - single.log_posterior) <= 1e-11 * abs(single.log_posterior)


@pytest.mark.gpu
def test_local_group_oracle_case_golden():
    from conftest import load_golden
    from helpers import fa, prior_from
    g = load_golden("oracle_case.json")
    ds = datagen.simulate(datagen.oracle_case_config())
    grp = sharding.LocalGroup(sharding.shard_dataset(ds, 4))
    for fit in g["fits"]:
        res = grp.fit(prior_from(fit["prior"]))
        ref = fa(fit["beta"])
        assert res.cycles_run == fit["cycles_run"]
        assert np.all(np.abs(res.beta_map - ref) <= 1e-6 * np.abs(ref))
        lp = float(fit["log_posterior"])
        assert abs(res.log_posterior - lp) <= 1e-8 * abs(lp)
    grp.close()


def _rank_worker(port_no, q):
    import os
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "oracle")]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    import numpy as np
    import torch.distributed as dist

    from paper_1208_0945_b200 import bsccs as Bw
    from paper_1208_0945_b200 import datagen as dg
    from paper_1208_0945_b200 import sharding as sh

    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        ds = dg.fast_sccs(6000, 30, 3.0)
        prior = Bw.laplace_prior(0.1)
        shard = sh.shard_dataset(ds, 1)[0]
        g = sh.RankGroup(shard, 0)
        r = g.fit(prior)
        g.close()
        s = Bw.fit(ds, prior)
        q.put(("ok", r.cycles_run, s.cycles_run, bool(np.array_equal(r.beta_map, s.beta_map)),
               r.log_posterior, s.log_posterior))
    except Exception as e:  # pragma: no cover
        q.put(("error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_rank_group_world1_matches_single_fit():
    """The multi-process entry points end to end on one device: exchange-area
    IPC handle export, peer open (own entry skipped), group fit through the
    rank's area -- bit for bit the single fit (same kernel and partition)"""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_rank_worker, args=(_free_port(), q))
    p.start()
    got = q.get(timeout=300)
    p.join(timeout=120)
    assert got[0] == "ok", got
    _, c1, c2, same, lp1, lp2 = got
    assert c1 == c2 and same and lp1 == lp2


@pytest.mark.gpu
@pytest.mark.parametrize("nshards", [2, 4, 8])
def test_hierarchical_exchange_bitwise_equals_flat(nshards, monkeypatch):
    """virtual ranks with the hierarchical exchange (each rank's CTAs add into
    its local area, its CTA 0 forwards the integer sums: one arrival per rank
    on every polled word) and with the flat one (every CTA into every area):
    the same integer sums, so the same bits -- and the unsharded fit to 1e-9"""
    ds = datagen.config_dataset("10k")
    prior = B.laplace_prior(0.1)
    out = {}
    for mode in ("flat", "hier"):
        monkeypatch.setenv("BSCCS_XCHG", mode)
        grp = sharding.LocalGroup(sharding.shard_dataset(ds, nshards), virtual_ranks=True)
        out[mode] = grp.fit(prior)
        grp.close()
    a, b = out["flat"], out["hier"]
    assert np.array_equal(a.beta_map, b.beta_map) and a.log_posterior == b.log_posterior
    assert a.cycles_run == b.cycles_run
    single = B.fit(ds, prior)
    assert a.cycles_run == single.cycles_run
    nz = single.beta_map != 0
    assert np.all(np.abs(a.beta_map[nz] - single.beta_map[nz]) <= 1e-9 * np.abs(single.beta_map[nz]))


@pytest.mark.gpu
@pytest.mark.slow
@pytest.mark.parametrize("nshards,virtual", [(2, False), (4, True)])
def test_sharded_config3_matches_reference_golden(nshards, virtual):
    """the north-star configuration (10M x 4,000, Laplace 0.1) patient-sharded:
    2 shards in one launch, and 4 virtual ranks (every CTA adds into every
    rank's exchange area, the multi-GPU protocol on one device) -- against
    the reference's fit of the same dataset"""
    from conftest import GOLDEN, load_golden
    from helpers import fa, prior_from
    if not (GOLDEN / "fit_10M_laplace.json").exists():
        pytest.skip("fit_10M_laplace.json not generated")
    g = load_golden("fit_10M_laplace.json")
    ds = datagen.config_dataset("10M")
    assert (ds.num_subjects, ds.num_eras, ds.nnz) == (g["sizes"]["N"], g["sizes"]["K"], g["sizes"]["nnz"])
    grp = sharding.LocalGroup(sharding.shard_dataset(ds, nshards), virtual_ranks=virtual)
    res = grp.fit(prior_from(g["prior"]))
    grp.close()
    ref = fa(g["beta"])
    assert res.cycles_run == g["cycles_run"]
    zero = ref == 0.0
    assert np.all(np.abs(res.beta_map[zero]) <= 1e-9)
    assert np.all(np.abs(res.beta_map[~zero] - ref[~zero]) <= 1e-6 * np.abs(ref[~zero]))
    lp = float(g["log_posterior"])
    assert abs(res.log_posterior - lp) <= 1e-8 * abs(lp)
