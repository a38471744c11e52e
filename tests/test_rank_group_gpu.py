"""The multi-process patient-sharded fit with world size 2 on
ONE B200: two processes, one shard each, the real multi-process path --
exchange areas exported and opened through CUDA IPC, every CTA of both ranks
adding its limbs into both ranks' areas inside the sweep kernel, host
collectives over gloo.  The two contexts time-slice the GPU, so every
exchange waits for the other process's slice (slow, but the protocol is the
one 8 GPUs run).  The result must equal the single-launch LocalGroup of the
same two shards bit for bit (same CTAs, same integer sums).

Also pinned here: a failure on one rank's host side reaches
every rank (status agreement, no hang), and a peer that stops publishing
turns into an error after the bounded exchange spin instead of a hang.
"""
import os
import socket
import time

import numpy as np
import pytest

from conftest import load_golden
from paper_1208_0945_b200 import bsccs as B
from paper_1208_0945_b200 import datagen, sharding

CTAS = 74  # each rank's launch: half the SMs (the two never run concurrently)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _skewed_dataset():
    """drug 0 appears only among the later subjects, so a huge beta_0
    overflows x'beta (|x'beta| > 700, engine.hpp:56-65) in the last shard only"""
    rng = B.Rng(77)
    recs = []
    for s in range(400):
        eras = []
        for _ in range(rng.uniform_int(2, 5)):
            exp = [j for j in range(1, 6) if rng.uniform() < 0.3]
            if s >= 300 and rng.uniform() < 0.5:
                exp = [0] + exp
            eras.append(B.Era(rng.uniform_int(5, 30), rng.uniform_int(0, 2), exp))
        recs.append(B.SubjectRecord(f"s{s}", eras))
    return B.build_dataset(recs, 6)


def _worker(rank, world, port_no, mode, q, go):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "oracle"), str(root / "tests")]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    os.environ["BSCCS_XCHG_TIMEOUT_S"] = "20"
    import torch.distributed as dist

    from paper_1208_0945_b200 import bsccs as Bw
    from paper_1208_0945_b200 import datagen as dg
    from paper_1208_0945_b200 import sharding as sh

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if mode == "fit":
            ds = dg.fast_sccs(10_300, 100, 2.0)
            shard = sh.shard_dataset(ds, world, only=rank)[0]
            g = sh.RankGroup(shard, 0, ctas=CTAS)
            t0 = time.time()
            r = g.fit(Bw.normal_prior(0.1))
            q.put((rank, "ok", r.beta_map.tobytes(), r.log_posterior, r.cycles_run, time.time() - t0))
            g.close()
        elif mode == "agree":
            ds = _skewed_dataset()
            shard = sh.shard_dataset(ds, world, only=rank)[0]
            g = sh.RankGroup(shard, 0, ctas=CTAS)
            init = np.zeros(ds.num_drugs)
            init[0] = 701.0
            try:
                g.fit(Bw.normal_prior(1.0), init_beta=init)
                q.put((rank, "no error"))
            except Exception as e:
                q.put((rank, type(e).__name__, str(e)))
            g.close()
        elif mode == "timeout":
            ds = dg.fast_sccs(10_300, 100, 2.0)
            shard = sh.shard_dataset(ds, world, only=rank)[0]
            g = sh.RankGroup(shard, 0, ctas=CTAS)
            if rank == 0:
                t0 = time.time()
                try:
                    g.fit(Bw.normal_prior(0.1))
                    q.put((rank, "no error", time.time() - t0))
                except Exception as e:
                    q.put((rank, type(e).__name__, str(e), time.time() - t0))
            else:  # joins the group, then never fits; stays alive until told
                q.put((rank, "idle"))
                go.wait(300)
            q.close()
            q.join_thread()  # flush the queue's feeder thread before the hard exit
            os._exit(0)  # no collective close: the peer is gone from the protocol
    except Exception as e:  # pragma: no cover
        q.put((rank, "error", repr(e)))
        raise
    finally:
        if mode != "timeout":
            dist.destroy_process_group()


def _run(mode, timeout=600):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q, go = ctx.Queue(), ctx.Event()
    port_no = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port_no, mode, q, go)) for r in range(2)]
    for p in ps:
        p.start()
    out = {}
    try:
        deadline = time.time() + timeout
        while len(out) < 2:
            item = q.get(timeout=max(1.0, deadline - time.time()))
            out[item[0]] = item
            if mode == "timeout" and 0 in out:
                go.set()
    finally:
        go.set()
        for p in ps:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    return out


@pytest.mark.gpu
def test_rank_group_world2_ipc_matches_local_group():
    out = _run("fit")
    for r in (0, 1):
        assert out[r][1] == "ok", out[r]
    b0, b1 = (np.frombuffer(out[r][2], dtype=np.float64) for r in (0, 1))
    assert np.array_equal(b0, b1) and out[0][3] == out[1][3] and out[0][4] == out[1][4]
    # the same two shards in one cooperative launch (same CTAs per shard)
    ds = datagen.fast_sccs(10_300, 100, 2.0)
    grp = sharding.LocalGroup(sharding.shard_dataset(ds, 2), 0, [CTAS, CTAS])
    loc = grp.fit(B.normal_prior(0.1))
    grp.close()
    assert np.array_equal(loc.beta_map, b0)
    assert loc.log_posterior == out[0][3] and loc.cycles_run == out[0][4]
    # and the reference's fit of the unsharded dataset (tests/golden/fast_10k.json)
    g = load_golden("fast_10k.json")
    ref = np.array([float(x) for x in g["beta"]])
    assert np.max(np.abs(b0 - ref) / np.maximum(np.abs(ref), 1e-300)) <= 1e-6
    assert abs(out[0][3] - float(g["log_posterior"])) <= 1e-8 * abs(float(g["log_posterior"]))
    assert out[0][4] == g["cycles_run"]


@pytest.mark.gpu
def test_rank_group_host_failure_reaches_every_rank():
    """init beta overflows x'beta in shard 1 only: rank 1's dense rebuild
    raises numeric_error (engine.hpp:56-65); rank 0 must raise too (status
    agreement through the exchange), not poll forever"""
    out = _run("agree", timeout=300)
    assert out[1][1] == "NumericError" and "overflow" in out[1][2], out[1]
    assert out[0][1] == "NumericError" and "another rank" in out[0][2], out[0]


@pytest.mark.gpu
def test_rank_group_silent_peer_times_out():
    """a peer that never publishes: the bounded spin ends the sweep with an
    error (BSCCS_XCHG_TIMEOUT_S = 20 in the workers) instead of a hang"""
    out = _run("timeout", timeout=300)
    assert out[1][1] == "idle"
    assert out[0][1] == "InternalError" and "stopped publishing" in out[0][2], out[0]
    assert out[0][3] < 120


def test_skewed_dataset_overflows_last_shard_only(port):
    """CPU check of the premise of the agreement test"""
    ds = _skewed_dataset()
    shards = sharding.shard_dataset(ds, 2)
    init = np.zeros(ds.num_drugs)
    init[0] = 701.0
    import pyoracle
    with pytest.raises(pyoracle.OracleError):
        port.init_state(shards[1].dataset, init)
    port.init_state(shards[0].dataset, init)
