"""bench.py's N > 1 path end to end (the driver's scaling run launches it
under torchrun, one rank per GPU): two ranks time-sliced on the one B200
(BSCCS_BENCH_SHARE_GPU=1, host collectives on gloo), the patient-sharded
fit through RankGroup with its e2e leg, and the many_fit block dealt to
both ranks as replicas.  Rank 0 prints one JSON line; parity against the
reference goldens must pass in both blocks."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_sharded_and_replicas():
    env = dict(os.environ, BSCCS_BENCH_SHARE_GPU="1", BSCCS_XCHG_TIMEOUT_S="60")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"),
           "--gpus", "2", "--workload", "10k", "--prior", "normal", "--steps", "1", "--warmup", "1"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert "patient-sharded x2" in d["config"]["parallelism"]
    assert d["parity_vs_reference_golden"]["pass"], d["parity_vs_reference_golden"]
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    m = d["many_fit"]
    assert m["n_gpus"] == 2 and m["failed"] == 0
    assert m["parity_vs_reference_replicates"]["pass"], m["parity_vs_reference_replicates"]
    assert "32 bootstrap refits" in m["workload"]
