#!/usr/bin/env python
"""Benchmark of the B200 CCD hot path (BASELINE.json north-star target, config 3).

Headline workload (default, every N): synthetic SCCS 10M patients (9.61M
kept, 145.1M eras) x 4,000 sparse indicators, Laplace prior sigma^2 = 0.1,
fp64, from the fast generator of SURVEY §8(d) (seed 20261017).  One step =
one full MAP fit to convergence (`fit()` entry with the dataset
device-resident -> FitResult on the host: init_state, every cycle, final
dense rebuild, log-posterior).  metric = coordinate updates/s (non-skipped
coordinate steps / fit time, solver.hpp:116-151); time to convergence =
ms_per_step.

  N = 1: one fit on one GPU.
  N > 1 (torchrun): ONE fit patient-sharded over the ranks (SURVEY §8(e),
         sharding.RankGroup: per-coordinate exchange inside the sweep kernel
         over peer memory); value = that fit's updates/s, time = max over
         ranks; scaling "strong".  --replicas runs N independent fits instead.

Secondary blocks at N = 1: config 2 (1M x 1,500 single fit, its own roofline,
e2e and parity) and many_fit (16 bootstrap refits of the 1M set in one
batched launch per cycle, parity against the reference's replicates).

  python bench.py [--gpus N --steps K --warmup W]          # this repo's path
  python bench.py --impl reference [...]                    # reference CPU arm

The reference arm runs the UNMODIFIED reference (oracle/_ref: the reference
headers compiled by oracle/Makefile) on the same synthetic dataset, built by
a generator on the reference's own Rng (no product library in its process):
each step is the reference's run_cycle (solver.hpp:101-166) over a fixed
column sample of the dataset against the full-size state -- a bounded
sample of the same workload, in the same unit.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "CCD coordinate updates/s (MAP fit to convergence)"
UNIT = "coordinate updates/s"
WORKLOADS = {  # name -> (attempts, drugs, lambda_x); SURVEY §8(d)
    "10k": (10_300, 100, 2.0),
    "1M": (1_030_000, 1500, 3.0),
    "10M": (10_300_000, 4000, 3.0),
}
CONFIG_NAME = {"1M": "BASELINE.json configs[1]", "10M": "BASELINE.json configs[2] (north-star target)",
               "10k": "SURVEY §6 10k row"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="10M", choices=list(WORKLOADS))
    ap.add_argument("--zipf", action="store_true")
    ap.add_argument("--prior", default="laplace", choices=["laplace", "normal"])
    ap.add_argument("--variance", type=float, default=0.1)
    ap.add_argument("--cpu-sample-coords", type=int, default=0,
                    help="columns in the CPU reference sample (0: ~1.5 s of single-core work per step)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-config2", action="store_true", help="skip the config-2 (1M) block")
    ap.add_argument("--no-many-fit", action="store_true", help="skip the batched 16-refit block (k_bccd)")
    ap.add_argument("--replicas", action="store_true", help="N>1: independent fits per rank instead of one sharded fit")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def parallelism(args, world):
    if world == 1:
        return "single GPU"
    if args.replicas:
        return f"replicas x{world} (independent fits per GPU)"
    return f"patient-sharded x{world} (one fit; per-coordinate exchange over NVLink peer memory)"


def workload_config(args, world, sizes):
    """identical keys in both arms (the driver compares them)"""
    N, K, J, nnz = sizes
    return {"workload": f"synthetic SCCS {args.workload} ({'zipf' if args.zipf else 'uniform'} prevalence) x {J}, "
                        f"{args.prior} prior sigma^2={args.variance}, fit to convergence ({CONFIG_NAME[args.workload]})",
            "generator": "SURVEY §8(d) fast generator, seed 20261017",
            "prior": args.prior, "variance": args.variance, "parallelism": parallelism(args, world),
            "N": int(N), "K": int(K), "J": int(J), "nnz": int(nnz),
            "l2": f"inputs larger than L2: {(8 * nnz + 8 * K + 16 * N) / 1e9:.2f} GB CSC + "
                  f"{(32 * K + 16 * N) / 1e9:.2f} GB state resident (L2 126 MB)"}


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = Path(f"/tmp/bench_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.15)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.path.exists():
            return None
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        self.path.unlink(missing_ok=True)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "samples": len(sm),
                "reasons": sorted(reasons)}


class Prior:  # duck-typed PriorSpec for the oracle bindings (no product import in the reference arm)
    def __init__(self, kind, variance):
        self.kind, self.variance, self.variance_is_laplace_scale = kind, variance, False


class Cfg:  # SolverConfig defaults (solver.hpp:21-46)
    epsilon, max_cycles, convergence, trust_init, precision, path = 0.0005, 1000, 0, 1.0, 1, 0
    dense_refresh_interval, random_cycle, cycle_seed, min_parallel_nnz = 50, 0, 0, 4096

    def __init__(self, partitions=1):
        self.partitions = partitions


def oracle_prior(args):
    return Prior(2 if args.prior == "laplace" else 1, args.variance)


def sample_columns(J, S):
    S = max(1, min(J, S))
    return np.unique((np.arange(S) * J) // S).astype(np.int32)


def default_sample(args):
    if args.cpu_sample_coords:
        return args.cpu_sample_coords
    # ~1.5 s of single-core reference work per step (24 ms per
    # coordinate at 10M, 3.7 ms at 1M)
    return {"10M": 64, "1M": 400, "10k": 100}[args.workload]


def reference_sample(rds, cols, args, steps, threads=1, partitions=1):
    """The reference's run_cycle over a column sample of `rds` (same subjects
    and eras, so the per-coordinate work and the state's footprint are the
    full workload's), `steps` cycles.  Returns seconds per cycle."""
    sample = rds.columns(cols)
    cfg = Cfg(partitions=partitions)
    st = sample.state(None, cfg)
    if threads > 1:
        st.set_threads(threads)
    prior = oracle_prior(args)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        st.run_cycle(prior, cfg)
        times.append(time.perf_counter() - t0)
    del st, sample
    return times


def golden_for(args):
    names = {"1M": "fit_1M_laplace.json", "10M": "fit_10M_laplace.json", "10k": "fast_10k.json"}
    if args.zipf:
        names = {"1M": "fit_1M_zipf_laplace.json"}
    name = names.get(args.workload)
    p = ROOT / "tests" / "golden" / (name or "")
    if not name or not p.exists():
        return None
    g = json.loads(p.read_text())
    if g["prior"]["kind"] != args.prior or float(g["prior"]["variance"]) != args.variance:
        return None
    return g


def digest(ds) -> str:
    h = hashlib.sha256()
    for a in ds.arrays():
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def parity_vs(g, beta, log_posterior, cycles, digest_ok=None):
    """the north-star bar: beta 1e-6 relative (1e-9 absolute for reference
    zeros), log-posterior 1e-8 relative, identical cycle count"""
    if g is None:
        return None
    ref = np.array([float(x) for x in g["beta"]])
    zero = ref == 0.0
    rel = np.abs(beta[~zero] - ref[~zero]) / np.abs(ref[~zero])
    za = np.abs(beta[zero]).max(initial=0.0)
    lp = float(g["log_posterior"])
    out = {"beta_max_rel": float(rel.max(initial=0.0)), "zeros_max_abs": float(za),
           "log_posterior_rel": abs(log_posterior - lp) / abs(lp), "cycles": [int(cycles), int(g["cycles_run"])]}
    ok = rel.max(initial=0.0) <= 1e-6 and za <= 1e-9 and abs(log_posterior - lp) <= 1e-8 * abs(lp) \
        and cycles == g["cycles_run"]
    if digest_ok is not None:
        out["dataset_digest_matches_golden"] = bool(digest_ok)
        ok = ok and digest_ok
    out["pass"] = bool(ok)
    return out


# ============================================================ reference arm


def main_reference(args, rank, world):
    if rank != 0:
        return  # rank 0 alone runs the CPU reference
    sys.path.insert(0, str(ROOT / "oracle"))
    import pyoracle  # the reference compiled untouched (oracle/_ref); no product library is loaded

    ref = pyoracle.Reference()
    cores = host_cores()
    attempts, drugs, lam = WORKLOADS[args.workload]
    t0 = time.time()
    rds = ref.fast_sccs(attempts, drugs, lam, args.zipf, threads=cores)
    gen_s = time.time() - t0
    sizes = rds.sizes()
    N, K, J, nnz = sizes["N"], sizes["K"], sizes["J"], sizes["nnz"]
    cols = sample_columns(J, default_sample(args))
    # canonical route: partitions = 1, one core (the anchor)
    times = reference_sample(rds, cols, args, args.warmup + args.steps)
    per = float(np.mean(times[args.warmup:]))
    value = cols.size / per
    # the reference's own parallel route beside it: partitions = P, ThreadPool(P - 1)
    pt = reference_sample(rds, cols, args, 1 + min(3, args.steps), threads=cores, partitions=cores)
    pper = float(np.mean(pt[1:]))
    sample = (f"reference run_cycle (solver.hpp:101-166, partitions=1, 1 core) over {cols.size} of the {J} columns "
              f"(evenly spaced) of the same {args.workload} dataset against its full-size state; one cycle of the "
              f"sample per step, {args.warmup} warm-up + {args.steps} timed")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True,
            "scaling": "strong" if (world > 1 and not args.replicas) else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": workload_config(args, world, (N, K, J, nnz)),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "reference", "sample": sample,
                             "cpu_model": cpu_model(), "host_cores": cores},
            "parallel_route": {"value": cols.size / pper, "unit": UNIT, "cores": cores, "partitions": cores,
                               "ms_per_step": pper * 1e3,
                               "note": "the reference's parallel route (ThreadPool(P-1)); its update stays serial "
                                       "(solver.hpp:147), so it is not faster"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "setup": {"generate_s": gen_s}}
    print(json.dumps(line), flush=True)


# ============================================================ our arm


def pinned_copy(ds):
    """the step's inputs in page-locked host memory (the caller's buffers)"""
    import torch
    from paper_1208_0945_b200 import bsccs as B
    held = []
    for a in ds.arrays():
        t = torch.empty(a.size, dtype={np.int32: torch.int32, np.int64: torch.int64}[a.dtype.type], pin_memory=True)
        v = t.numpy()
        v[:] = a
        held.append((t, v))
    return held, B.Dataset(*[v for _, v in held])


def upload_bytes(host):
    """bytes the e2e legs copy host -> device: every CSC array but the per-pair
    subjects, which bsccs_dataset_create derives on the device from the rows
    (subjects = NULL)"""
    return int(sum(a.nbytes for a in host.arrays()) - host.subjects.nbytes)


def sweep_kernel():
    """which sweep kernel the last cycle launched (bsccs_debug_last_sweep)"""
    from paper_1208_0945_b200 import _native
    k = _native.lib().bsccs_debug_last_sweep()
    return {1: "k_ccd", 2: "k_rcd", 3: "k_rcd+k_ccd"}.get(k, "k_ccd")


KERNEL_DESC = {"k_rcd": "k_rcd (resident-beta persistent sweep, 1 launch per cycle)",
               "k_ccd": "k_ccd (per-era-state persistent sweep, 1 launch per cycle)",
               "k_rcd+k_ccd": "k_rcd handing over to k_ccd"}


def roofline_of(results, elapsed_ms, peak, peak_src, traffic_key):
    sweeps = sum(r.cycles_run for r in results)
    sweep_s = sum(r.sweep_seconds for r in results)
    alg = sum(r.algorithmic_bytes for r in results)
    achieved = alg / sweep_s / 1e9
    kern = sweep_kernel()
    traffic = None
    tp = ROOT / "profiles" / "sweep_traffic.json"
    if tp.exists():
        try:
            traffic = json.loads(tp.read_text()).get(kern, {}).get(traffic_key)
        except Exception:
            traffic = None
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "kernel": KERNEL_DESC.get(kern, kern),
            "bytes_per_launch": alg / sweeps, "ms_per_launch": sweep_s / sweeps * 1e3,
            "share_of_step": sweep_s * 1e3 / elapsed_ms, "peak_source": peak_src,
            "algorithmic_bytes": "SURVEY §8(d): per visited coordinate 16*nnz_j + 12*u_j, per moved one "
                                 "+ 28*nnz_j + 8*u_j, per cycle + 32*K (counted per launch by the library)",
            "traffic_note": "ncu dram__bytes_read.sum + dram__bytes_write.sum of one launch "
                            "(profiles/sweep_traffic.json); k_rcd streams 32-B pair records instead of "
                            "gathering per-era state, so its DRAM bytes fall below the algorithmic count"}


def timed_region(fn, steps, barrier, torch):
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = []
    barrier()
    start.record()
    for _ in range(steps):
        out.append(fn())
    end.record()
    barrier()
    return out, start.elapsed_time(end)


def main_ours(args, rank, world, local):
    import torch

    from paper_1208_0945_b200 import bsccs as B
    from paper_1208_0945_b200 import datagen

    # test hook: BSCCS_BENCH_SHARE_GPU=1 puts every rank on device 0 (the
    # protocol on one GPU, time-sliced; NCCL refuses two ranks per device, so
    # the host collectives then run on gloo)
    share = os.environ.get("BSCCS_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sharded = world > 1 and not args.replicas

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device="cpu" if share else "cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    attempts, drugs, lam = WORKLOADS[args.workload]
    t0 = time.time()
    ds = datagen.fast_sccs(attempts, drugs, lam, args.zipf,
                           threads=max(1, host_cores() // world) if world > 1 else 0)
    gen_s = time.time() - t0
    g = golden_for(args)
    digest_ok = (digest(ds) == g["digest"]) if (g is not None and rank == 0) else None
    prior = B.laplace_prior(args.variance) if args.prior == "laplace" else B.normal_prior(args.variance)
    cfg = B.SolverConfig()
    t0 = time.time()
    if sharded:
        from paper_1208_0945_b200 import sharding
        shard = sharding.shard_dataset(ds, world, only=rank)[0]
        grp = sharding.RankGroup(shard, local)
        info = grp.dds.info()
        fit_fn = lambda: grp.fit(prior, cfg)  # noqa: E731
    else:
        shard = None
        dds = B.DeviceDataset(ds, device=local)
        info = dds.info()
        fit_fn = lambda: B.fit(dds, prior, cfg)  # noqa: E731
    upload_s = time.time() - t0

    for _ in range(args.warmup):
        fit_fn()
    launches0 = B.launch_count()
    with ClockSampler(local) as clk:
        results, elapsed_ms = timed_region(fit_fn, args.steps, barrier, torch)
    launches = B.launch_count() - launches0
    elapsed_ms = max_over_ranks(elapsed_ms)
    visited = sum(r.coordinates_visited for r in results)
    value = visited * (1 if sharded else world) / (elapsed_ms * 1e-3)
    ms_per_step = elapsed_ms / args.steps
    peak, peak_src = load_peaks()
    key = args.workload + ("_zipf" if args.zipf else "") + (f"_shard{world}" if sharded else "")
    roofline = roofline_of(results, elapsed_ms, peak, peak_src, key)
    if sharded:
        roofline["note"] = f"rank {rank}'s shard ({info['nnz']} of {ds.nnz} pairs); bytes are this rank's"

    # end to end through the public API with host buffers: pinned CSC arrays
    # (or this rank's shard) -> device build -> fit -> beta to the host
    e2e = None
    if not args.no_e2e:
        held, host = pinned_copy(shard.dataset if sharded else ds)
        h2d = upload_bytes(host)
        d2h = ds.num_drugs * 8

        def e2e_step():
            if sharded:
                from paper_1208_0945_b200 import sharding
                sh = sharding.Shard(host, shard.subject_begin, shard.subject_end, shard.era_begin,
                                    shard.y_dot_x_global, shard.col_nnz_global)
                gg = sharding.RankGroup(sh, local, upload_subjects=False)
                r = gg.fit(prior, cfg)
                gg.close()
                return r
            d = B.DeviceDataset(host, device=local, upload_subjects=False)
            r = B.fit(d, prior, cfg)
            d.close()
            return r

        for _ in range(min(args.warmup, 2)):
            e2e_step()
        l0 = B.launch_count()
        eres, e_ms = timed_region(e2e_step, args.steps, barrier, torch)
        e_ms = max_over_ranks(e_ms)
        e2e = {"value": sum(r.coordinates_visited for r in eres) * (1 if sharded else world) / (e_ms * 1e-3),
               "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e_ms / args.steps,
               "path": ("bsccs_dataset_create_shard + RankGroup (IPC handles over torch.distributed) + "
                        "bsccs_group_fit" if sharded else "bsccs_dataset_create") +
                       " (pinned host CSC arrays -> HBM, per-pair subjects derived on the device, CSR/split build) + fit + "
                       "beta to host + destroy",
               "gpu_launches": B.launch_count() - l0}
        del held, host

    r0 = results[-1]
    parity = parity_vs(g, r0.beta_map, r0.log_posterior, r0.cycles_run, digest_ok) if rank == 0 else None

    # ---- config 2 and many-fit blocks (one GPU) --------------------------
    config2 = None
    many = None
    if world == 1 and not args.no_config2 and args.workload != "1M":
        config2 = bench_config2(args, B, datagen, torch, barrier, peak, peak_src, local)
    if not args.no_many_fit:  # N > 1: replicates dealt to ranks (configs 4/5 run as replicas)
        many = bench_many_fit(args, B, datagen, torch, barrier, peak, peak_src, local, rank, world, max_over_ranks)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sys.path.insert(0, str(ROOT / "oracle"))
        import pyoracle
        if pyoracle.available_ref():
            cols = sample_columns(ds.num_drugs, default_sample(args))
            rds = pyoracle.Reference().dataset(ds)
            times = reference_sample(rds, cols, args, 3)
            per = float(np.mean(times[1:]))
            cpu = {"value": cols.size / per, "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": f"reference run_cycle (partitions=1, 1 core) over {cols.size} evenly spaced columns of "
                             f"the same {args.workload} dataset against its full-size state; {per:.2f} s per sample "
                             f"cycle (2 timed after 1 warm-up)",
                   "cpu_model": cpu_model(), "host_cores": host_cores()}
            del rds

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, world, (ds.num_subjects, ds.num_eras, ds.num_drugs, ds.nnz)),
            "time_to_convergence_s": ms_per_step * 1e-3, "cycles_per_fit": r0.cycles_run,
            "sweeps_per_s": sum(r.cycles_run for r in results) / (elapsed_ms * 1e-3) * (1 if sharded else world),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "parity_vs_reference_golden": parity,
            "ctas_per_gpu": info["ctas"], "config2": config2, "many_fit": many,
            "setup": {"generate_s": gen_s, "upload_and_build_s": upload_s},
        }
        print(json.dumps(line), flush=True)
    if sharded:
        grp.close()
    if world > 1:
        torch.distributed.destroy_process_group()


def bench_config2(args, B, datagen, torch, barrier, peak, peak_src, local):
    """config 2 (1M x 1,500, Laplace 0.1) on one GPU: fit, roofline, e2e, parity"""
    attempts, drugs, lam = WORKLOADS["1M"]
    ds = datagen.fast_sccs(attempts, drugs, lam)
    prior = B.laplace_prior(0.1)
    cfg = B.SolverConfig()
    dds = B.DeviceDataset(ds, device=local)
    for _ in range(args.warmup):
        B.fit(dds, prior, cfg)
    res, ms = timed_region(lambda: B.fit(dds, prior, cfg), args.steps, barrier, torch)
    held, host = pinned_copy(ds)

    def e2e_step():
        d = B.DeviceDataset(host, device=local, upload_subjects=False)
        r = B.fit(d, prior, cfg)
        d.close()
        return r

    e2e_step()
    eres, ems = timed_region(e2e_step, args.steps, barrier, torch)
    p = ROOT / "tests" / "golden" / "fit_1M_laplace.json"
    g = json.loads(p.read_text()) if p.exists() else None
    r0 = res[-1]
    out = {"workload": "synthetic SCCS 1M (uniform) x 1500, laplace prior sigma^2=0.1, fit to convergence "
                       "(BASELINE.json configs[1])",
           "N": ds.num_subjects, "K": ds.num_eras, "J": ds.num_drugs, "nnz": ds.nnz,
           "value": sum(r.coordinates_visited for r in res) / (ms * 1e-3), "unit": UNIT,
           "time_to_convergence_s": ms / args.steps * 1e-3, "cycles_per_fit": r0.cycles_run,
           "roofline": roofline_of(res, ms, peak, peak_src, "1M"),
           "e2e": {"value": sum(r.coordinates_visited for r in eres) / (ems * 1e-3), "unit": UNIT,
                   "h2d_bytes_per_step": upload_bytes(host),
                   "d2h_bytes_per_step": ds.num_drugs * 8, "ms_per_step": ems / args.steps},
           "parity_vs_reference_golden": parity_vs(g, r0.beta_map, r0.log_posterior, r0.cycles_run,
                                                   digest(ds) == g["digest"] if g else None)}
    dds.close()
    del held, host
    return out


def bench_many_fit(args, B, datagen, torch, barrier, peak, peak_src, local, rank=0, world=1, max_over_ranks=None):
    """configs 4/5 shape: 16 bootstrap refits of the 1M set (resample seed 77,
    Normal 0.1, warm from the full-data fit) in one batched launch per cycle
    (k_bccd); replicates 0..3 checked against the reference's own replicate
    fits (tests/golden/drivers_1M.json, bootstrap.hpp:103-112).  With N ranks
    rank q fits replicates 16q .. 16q + 15 (independent fits are replicas:
    no data-path collective); the time is the max over ranks and the
    throughput counts every rank's fits."""
    mx = max_over_ranks or (lambda x: x)
    attempts, drugs, lam = WORKLOADS["1M"]
    ds = datagen.fast_sccs(attempts, drugs, lam)
    dds = B.DeviceDataset(ds, device=local)
    cfg = B.SolverConfig()
    mprior = B.normal_prior(0.1)
    full = B.fit(dds, mprior, cfg)
    R = 16
    W = np.stack([np.bincount(B.resample(ds, 77, rank * R + r + 1), minlength=ds.num_subjects)
                  for r in range(R)]).astype(np.int32)
    # the caller's weights in page-locked memory, like the CSC arrays of the
    # e2e legs (the 64 MB upload is then one DMA instead of staged copies)
    w_pinned = torch.empty(W.shape, dtype=torch.int32, pin_memory=True)
    w_pinned.numpy()[:] = W
    W = w_pinned.numpy()
    init = np.tile(full.beta_map, (R, 1))
    B.fit_batch(dds, [mprior] * R, W, init, cfg)  # warm-up
    barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    fits, st = B.fit_batch(dds, [mprior] * R, W, init, cfg)
    e.record()
    barrier()
    b_ms = mx(s.elapsed_time(e))
    ncyc = max(f.cycles_run for f in fits)
    bsweep, bbytes = fits[0].sweep_seconds, fits[0].algorithmic_bytes
    parity = None
    p = ROOT / "tests" / "golden" / "drivers_1M.json"
    if p.exists() and rank == 0:
        gd = json.loads(p.read_text())
        rows = []
        for rep in gd.get("replicates", []):
            f = fits[rep["r"]]
            rows.append(parity_vs(rep, f.beta_map, f.log_posterior, f.cycles_run))
        parity = {"replicates_checked": len(rows), "dataset_digest_matches_golden": digest(ds) == gd["digest"],
                  "beta_max_rel": max(x["beta_max_rel"] for x in rows) if rows else None,
                  "log_posterior_rel": max(x["log_posterior_rel"] for x in rows) if rows else None,
                  "cycles_equal": all(x["cycles"][0] == x["cycles"][1] for x in rows),
                  "pass": bool(rows) and all(x["pass"] for x in rows) and digest(ds) == gd["digest"]}
    # end to end through the public API: the 1M dataset from pinned host CSC
    # arrays, the 16 replicates' subject multiplicities and warm starts from
    # the host, the batched fit, every replicate's beta back to the host
    held, host = pinned_copy(ds)

    def e2e_step():
        d = B.DeviceDataset(host, device=local, upload_subjects=False)
        f, _ = B.fit_batch(d, [mprior] * R, W, init, cfg)
        d.close()
        return f

    e2e_step()
    eres, ems = timed_region(e2e_step, 1, barrier, torch)
    ems = mx(ems)
    e2e = {"value": world * R / (ems * 1e-3), "unit": "fits/s", "ms_per_step": ems, "fits_per_step": world * R,
           "coordinate_updates_per_s": world * sum(f.coordinates_visited for f in eres[0]) / (ems * 1e-3),
           "h2d_bytes_per_step": int(upload_bytes(host) + W.nbytes + init.nbytes),
           "d2h_bytes_per_step": int(R * ds.num_drugs * 8),
           "path": "bsccs_dataset_create (pinned host CSC) + bsccs_fit_batch (weights, warm starts from the host) + "
                   "betas to host + destroy"}
    del held, host
    out = {"workload": f"{world * R} bootstrap refits (config-5 shape: resample seed 77, Normal 0.1, warm start) of the "
                       f"1M dataset, {R} per GPU in one batched launch per cycle",
           "n_gpus": world, "scaling": "weak",
           "fits_per_s": world * R / (b_ms * 1e-3), "ms_per_fit": b_ms / (world * R),
           "single_fit_ms": full.device_seconds * 1e3,
           "coordinate_updates_per_s": world * sum(f.coordinates_visited for f in fits) / (b_ms * 1e-3),
           "failed": sum(x is not None for x in st), "cycles": ncyc,
           "roofline": {"bound": "hbm", "kernel": "k_bccd (batched weighted sweep, 16 fits)",
                        "achieved": bbytes / bsweep / 1e9, "peak": peak, "unit": "GB/s",
                        "frac": bbytes / bsweep / 1e9 / peak, "bytes_per_launch": bbytes / ncyc,
                        "ms_per_launch": bsweep / ncyc * 1e3, "peak_source": peak_src},
           "e2e": e2e, "parity_vs_reference_replicates": parity}
    dds.close()
    return out


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return main_reference(args, rank, world)
    return main_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
