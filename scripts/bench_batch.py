"""Many-fit workloads (BASELINE.json configs 4 and 5 shapes) on one B200:
the batched weighted engine against the materialised-subset engine, plus
the batched kernel's roofline.  Not the driver's bench line (bench.py keeps
config 2); results go to profiles/.

  python scripts/bench_batch.py [--workload 1M] [--replicates 16] [--cv]
"""
import argparse
import json
import sys
import time

sys.path[:0] = ['.', 'oracle']
import numpy as np

from paper_1208_0945_b200 import bootstrap as BT
from paper_1208_0945_b200 import bsccs as B
from paper_1208_0945_b200 import cross_validation as CV
from paper_1208_0945_b200 import datagen


def peak():
    try:
        return float(json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="1M")
    ap.add_argument("--replicates", type=int, default=16)
    ap.add_argument("--cv", action="store_true")
    ap.add_argument("--subset", action="store_true", help="also time the materialised-subset engine")
    a = ap.parse_args()
    ds = datagen.config_dataset(a.workload)
    dds = ds.on_device()
    N, J = ds.num_subjects, ds.num_drugs
    pk, src = peak()
    prior = B.normal_prior(0.1)
    full = B.fit(dds, prior)
    B.fit(dds, prior)
    # one batch of 16 bootstrap replicates, warm from the full fit (config 5)
    R = 16
    W = np.stack([np.bincount(B.resample(ds, 77, r + 1), minlength=N) for r in range(R)]).astype(np.int32)
    init = np.tile(full.beta_map, (R, 1))
    for rep in range(2):
        t0 = time.perf_counter()
        fits, st = B.fit_batch(dds, [prior] * R, W, init)
        wall = time.perf_counter() - t0
    sweep = fits[0].sweep_seconds
    byt = fits[0].algorithmic_bytes
    cyc = max(f.cycles_run for f in fits)
    print(json.dumps({"what": "k_bccd batch of 16 bootstrap refits (warm), Normal 0.1", "workload": a.workload,
                      "N": N, "J": J, "fits": R, "cycles": cyc, "wall_s": wall, "sweep_s": sweep,
                      "alg_bytes": byt, "achieved_gbs": byt / sweep / 1e9, "peak_gbs": pk,
                      "frac": byt / sweep / 1e9 / pk, "peak_source": src,
                      "per_fit_ms": wall / R * 1e3, "single_fit_ms": full.device_seconds * 1e3,
                      "coordinate_updates_per_s": sum(f.coordinates_visited for f in fits) / sweep}), flush=True)
    # bootstrap driver, both engines
    for eng in (["batched", "subset"] if a.subset else ["batched"]):
        cfg = BT.BootstrapConfig(replicates=a.replicates, seed=77, prior=prior, engine=eng)
        t0 = time.perf_counter()
        r = BT.run_bootstrap(dds, cfg)
        wall = time.perf_counter() - t0
        print(json.dumps({"what": f"run_bootstrap engine={eng}", "replicates": a.replicates, "wall_s": wall,
                          "per_replicate_ms": wall / a.replicates * 1e3, "used": r.used,
                          "total_cycles": r.total_cycles}), flush=True)
    if a.cv:
        lo, hi = np.log(0.001), np.log(10.0)
        grid = [float(np.exp(lo + (hi - lo) * i / 7.0)) for i in range(8)]
        for eng in (["batched", "subset"] if a.subset else ["batched"]):
            cfg = CV.CVConfig(folds=8, variance_grid=grid, seed=17, engine=eng)
            t0 = time.perf_counter()
            r = CV.grid_search_cv(dds, cfg)
            wall = time.perf_counter() - t0
            print(json.dumps({"what": f"grid_search_cv engine={eng} (8 folds x 8 points, laplace)", "wall_s": wall,
                              "fits": r.fits, "selected_variance": r.selected_variance,
                              "total_cycles": r.total_cycles,
                              "mean_pll": [float(x) for x in r.mean_predictive_ll]}), flush=True)


if __name__ == "__main__":
    main()
