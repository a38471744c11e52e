"""Generates tests/golden/*.json from the REFERENCE ITSELF.

Run here (where /root/reference exists and oracle/_ref/libbsccs_ref.so was
built from its untouched headers by oracle/Makefile):

    python tests/golden/make_golden.py [--large]

Every dataset is regenerated on the GPU box by our own generators
(paper_1208_0945_b200.datagen), so the fixtures store only a sha256 digest
of the flat CSC arrays plus the reference outputs.  --large adds the
config-2 (1M x 1500, Laplace 0.1) and config-3 (10M x 4000, Laplace 0.1)
reference fits (about 40 s and 11 min of CPU).
"""
from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import pyoracle as po  # noqa: E402
from paper_1208_0945_b200 import bsccs as B  # noqa: E402
from paper_1208_0945_b200 import datagen  # noqa: E402

OUT = Path(__file__).resolve().parent


def digest(ds: B.Dataset) -> str:
    h = hashlib.sha256()
    for a in ds.arrays():
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def prior_dict(p: B.PriorSpec):
    return {"kind": p.kind.name, "variance": p.variance}


def fit_dict(r):
    return {"beta": [repr(float(b)) for b in r["beta"]], "log_posterior": repr(r["log_posterior"]),
            "cycles_run": r["cycles_run"], "converged": r["converged"],
            "final_criterion": repr(r["final_criterion"])}


# testutil::random_records / random_dataset / random_beta (test_util.hpp:17-66)
def random_records(rng: B.Rng, num_drugs, num_subjects, exposure_prob=0.35, max_events=2):
    recs = []
    for s in range(num_subjects):
        eras = []
        for _ in range(rng.uniform_int(1, 6)):
            length = rng.uniform_int(1, 40)
            y = rng.uniform_int(0, max_events)
            exp = [j for j in range(num_drugs) if rng.uniform() < exposure_prob]
            eras.append(B.Era(length, y, exp))
        recs.append(B.SubjectRecord(f"s{s}", eras))
    return recs


def random_dataset(rng, num_drugs, num_subjects, exposure_prob=0.35):
    while True:
        recs = random_records(rng, num_drugs, num_subjects, exposure_prob)
        if any(e.event_count > 0 for r in recs for e in r.eras):
            return B.build_dataset(recs, num_drugs)


def random_beta(rng, num_drugs, scale=0.5):
    return [-scale + 2 * scale * rng.uniform() for _ in range(num_drugs)]


def ds_dict(ds: B.Dataset):
    return {k: v.tolist() for k, v in zip(
        ("subject_offsets", "events_per_subject", "era_lengths", "event_counts", "col_ptr", "rows", "subjects",
         "y_dot_x"), ds.arrays())}


def engine_cases(ref: po.Reference):
    """Random small datasets with reference engine outputs at a random beta:
    state vectors, (g, h) per coordinate, and state after sparse updates."""
    rng = B.Rng(4242)
    cases = []
    for trial in range(12):
        J = rng.uniform_int(1, 8)
        ds = random_dataset(rng, J, rng.uniform_int(5, 60))
        beta = random_beta(rng, J, 1.0)
        rds = ref.dataset(ds)
        st = rds.state(beta)
        s0 = st.get()
        gh = [st.grad_hess(j) for j in range(J)]
        ll0 = st.log_likelihood()
        steps = []
        for _ in range(6):
            j = rng.uniform_int(0, J - 1)
            d = -0.3 + 0.6 * rng.uniform()
            st.sparse_update(j, d)
            steps.append([j, repr(d)])
        s1 = st.get()
        cases.append({
            "dataset": ds_dict(ds), "beta": [repr(float(b)) for b in beta],
            "xbeta": [repr(float(x)) for x in s0["xbeta"]],
            "l_exp_xbeta": [repr(float(x)) for x in s0["l_exp_xbeta"]],
            "denominators": [repr(float(x)) for x in s0["denominators"]],
            "grad_hess": [[repr(g), repr(h)] for g, h in gh], "log_likelihood": repr(ll0),
            "updates": steps,
            "after": {k: [repr(float(x)) for x in s1[k]] for k in ("beta", "xbeta", "l_exp_xbeta", "denominators")},
            "ll_after": repr(st.log_likelihood()),
        })
    return cases


def small_suite(ref: po.Reference):
    """acceptance.cpp:65-95 small_suite (100 seeded simulate() instances),
    with reference fits for Normal(1.0) and Laplace(1.0) at epsilon 1e-8."""
    knobs = B.Rng(9001)
    seed = 1000
    out = []
    while len(out) < 100:
        drugs = None
        subjects = knobs.uniform_int(15, 50)
        drugs = knobs.uniform_int(2, 10)
        prev = 0.2 + 0.2 * knobs.uniform()
        tb = [1.6 * knobs.uniform() - 0.8 for _ in range(drugs)]
        cfg = datagen.SimConfig(subjects=subjects, drugs=drugs, min_eras=1, max_eras=6, min_era_length=5,
                                max_era_length=30, prevalence=[prev] * drugs, true_beta=tb,
                                baseline_log_rate_mean=-3.0, baseline_log_rate_sd=0.4, seed=seed)
        seed += 1
        try:
            rds = ref.simulate(cfg)
        except po.OracleError:
            continue
        ds = rds.to_host()
        if ds.num_subjects < 5:
            continue
        entry = {"sim": {"subjects": subjects, "drugs": drugs, "prevalence": repr(prev),
                         "true_beta": [repr(b) for b in tb], "seed": cfg.seed},
                 "digest": digest(ds), "fits": []}
        scfg = B.SolverConfig(epsilon=1e-8, max_cycles=10000)
        for prior in (B.normal_prior(1.0), B.laplace_prior(1.0)):
            entry["fits"].append({"prior": prior_dict(prior), **fit_dict(rds.fit(prior, scfg))})
        out.append(entry)
    return out


def oracle_case(ref: po.Reference):
    cfg = datagen.oracle_case_config()
    rds = ref.simulate(cfg)
    ds = rds.to_host()
    out = {"config": "BASELINE.json configs[0]: simulate() 10300 x 100, seed 12080945",
           "sizes": rds.sizes(), "digest": digest(ds), "fits": []}
    for prior in (B.normal_prior(0.1), B.normal_prior(1.0), B.laplace_prior(0.1)):
        out["fits"].append({"prior": prior_dict(prior), **fit_dict(rds.fit(prior, B.SolverConfig()))})
    # first-cycle trace (Normal 0.1): g, h, delta per coordinate through the
    # reference engine + penalized_step + clamp (solver.hpp:116-151)
    prior = B.normal_prior(0.1)
    st = rds.state()
    trace = []
    trust = np.ones(ds.num_drugs)
    beta = np.zeros(ds.num_drugs)
    for j in range(ds.num_drugs):
        g, h = st.grad_hess(j)
        step = ref.penalized_step(prior, beta[j], g, h)
        d = float(np.clip(step, -trust[j], trust[j]))
        if d != 0.0:
            st.sparse_update(j, d)
            beta[j] += d
        trust[j] = max(2 * abs(d), trust[j] / 2)
        trace.append([repr(g), repr(h), repr(d)])
    out["cycle1_trace_normal_0.1"] = trace
    return out


def fast_case(ref: po.Reference, name, attempts, drugs, lam, prior, zipf=False):
    t0 = time.time()
    ds = datagen.fast_sccs(attempts, drugs, lam, zipf)
    rds = ref.dataset(ds)
    r = rds.fit(prior, B.SolverConfig())
    print(f"  {name}: N={ds.num_subjects} K={ds.num_eras} nnz={ds.nnz} fit {r['seconds']:.1f}s "
          f"cycles={r['cycles_run']} (total {time.time() - t0:.1f}s)", flush=True)
    return {"workload": name, "attempts": attempts, "drugs": drugs, "lambda_x": lam, "zipf": zipf,
            "seed": datagen.FAST_SEED,
            "sizes": {"N": ds.num_subjects, "K": ds.num_eras, "J": ds.num_drugs, "nnz": ds.nnz},
            "digest": digest(ds), "prior": prior_dict(prior), "reference_fit_seconds_1core": r["seconds"],
            **fit_dict(r)}


def drivers_case(ref: po.Reference):
    """grid_search_cv (config 4's shape, scaled to the oracle case) and
    run_bootstrap (config 5's shape, 16 replicates) by the reference."""
    cfg = datagen.oracle_case_config()
    rds = ref.simulate(cfg)
    ds = rds.to_host()
    lo, hi = np.log(0.001), np.log(10.0)
    grid = [float(np.exp(lo + (hi - lo) * i / 7.0)) for i in range(8)]  # 8 points
    cv = {"folds": 8, "grid": grid,
          "prior": "laplace", "seed": 17, "warm_start": True}
    r = rds.grid_search_cv(cv["folds"], cv["grid"], B.PriorKind.laplace, cv["seed"], B.SolverConfig(),
                           warm_start=True, threads=8)
    cv["expected"] = {"variance_grid": r["variance_grid"].tolist(),
                      "predictive_ll": [[repr(float(x)) for x in row] for row in r["predictive_ll"]],
                      "cycles": r["cycles"].tolist(), "converged": r["converged"].tolist(),
                      "valid": r["valid"].tolist(),
                      "mean_predictive_ll": [repr(float(x)) for x in r["mean_predictive_ll"]],
                      "selected_index": r["selected_index"], "selected_variance": r["selected_variance"],
                      "total_cycles": r["total_cycles"]}
    boot = {"replicates": 16, "level": 0.95, "seed": 77, "prior": "normal", "variance": 0.1, "warm_start": True}
    b = rds.run_bootstrap(16, 0.95, 77, B.normal_prior(0.1), B.SolverConfig(), warm_start=True, threads=8)
    boot["expected"] = {k: ([repr(float(x)) for x in v] if isinstance(v, np.ndarray) else v) for k, v in b.items()}
    return {"config": "oracle case (simulate 10300 x 100, seed 12080945)", "digest": digest(ds),
            "resample_77_1_head": rds.resample(77, 1)[:32].tolist(), "cv": cv, "bootstrap": boot}


def drivers_1M(ref: po.Reference):
    """Configs 4 and 5 at their named size (1M x 1500) by the reference:
    the full config-4 grid_search_cv (8 folds x 8 points, Laplace, seed 17,
    warm), a 16-replicate prefix of config 5's run_bootstrap (Normal 0.1,
    seed 77, warm; replicate r depends only on (seed, r), so the prefix is
    an exact sub-run) and the per-replicate estimates of r = 0..3
    (bootstrap.hpp:103-112).  About 30 min on 8 cores."""
    from concurrent.futures import ThreadPoolExecutor
    t0 = time.time()
    ds = datagen.fast_sccs(1_030_000, 1500, 3.0)
    rds = ref.fast_sccs(1_030_000, 1500, 3.0, threads=8)
    out = {"workload": "1M", "attempts": 1_030_000, "drugs": 1500, "lambda_x": 3.0, "seed": datagen.FAST_SEED,
           "digest": digest(ds), "sizes": {"N": ds.num_subjects, "K": ds.num_eras, "J": ds.num_drugs,
                                            "nnz": ds.nnz}}
    lo, hi = np.log(0.001), np.log(10.0)
    grid = [float(np.exp(lo + (hi - lo) * i / 7.0)) for i in range(8)]
    cv = {"folds": 8, "grid": grid, "prior": "laplace", "seed": 17, "warm_start": True}
    r = rds.grid_search_cv(8, grid, B.PriorKind.laplace, 17, B.SolverConfig(), warm_start=True, threads=8)
    cv["expected"] = {"variance_grid": r["variance_grid"].tolist(),
                      "predictive_ll": [[repr(float(x)) for x in row] for row in r["predictive_ll"]],
                      "cycles": r["cycles"].tolist(), "converged": r["converged"].tolist(),
                      "valid": r["valid"].tolist(),
                      "mean_predictive_ll": [repr(float(x)) for x in r["mean_predictive_ll"]],
                      "selected_index": r["selected_index"], "selected_variance": r["selected_variance"],
                      "total_cycles": r["total_cycles"]}
    cv["reference_seconds_8_threads"] = time.time() - t0
    out["cv"] = cv
    print(f"  cv done {time.time() - t0:.0f}s", flush=True)
    t1 = time.time()
    boot = {"replicates": 16, "level": 0.95, "seed": 77, "prior": "normal", "variance": 0.1, "warm_start": True}
    b = rds.run_bootstrap(16, 0.95, 77, B.normal_prior(0.1), B.SolverConfig(), warm_start=True, threads=8)
    boot["expected"] = {k: ([repr(float(x)) for x in v] if isinstance(v, np.ndarray) else v) for k, v in b.items()}
    boot["reference_seconds_8_threads"] = time.time() - t1
    out["bootstrap"] = boot
    print(f"  bootstrap done {time.time() - t0:.0f}s", flush=True)
    beta_full = b["beta_full"]
    with ThreadPoolExecutor(4) as ex:
        reps = list(ex.map(lambda rr: rds.bootstrap_replicate(77, rr, B.normal_prior(0.1), B.SolverConfig(),
                                                                beta_full), range(4)))
    out["replicates"] = [{"r": i, **fit_dict(x)} for i, x in enumerate(reps)]
    print(f"  replicates done {time.time() - t0:.0f}s", flush=True)
    return out


def main():
    ref = po.Reference()
    large = "--large" in sys.argv
    only = [a for a in sys.argv[1:] if not a.startswith("--")]

    def want(n):
        return not only or n in only

    if want("oracle_case"):
        (OUT / "oracle_case.json").write_text(json.dumps(oracle_case(ref), indent=1))
        print("oracle_case.json")
    if want("drivers"):
        (OUT / "drivers_oracle_case.json").write_text(json.dumps(drivers_case(ref), indent=1))
        print("drivers_oracle_case.json")
    if want("engine_cases"):
        (OUT / "engine_cases.json").write_text(json.dumps(engine_cases(ref)))
        print("engine_cases.json")
    if want("small_suite"):
        (OUT / "small_suite.json").write_text(json.dumps(small_suite(ref)))
        print("small_suite.json")
    if want("fast_10k"):
        (OUT / "fast_10k.json").write_text(json.dumps(
            fast_case(ref, "10k", 10_300, 100, 2.0, B.normal_prior(0.1)), indent=1))
        print("fast_10k.json")
    if large and want("fit_1M"):
        (OUT / "fit_1M_laplace.json").write_text(json.dumps(
            fast_case(ref, "1M", 1_030_000, 1500, 3.0, B.laplace_prior(0.1)), indent=1))
        print("fit_1M_laplace.json")
    if large and want("fit_1M_zipf"):  # the skewed variant, reported beside the uniform one
        (OUT / "fit_1M_zipf_laplace.json").write_text(json.dumps(
            fast_case(ref, "1M", 1_030_000, 1500, 3.0, B.laplace_prior(0.1), zipf=True), indent=1))
        print("fit_1M_zipf_laplace.json")
    if large and want("fit_10M"):
        (OUT / "fit_10M_laplace.json").write_text(json.dumps(
            fast_case(ref, "10M", 10_300_000, 4000, 3.0, B.laplace_prior(0.1)), indent=1))
        print("fit_10M_laplace.json")
    if large and want("drivers_1M"):
        (OUT / "drivers_1M.json").write_text(json.dumps(drivers_1M(ref), indent=1))
        print("drivers_1M.json")


if __name__ == "__main__":
    main()
