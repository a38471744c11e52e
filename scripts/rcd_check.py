"""Resident-beta sweep (k_rcd) against the reference goldens and the classic
sweep (k_ccd, BSCCS_SWEEP=classic): fit time, cycles, parity.

  python scripts/rcd_check.py [workloads...]      (default: oracle 10k 1M 10M)
"""
import json
import os
import sys
import time
from pathlib import Path

sys.path[:0] = ['.', 'oracle']
import numpy as np
from paper_1208_0945_b200 import bsccs as B, datagen

GOLD = {"1M": "fit_1M_laplace.json", "10M": "fit_10M_laplace.json"}
mode = os.environ.get("BSCCS_SWEEP", "rcd")
for wl in (sys.argv[1:] or ["oracle", "10k", "1M", "10M"]):
    zipf = wl.endswith("z")
    name = wl.rstrip("z")
    t0 = time.time()
    ds = datagen.config_dataset(name, zipf)
    dds = B.DeviceDataset(ds, 0)
    prior = B.normal_prior(0.1) if name == "oracle" else B.laplace_prior(0.1)
    ts = []
    for i in range(4):
        r = B.fit(dds, prior)
        ts.append(r.device_seconds)
    line = f"[{mode}] {wl}: fit {1e3 * np.median(ts[1:]):.2f} ms, cycles {r.cycles_run}, " \
           f"sweep {1e3 * r.sweep_seconds / r.cycles_run:.3f} ms/cycle, lp {r.log_posterior:.17g}"
    g = None
    if name == "oracle":
        g = json.loads(Path("tests/golden/oracle_case.json").read_text())["fits"][0]
    elif name in GOLD and not zipf:
        g = json.loads(Path("tests/golden", GOLD[name]).read_text())
    if g is not None:
        ref = np.array([float(x) for x in g["beta"]])
        nz = ref != 0
        rel = np.abs(r.beta_map[nz] - ref[nz]) / np.abs(ref[nz])
        za = np.abs(r.beta_map[~nz]).max(initial=0.0)
        lp = float(g["log_posterior"])
        line += f" | beta rel {rel.max(initial=0):.3g} zeros {za:.3g} lp rel {abs(r.log_posterior - lp) / abs(lp):.3g}" \
                f" cycles ref {g['cycles_run']}"
    print(line, flush=True)
    dds.close()
