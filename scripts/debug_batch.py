"""Debug probe: batched engine vs single fits on the oracle case."""
import sys
sys.path[:0] = ['.', 'oracle', 'tests']
import numpy as np
from paper_1208_0945_b200 import bsccs as B, datagen
import pyoracle

ds = datagen.simulate(datagen.oracle_case_config())
ref = pyoracle.Reference().dataset(ds)
N = ds.num_subjects
for prior in [B.normal_prior(0.1), B.laplace_prior(0.1)]:
    t = ref.fit(prior, B.SolverConfig())
    for R in (1, 2, 8, 9):
        fits, st = B.fit_batch(ds, [prior] * R, None, None, B.SolverConfig(max_cycles=30))
        f = fits[0]
        print(prior.kind.name, R, "cycles", [x.cycles_run for x in fits], "ref", t["cycles_run"],
              "crit", f.final_criterion, "dbeta", np.abs(f.beta_map - t["beta"]).max(), "lp", f.log_posterior,
              t["log_posterior"], st[:2], flush=True)
held = np.sort(B.kfold_split(ds, 8, 17)[0])
rest = np.setdiff1d(np.arange(N), held).astype(np.int32)
w = np.zeros((1, N), np.int32)
w[0][rest] = 1
prior = B.laplace_prior(0.001)
fits, st = B.fit_batch(ds, [prior], w, None, B.SolverConfig(max_cycles=30))
t = ref.subset(rest).fit(prior, B.SolverConfig())
print("fold0", fits[0].cycles_run, t["cycles_run"], np.abs(fits[0].beta_map - t["beta"]).max(), fits[0].final_criterion)
