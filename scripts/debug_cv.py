"""Debug probe: batched CV chain vs subset CV on the oracle case."""
import sys
sys.path[:0] = ['.', 'oracle', 'tests']
import numpy as np
from paper_1208_0945_b200 import bsccs as B, datagen, cross_validation as CV
import pyoracle

ds = datagen.simulate(datagen.oracle_case_config())
N = ds.num_subjects
lo, hi = np.log(0.001), np.log(10.0)
grid = [float(np.exp(lo + (hi - lo) * i / 7.0)) for i in range(8)]
for eng in ("subset", "batched"):
    r = CV.grid_search_cv(ds, CV.CVConfig(folds=8, variance_grid=grid, seed=17, engine=eng))
    print(eng, r.selected_index, r.total_cycles)
    print(np.array([[c.cycles for c in row] for row in r.cells]))
    print(np.array([[c.predictive_ll for c in row] for row in r.cells])[:3, :3])
folds = B.kfold_split(ds, 8, 17)
W = np.zeros((8, N), np.int32)
for f in range(8):
    W[f] = 1
    W[f][folds[f]] = 0
carried = None
for g in range(3):
    fits, st = B.fit_batch(ds, [B.laplace_prior(grid[g])] * 8, W, carried, B.SolverConfig(max_cycles=40))
    print("g", g, [x.cycles_run for x in fits], st)
    carried = np.stack([x.beta_map for x in fits])
