"""One batched fit of the bench's many_fit block (16 bootstrap refits of the
1M set, Normal 0.1, warm start) after a warm-up: for a launch list of the
batched path (ncu --metrics gpu__time_duration.sum).

  python scripts/probe_bfit.py"""
import sys
import time

sys.path[:0] = ['.', 'oracle']
import numpy as np
from paper_1208_0945_b200 import bsccs as B, datagen

ds = datagen.config_dataset("1M")
dds = B.DeviceDataset(ds, 0)
cfg = B.SolverConfig()
prior = B.normal_prior(0.1)
full = B.fit(dds, prior, cfg)
R = 16
W = np.stack([np.bincount(B.resample(ds, 77, r + 1), minlength=ds.num_subjects) for r in range(R)]).astype(np.int32)
init = np.tile(full.beta_map, (R, 1))
for rep in range(3):
    t0 = time.perf_counter()
    fits, st = B.fit_batch(dds, [prior] * R, W, init, cfg)
    t1 = time.perf_counter()
    print(f"rep {rep}: {1e3 * (t1 - t0):.1f} ms, cycles {max(f.cycles_run for f in fits)}, "
          f"sweep {1e3 * fits[0].sweep_seconds:.1f} ms", flush=True)
