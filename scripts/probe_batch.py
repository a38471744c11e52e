"""One batched fit (16 bootstrap refits of the 1M set) for ncu captures."""
import sys
sys.path[:0] = ['.', 'oracle']
import numpy as np
from paper_1208_0945_b200 import bsccs as B, datagen

ds = datagen.config_dataset(sys.argv[1] if len(sys.argv) > 1 else "1M")
dds = ds.on_device()
N = ds.num_subjects
prior = B.normal_prior(0.1)
full = B.fit(dds, prior)
W = np.stack([np.bincount(B.resample(ds, 77, r + 1), minlength=N) for r in range(16)]).astype(np.int32)
fits, st = B.fit_batch(dds, [prior] * 16, W, np.tile(full.beta_map, (16, 1)))
print("cycles", [f.cycles_run for f in fits], "sweep_s", fits[0].sweep_seconds)
