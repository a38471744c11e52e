"""Median fit time of a config workload (A/B of library variants via BSCCS_B200_LIB)."""
import sys
import time
sys.path[:0] = ['.', 'oracle']
import numpy as np
from paper_1208_0945_b200 import bsccs as B, datagen

wl = sys.argv[1] if len(sys.argv) > 1 else "1M"
zipf = len(sys.argv) > 2 and sys.argv[2] == "zipf"
ds = datagen.config_dataset(wl, zipf)
dds = B.DeviceDataset(ds, 0)
prior = B.laplace_prior(0.1)
ts = []
for i in range(5):
    r = B.fit(dds, prior)
    ts.append(r.device_seconds)
print(f"{wl}{' zipf' if zipf else ''}: fit {1e3*np.median(ts[1:]):.2f} ms, cycles {r.cycles_run}, "
      f"sweep {1e3*r.sweep_seconds/r.cycles_run:.3f} ms/cycle", flush=True)
