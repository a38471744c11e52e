"""Fit time against the CTA count of the dataset split (148 / 128 / 112 / 96 / 74
of the 148 SMs): python scripts/probe_ctas.py 1M 10M."""
import sys
sys.path[:0] = ['.', 'oracle']
import numpy as np
from paper_1208_0945_b200 import bsccs as B, datagen
for wl in sys.argv[1:]:
    ds = datagen.config_dataset(wl)
    for ctas in (148, 128, 112, 96, 74):
        d = B.DeviceDataset(ds, 0, ctas)
        ts = []
        for i in range(3):
            r = B.fit(d, B.laplace_prior(0.1))
            ts.append(r.device_seconds)
        print(f"{wl} ctas={ctas}: fit {1e3*np.median(ts[1:]):.2f} ms cycles {r.cycles_run} sweep {1e3*r.sweep_seconds/r.cycles_run:.3f} ms/cycle", flush=True)
        d.close()
