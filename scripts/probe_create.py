"""Time of the end-to-end pieces at a config workload: dataset create from
pinned host arrays (H2D + device build), fit on it, destroy.

  python scripts/probe_create.py [10M|1M] [reps]"""
import sys
import time

sys.path[:0] = ['.', 'oracle']
import numpy as np
import torch
from paper_1208_0945_b200 import bsccs as B, datagen

wl = sys.argv[1] if len(sys.argv) > 1 else "10M"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ds = datagen.config_dataset(wl)
held = []
for a in ds.arrays():
    t = torch.empty(a.size, dtype={np.int32: torch.int32, np.int64: torch.int64}[a.dtype.type], pin_memory=True)
    t.numpy()[:] = a
    held.append(t)
host = B.Dataset(*[t.numpy() for t in held])
prior = B.laplace_prior(0.1)
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d = B.DeviceDataset(host, device=0, upload_subjects=False)
    t1 = time.perf_counter()
    res = B.fit(d, prior)
    t2 = time.perf_counter()
    d.close()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"{wl} rep {r}: create {1e3 * (t1 - t0):.1f} ms  fit {1e3 * (t2 - t1):.1f} ms (device {1e3 * res.device_seconds:.1f})"
          f"  destroy {1e3 * (t3 - t2):.1f} ms", flush=True)
