"""Where the end-to-end step goes: dataset upload + device build, fit, free."""
import sys
import time
sys.path[:0] = ['.', 'oracle']
import numpy as np
import torch
from paper_1208_0945_b200 import bsccs as B, datagen

ds = datagen.config_dataset("1M")
prior = B.laplace_prior(0.1)
nbytes = sum(a.nbytes for a in ds.arrays())
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d = B.DeviceDataset(ds, 0)
    t1 = time.perf_counter()
    r = B.fit(d, prior)
    t2 = time.perf_counter()
    d.close()
    t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):7.2f} ms ({nbytes/(t1-t0)/1e9:5.1f} GB/s)  fit {1e3*(t2-t1):7.2f} ms  "
          f"destroy {1e3*(t3-t2):6.2f} ms", flush=True)
# raw copy rates for the same bytes
a = np.concatenate([x.view(np.uint8) for x in ds.arrays()])
dev = torch.empty(a.size, dtype=torch.uint8, device="cuda")
pin = torch.empty(a.size, dtype=torch.uint8, pin_memory=True)
pin.numpy()[:] = a
for name, src in [("pageable", torch.from_numpy(a)), ("pinned", pin)]:
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.copy_(src, non_blocking=False)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
    print(f"H2D {name}: {a.size/t/1e9:.1f} GB/s", flush=True)
import os
print("host cpus", os.cpu_count(), len(os.sched_getaffinity(0)))
