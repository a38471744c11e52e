"""Where the end-to-end step goes (bench.py's e2e leg): dataset upload +
device build from pinned host arrays, fit (state create, cycles, final
rebuild), free -- wall time of each C-ABI call."""
import sys
import time
sys.path[:0] = ['.', 'oracle']
import numpy as np
import torch
from paper_1208_0945_b200 import bsccs as B, datagen

wl = sys.argv[1] if len(sys.argv) > 1 else "1M"
derive = "--derive-subjects" in sys.argv  # bench.py's e2e leg: per-pair subjects derived on the device
ds = datagen.config_dataset(wl)
prior = B.laplace_prior(0.1)


def pinned(a):
    t = torch.empty(a.size, dtype={np.int32: torch.int32, np.int64: torch.int64}[a.dtype.type], pin_memory=True)
    v = t.numpy()
    v[:] = a
    return t, v


held = [pinned(a) for a in ds.arrays()]
ds_host = B.Dataset(*[v for _, v in held])
nbytes = sum(a.nbytes for a in ds_host.arrays()) - (ds_host.subjects.nbytes if derive else 0)
for it in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d = B.DeviceDataset(ds_host, 0, upload_subjects=not derive)
    t1 = time.perf_counter()
    r = B.fit(d, prior)
    t2 = time.perf_counter()
    d.close()
    t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):7.2f} ms ({nbytes/(t1-t0)/1e9:5.1f} GB/s)  fit {1e3*(t2-t1):7.2f} ms "
          f"(device {1e3*r.device_seconds:6.2f}, sweeps {1e3*r.sweep_seconds:6.2f})  destroy {1e3*(t3-t2):6.2f} ms",
          flush=True)
dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
pin = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev.copy_(pin, non_blocking=False)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
print(f"raw pinned H2D of the same bytes: {1e3*t:.2f} ms ({nbytes/t/1e9:.1f} GB/s)", flush=True)
