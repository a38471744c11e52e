"""Cost of the multi-rank exchange protocol on one GPU: the config-2 fit as
n patient shards bound into one launch, either as a local group (one
exchange area) or as virtual ranks (every CTA adds into n exchange areas, as
n GPUs would).  Compare with the unsharded fit."""
import sys
import time
sys.path[:0] = ['.', 'oracle']
import numpy as np
from paper_1208_0945_b200 import bsccs as B, datagen, sharding

wl = sys.argv[1] if len(sys.argv) > 1 else "1M"
ds = datagen.config_dataset(wl)
prior = B.laplace_prior(0.1)
dds = B.DeviceDataset(ds, 0)
ts = [B.fit(dds, prior).device_seconds for _ in range(4)]
print(f"{wl} unsharded: {1e3 * np.median(ts[1:]):.2f} ms", flush=True)
dds.close()
for n in (2, 4, 8):
    shards = sharding.shard_dataset(ds, n)
    for virtual in (False, True):
        g = sharding.LocalGroup(shards, virtual_ranks=virtual)
        ts = []
        for _ in range(4):
            t0 = time.perf_counter()
            r = g.fit(prior)
            ts.append(time.perf_counter() - t0)
        print(f"{wl} {n} shards {'virtual ranks' if virtual else 'local group  '}: "
              f"{1e3 * np.median(ts[1:]):.2f} ms (cycles {r.cycles_run})", flush=True)
        g.close()
