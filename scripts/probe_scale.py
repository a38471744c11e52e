"""What one rank of an N-GPU sharded config-3 fit does on its own GPU: rank
0's patient shard (sharding.shard_dataset(ds, N, only=0)) fitted as a
standalone dataset on all 148 SMs.  Its per-cycle sweep time is the rank's
data work per cycle without the cross-GPU hop of the hierarchical exchange;
the per-coordinate period bounds what the sharded fit can gain from N."""
import sys
sys.path[:0] = ['.', 'oracle']
import numpy as np
from paper_1208_0945_b200 import _native, bsccs as B, datagen, sharding

wl = sys.argv[1] if len(sys.argv) > 1 else "10M"
ds = datagen.config_dataset(wl)
prior = B.laplace_prior(0.1)
KN = {1: 'k_ccd', 2: 'k_rcd', 3: 'k_rcd+k_ccd'}
for n in (1, 2, 4, 8):
    part = ds if n == 1 else sharding.shard_dataset(ds, n, only=0)[0].dataset
    dds = B.DeviceDataset(part, 0)
    rs = [B.fit(dds, prior) for _ in range(4)]
    sw = [r.sweep_seconds / r.cycles_run for r in rs[1:]]
    per = 1e6 * np.median(sw) / ds.num_drugs
    print(f"{wl} rank-0 shard of {n}: {dds.info()['nnz']} pairs, sweep {1e3 * np.median(sw):.3f} ms/cycle "
          f"({per:.2f} us per coordinate), fit {1e3 * np.median([r.device_seconds for r in rs[1:]]):.1f} ms "
          f"({rs[-1].cycles_run} cycles), kernel {KN.get(_native.lib().bsccs_debug_last_sweep(), 'k_ccd')}",
          flush=True)
    dds.close()
