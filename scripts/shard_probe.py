"""Time the virtual-rank sharded fit (multi-GPU protocol on one device)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1208_0945_b200 import bsccs as B, datagen, sharding  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "1M"
ds = datagen.config_dataset(wl)
prior = B.laplace_prior(0.1)
single = B.fit(ds, prior)
single = B.fit(ds, prior)
print(f"{wl} single: {single.device_seconds * 1e3:.1f} ms cycles={single.cycles_run}")
for n in (2, 4, 8):
    for virtual in (False, True):
        g = sharding.LocalGroup(sharding.shard_dataset(ds, n), virtual_ranks=virtual)
        g.fit(prior)
        r = g.fit(prior)
        ok = r.cycles_run == single.cycles_run and abs(r.log_posterior - single.log_posterior) <= 1e-10 * abs(
            single.log_posterior)
        print(f"{wl} shards={n} virtual={virtual}: {r.device_seconds * 1e3:.1f} ms parity={ok}")
        g.close()
