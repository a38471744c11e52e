"""Per-CTA phase timeline of the batched kernel k_bccd (globaltimer stamps):
16 bootstrap refits of a config dataset."""
import ctypes as C
import sys
sys.path[:0] = ['.', 'oracle']
import numpy as np
from paper_1208_0945_b200 import _native, bsccs as B, datagen

wl = sys.argv[1] if len(sys.argv) > 1 else "1M"
NT = 300
ds = datagen.config_dataset(wl)
dds = ds.on_device()
N, ctas = ds.num_subjects, dds.ctas
prior = B.normal_prior(0.1)
full = B.fit(dds, prior)
W = np.stack([np.bincount(B.resample(ds, 77, r + 1), minlength=N) for r in range(16)]).astype(np.int32)
lib = _native.lib()
lib.bsccs_debug_trace(NT, ctas, None, 0)
cfg = B.SolverConfig(max_cycles=1)
fits, st = B.fit_batch(dds, [prior] * 16, W, np.tile(full.beta_map, (16, 1)), cfg)
buf = np.zeros(NT * ctas * 6, dtype=np.uint64)
lib.bsccs_debug_trace(NT, ctas, buf.ctypes.data_as(C.c_void_p), buf.size)
lib.bsccs_debug_trace(0, ctas, None, 0)
t = buf.reshape(NT, ctas, 6).astype(np.int64)[20:NT - 1]
per = np.diff(t[:, 0, 0])
print(f"{wl}: per-coordinate period median {np.median(per):.0f} ns (sweep {fits[0].sweep_seconds*1e3:.2f} ms)")
names = ["top->gh done", "gh done->reduced", "reduced->step seen", "step->update done", "update->end"]
for i, nm in enumerate(names):
    d = t[:, :, i + 1] - t[:, :, i]
    print(f"  {nm:20s} median {np.median(d):7.0f}  max-over-CTAs median {np.median(d.max(axis=1)):7.0f} ns")
print(f"  spread of top across CTAs: median {np.median(t[:, :, 0].max(1) - t[:, :, 0].min(1)):.0f} ns")
print(f"  last reduced -> first step seen: median {np.median(t[:, :, 3].min(1) - t[:, :, 2].max(1)):.0f} ns")
