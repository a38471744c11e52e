"""Per-CTA timeline of the persistent sweep kernel (globaltimer stamps)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import os  # noqa: E402
if "BSCCS_B200_LIB" not in os.environ:  # the resident-beta sweep stamps only in the RCD_TRACE=1 variant
    # (build_native(variant={"RCD_TRACE": 1}) makes it; set before the package loads its library)
    os.environ["BSCCS_B200_LIB"] = str(Path(__file__).resolve().parents[1] / "paper_1208_0945_b200" / "_lib" /
                                       "libbsccs_b200_rcdtrace1.so")
from paper_1208_0945_b200 import _native, bsccs as B, datagen  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "1M"
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
zipf = "zipf" in sys.argv[3:]
per_coord = "per-coord" in sys.argv[3:]
NT = 300
ds = datagen.config_dataset(wl, zipf)
dds = B.DeviceDataset(ds, 0)
ctas = dds.ctas
lib = _native.lib()
prior, cfg = B.laplace_prior(0.1), B.SolverConfig()
st = B.init_state(dds)
solver = B.SolverState(dds, cfg)
B.run_cycle(dds, st, solver, prior, cfg)  # warm
lib.bsccs_debug_set_sweep_flags(flags)
lib.bsccs_debug_trace(NT, ctas, None, 0)
B.run_cycle(dds, st, solver, prior, cfg)
KT = 16  # stamps per CTA and coordinate (ccd_kernels.cu kTr)
buf = np.zeros(NT * ctas * KT, dtype=np.uint64)
lib.bsccs_debug_trace(NT, ctas, buf.ctypes.data_as(C.c_void_p), buf.size)
lib.bsccs_debug_trace(0, ctas, None, 0)
lib.bsccs_debug_set_sweep_flags(0)
t = buf.reshape(NT, ctas, KT).astype(np.int64)
if per_coord:  # first coordinates in visit order (fixed order: j = 0, 1, ...): the head columns of a skewed set
    full = t[:NT - 1, 0, 0]
    nnz = np.diff(ds.col_ptr)
    per = np.diff(t[:NT, 0, 0])
    for i in range(0, 40):
        print(f"  coord {i:3d} nnz {nnz[i]:8d}  period {per[i]:8d} ns")
    print(f"  coords 0-39 total {per[:40].sum() / 1e3:.1f} us, coords 40-298 median {np.median(per[40:]):.0f} ns")
t = t[20:NT - 1]  # skip the start
t0 = t[:, :, 0]
pub = t[:, :, 1]
got = t[:, :, 2]
done = t[:, :, 3]
coord = np.diff(t[:, 0, 0])
print(f"{wl} flags={flags} ctas={ctas}: per-coordinate period (CTA0 loop top) median {np.median(coord):.0f} ns")
gh = pub - t0
print(f"  gh+reduce (top->publish) per CTA: median {np.median(gh):.0f}  p90 {np.percentile(gh, 90):.0f}  "
      f"max-over-CTAs median {np.median(gh.max(1)):.0f} ns")
last_pub = pub.max(1)
first_top = t0.min(1)
print(f"  spread of loop-top across CTAs: median {np.median(t0.max(1) - t0.min(1)):.0f} ns")
print(f"  last publish -> gather done: median over coords of (median over CTAs) "
      f"{np.median(np.median(got, 1) - last_pub):.0f}  (max CTA) {np.median(got.max(1) - last_pub):.0f} ns")
print(f"  first top -> last publish: {np.median(last_pub - first_top):.0f} ns")
upd = done - got
print(f"  gather done -> update done: median {np.median(upd):.0f}  max-over-CTAs median {np.median(upd.max(1)):.0f}")
nxt = t[1:, :, 0] - done[:-1]
print(f"  update done -> next top (finalize): median {np.median(nxt):.0f}")
iss = t[:, :, 4]
poll = t[:, :, 5]
print(f"  publish -> prefetch issued: median {np.median(iss - pub):.0f}")
print(f"  last publish -> poll done (lane 0, warp 0): median {np.median(np.median(poll, 1) - last_pub):.0f}  "
      f"first CTA {np.median(poll.min(1) - last_pub):.0f}  last CTA {np.median(poll.max(1) - last_pub):.0f}")
print(f"  poll done -> gather done: median {np.median(got - poll):.0f}")
print(f"  own publish -> poll done: median {np.median(poll - pub):.0f}")
slow = np.argmax(pub, axis=1)
vals, cnt = np.unique(slow, return_counts=True)
order = np.argsort(-cnt)[:8]
print("  most frequent last publisher CTAs:", [(int(vals[i]), int(cnt[i])) for i in order])
dat = t[:, :, 6]
stp = t[:, :, 7]
print(f"  poll done -> step computed (warp 0): median {np.median(stp - poll):.0f}")
print(f"  poll done -> data warp 1 at barrier: median {np.median(dat - poll):.0f}  "
      f"(publish -> data warp at barrier {np.median(dat - pub):.0f})")
print(f"  data warp at barrier -> released: median {np.median(got - dat):.0f}")

if t[:, :, 12].any():  # resident-beta sweep: data warp 1 phase stamps (k_rcd)
    def ph(a, b, label):
        d = t[:, :, b] - t[:, :, a]
        ok = (t[:, :, a] > 0) & (t[:, :, b] > 0)
        if ok.any():
            dm = np.where(ok, d, 0)
            print(f"  [warp 1] {label}: median {np.median(d[ok]):.0f}  max-over-CTAs median {np.median(dm.max(1)):.0f} ns")
    ph(0, 11, "top -> repaired")
    ph(11, 12, "repaired -> gh staged (barrier)")
    ph(12, 13, "gh staged -> run terms done")
    ph(13, 1, "run terms -> reduced (tid 0)")
    ph(1, 14, "publish -> window issued")
    ph(14, 15, "wait records of idx+1")
    ph(15, 6, "speculate idx+1")
    ph(2, 8, "step barrier -> update diffs")
    ph(8, 9, "diffs -> staged (barrier)")
    ph(9, 10, "staged -> heads done")
    ph(10, 3, "heads done -> end barrier")
