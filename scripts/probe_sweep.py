"""Phase timing of the persistent sweep kernel (profiling aid).

Runs run_cycle on a workload with phases of k_ccd disabled through the
debug flag hook and prints ms per sweep for several CTA counts."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1208_0945_b200 import _native, bsccs as B, datagen  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "1M"
ctas_list = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [148, 74]
ds = datagen.config_dataset(wl)
prior = B.laplace_prior(0.1)
cfg = B.SolverConfig()
lib = _native.lib()
modes = {"full": 0, "late_lexp": 64, "nospec": 16, "no_update": 2, "no_xchg": 4, "xchg_only": 3,
         "no_gh": 1, "xchg_only_late": 67, "xchg_only_nospec": 19, "nothing": 7, "nothing_nospec": 23}
if len(sys.argv) > 3:
    modes = {k: v for k, v in modes.items() if k in sys.argv[3].split(",")}
for ctas in ctas_list:
    dds = B.DeviceDataset(ds, 0, ctas)
    for name, f in modes.items():
        lib.bsccs_debug_set_sweep_flags(f)
        st = B.init_state(dds)
        solver = B.SolverState(dds, cfg)
        ts = []
        for it in range(4):
            import ctypes as C
            t0 = time.perf_counter()
            B.run_cycle(dds, st, solver, prior, cfg)
            ts.append(time.perf_counter() - t0)
        lib.bsccs_debug_set_sweep_flags(0)
        print(f"{wl} ctas={ctas:4d} {name:10s} ms/sweep={1e3 * np.median(ts[1:]):8.3f}  "
              f"us/coord={1e6 * np.median(ts[1:]) / ds.num_drugs:7.2f}", flush=True)
        st.close()
    dds.close()
