"""One CCD cycle of a config dataset (for ncu captures of k_ccd)."""
import sys
sys.path[:0] = ['.', 'oracle']
from paper_1208_0945_b200 import bsccs as B, datagen

ds = datagen.config_dataset(sys.argv[1] if len(sys.argv) > 1 else "1M")
dds = B.DeviceDataset(ds, 0)
prior, cfg = B.laplace_prior(0.1), B.SolverConfig()
st = B.init_state(dds)
solver = B.SolverState(dds, cfg)
for _ in range(3):
    B.run_cycle(dds, st, solver, prior, cfg)
print("done")
