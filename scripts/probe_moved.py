"""How many coordinates of a fit move (delta != 0) against those visited, and
the fit's log posterior: python scripts/probe_moved.py 1M|10M."""
import sys
sys.path[:0] = ['.', 'oracle']
from paper_1208_0945_b200 import bsccs as B, datagen
ds = datagen.config_dataset(sys.argv[1])
dds = B.DeviceDataset(ds, 0)
r = B.fit(dds, B.laplace_prior(0.1))
print(sys.argv[1], "visited", r.coordinates_visited, "moved", r.coordinates_moved, "lp", repr(r.log_posterior))
