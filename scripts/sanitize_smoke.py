"""Small runs of every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck): dataset build, subset, single fit (sparse + dense
route), tier-1 ops, batched fits, CV and bootstrap drivers, loader."""
import sys
import tempfile
sys.path[:0] = ['.', 'oracle']
import numpy as np
import ctypes as C
from paper_1208_0945_b200 import _native, bootstrap as BT, bsccs as B, cross_validation as CV, datagen, sharding

set_sweep = _native.lib().bsccs_debug_set_sweep
ds = datagen.fast_sccs(3000, 20, 3.0)
dds = ds.on_device()
r = B.fit(dds, B.laplace_prior(0.1))  # k_rcd, subject tile
dnull = B.DeviceDataset(ds, 0, upload_subjects=False)  # per-pair subjects derived on the device (chunked rows)
B.fit(dnull, B.laplace_prior(0.1))
B.fit(dnull, B.laplace_prior(0.1), init_beta=np.full(ds.num_drugs, 0.01))  # warm start: full dense prologue
dnull.close()
set_sweep(0, 0.05)
B.fit(dds, B.normal_prior(2.0))  # k_rcd handing cycles over to k_ccd (lowered range bound)
set_sweep(0, 0.0)
big = datagen.fast_sccs(50000, 1500, 3.0)
bdd = B.DeviceDataset(big, 0, 2)  # k_rcd without the subject tile (touched-subject bitmaps), 2 CTAs
B.fit(bdd, B.laplace_prior(0.1), B.SolverConfig(max_cycles=2))
bdd.close()
few = B.DeviceDataset(ds, 0, 2)  # two CTAs: k_ccd's slices beyond the register tiles take the streamed path
set_sweep(1, 0.0)
B.fit(few, B.laplace_prior(0.1))
set_sweep(0, 0.0)
stf = B.init_state(few)
B.fused_grad_hess(few, stf, 1)
B.sparse_delta_update(few, stf, 1, 0.05)
few.close()
B.fit(dds, B.normal_prior(0.1), B.SolverConfig(path=B.UpdatePath.dense))
st = B.init_state(dds)
B.fused_grad_hess(dds, st, 3)
B.sparse_delta_update(dds, st, 3, 0.1)
B.log_likelihood(dds, st)
sub = dds.subset(B.resample(ds, 7, 1))
B.fit(sub, B.normal_prior(0.1))
w = np.stack([np.bincount(B.resample(ds, 5, k + 1), minlength=ds.num_subjects) for k in range(3)]).astype(np.int32)
B.fit_batch(dds, [B.normal_prior(0.1)] * 3, w)
CV.grid_search_cv(ds, CV.CVConfig(folds=3, variance_grid=[0.1, 1.0], engine="batched"))
BT.run_bootstrap(ds, BT.BootstrapConfig(replicates=3, prior=B.normal_prior(0.1), engine="batched"))
with tempfile.NamedTemporaryFile("w", suffix=".tsv", delete=False) as f:
    f.write("p1\t5\t0\ta\np1\t5\t1\tb a\np2\t7\t1\tb\n")
B.read_long_format(f.name)
for virtual in (False, True):  # multi-shard launches: local and virtual-rank exchange
    grp = sharding.LocalGroup(sharding.shard_dataset(ds, 3), virtual_ranks=virtual)
    grp.fit(B.laplace_prior(0.1))
    grp.close()
vals = np.random.default_rng(1).uniform(0, 1e6, 1500)
out, stc = C.c_double(), C.c_int32()
_native.lib().bsccs_debug_exchange_sum(0, vals.ctypes.data_as(C.c_void_p), len(vals), C.byref(out), C.byref(stc))
print("sanitize smoke done", r.cycles_run)
