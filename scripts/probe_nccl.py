"""Latency of a 16-byte NCCL all-reduce issued per coordinate from the host
(world size 1: the floor of its per-call cost -- launch, stream ordering --
before any NVLink transfer), against the in-kernel exact exchange
(scripts/xbench5.cu: ~1.07 us for 148 CTAs).

  python scripts/probe_nccl.py"""
import os
import time

import torch
import torch.distributed as dist

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
t = torch.zeros(2, dtype=torch.float64, device="cuda")
for _ in range(100):
    dist.all_reduce(t)
torch.cuda.synchronize()
n = 2000
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(n):
    dist.all_reduce(t)
e.record()
torch.cuda.synchronize()
print(f"ncclAllReduce 16 B, back to back on the stream: {s.elapsed_time(e) * 1e3 / n:.2f} us per call")
# a CCD coordinate needs the result on the device before the step and the
# step before the next coordinate: with host-driven collectives that is a
# kernel + all-reduce + kernel per coordinate, each waiting for the last
k = torch.zeros(1, device="cuda")
t0 = time.perf_counter()
for _ in range(n):
    k.add_(1.0)       # the coordinate's grad/hess kernel (stand-in)
    dist.all_reduce(t)
    k.mul_(1.0)       # the step + update kernel (stand-in)
torch.cuda.synchronize()
print(f"kernel + ncclAllReduce + kernel per coordinate: {(time.perf_counter() - t0) * 1e6 / n:.2f} us")
dist.destroy_process_group()
