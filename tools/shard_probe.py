"""Stage times of the sharded batch compress (bench rtm8 leg, one process:
SimComm over `world` simulated slabs): wall time per stage with a device
sync after each, to split host overhead from kernel time.
Usage: shard_probe.py [world]"""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2312_05492_b200 import distributed as D
from bench import smooth_field_gpu

world = int(sys.argv[1]) if len(sys.argv) > 1 else 1
shape = (449, 449, 235)
xs = [smooth_field_gpu(shape, phase=2 * math.pi * k / 8) for k in range(8)]
for _ in range(3):
    D.compress_simulated_batch(xs, world, 1e-3)
torch.cuda.synchronize()
# instrument the backend: wall time per method
times = {}
B = D.GpuSlabBackend
for name in ("range_keys", "set_range", "samples", "tune", "predict", "codebook", "piece_bits",
             "encode", "anchors", "pieces", "assemble"):
    f = getattr(B, name)

    def wrap(self, *a, _f=f, _n=name, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = _f(self, *a, **k)
        torch.cuda.synchronize()
        times[_n] = times.get(_n, 0.0) + time.perf_counter() - t0
        return r

    setattr(B, name, wrap)
reps = 5
t0 = time.perf_counter()
for _ in range(reps):
    D.compress_simulated_batch(xs, world, 1e-3)
torch.cuda.synchronize()
tot = (time.perf_counter() - t0) / reps
print(f"world {world}: {1e3 * tot:.2f} ms per batch of 8 (instrumented)")
for k, v in sorted(times.items(), key=lambda kv: -kv[1]):
    print(f"  {k:12s} {1e3 * v / reps:8.3f} ms")
print(f"  (other)      {1e3 * (tot - sum(times.values()) / reps):8.3f} ms")
