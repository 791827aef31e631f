"""Per-call wall time of compress_device / decompress_device on a tiny grid
(device work ~negligible, so the wall time is the host path + one sync),
with and without the ctl read-back.  Usage: host_wall.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2312_05492_b200 as P
from bench import smooth_field_gpu

shape = (32, 32, 32)
x = smooth_field_gpu(shape)
dims = P.Dims(shape)
for _ in range(20):
    a = P.compress_device(P.Grid(dims, x), 1e-3)
    P.decompress_device(a)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    for _ in range(500):
        a = P.compress_device(P.Grid(dims, x), 1e-3)
    t1 = time.perf_counter()
    for _ in range(500):
        P.decompress_device(a)
    t2 = time.perf_counter()
    print(f"compress {(t1 - t0) / 500 * 1e6:6.1f} us/call  decompress {(t2 - t1) / 500 * 1e6:6.1f} us/call",
          flush=True)
