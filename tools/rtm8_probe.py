"""RTM x 8 batch at N=1: compress_sharded_batch vs the plain per-snapshot
compress_device loop, timed repeatedly (CUDA events) to separate noise from a
path difference.  Usage: rtm8_probe.py"""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2312_05492_b200 as P
from bench import RTM_SHAPE, events_ms, smooth_field_gpu
from paper_2312_05492_b200.distributed import SimComm, compress_sharded_batch

shape = RTM_SHAPE
xs = [smooth_field_gpu(shape, phase=2 * math.pi * k / 8, zrange=(0, shape[0])) for k in range(8)]
comm = SimComm(1)
total = 8 * 4 * math.prod(shape)
for rep in range(3):
    b_ms, _ = events_ms(lambda: compress_sharded_batch(xs, shape, 0, shape[0], 1e-3, comm=comm), 10, 1)
    s_ms, _ = events_ms(lambda: [P.compress_device(P.Grid(P.Dims(shape), x), 1e-3) for x in xs], 10, 1)
    t0 = time.perf_counter()
    for _ in range(10):
        compress_sharded_batch(xs, shape, 0, shape[0], 1e-3, comm=comm)
    torch.cuda.synchronize()
    w = (time.perf_counter() - t0) / 10 * 1e3
    print(f"rep {rep}: batch {b_ms:.3f} ms ({total / b_ms / 1e6:.1f} GB/s)  single loop {s_ms:.3f} ms"
          f" ({total / s_ms / 1e6:.1f} GB/s)  batch wall {w:.3f} ms", flush=True)
