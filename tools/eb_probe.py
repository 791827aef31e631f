"""Compress / decompress step time (CUDA events, device-resident) of the
512^3 bench field at several bounds, repeated, for A/B of library builds
(CSZI_LIB=...).  Usage: eb_probe.py [eb ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2312_05492_b200 as P
from bench import events_ms, smooth_field_gpu

shape = (512, 512, 512)
x = smooth_field_gpu(shape)
dims = P.Dims(shape)
ebs = [float(v) for v in sys.argv[1:]] or [1e-3, 1e-4]
for rep in range(2):
    for eb in ebs:
        for _ in range(3):
            a = P.compress_device(P.Grid(dims, x), eb)
            P.decompress_device(a)
        c_ms, a = events_ms(lambda: P.compress_device(P.Grid(dims, x), eb), 25, 1)
        d_ms, _ = events_ms(lambda: P.decompress_device(a), 25, 1)
        print(f"rep {rep} eb {eb:g}: compress {1e3 * c_ms:7.1f} us  decompress {1e3 * d_ms:7.1f} us",
              flush=True)
