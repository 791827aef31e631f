"""Sharded decompress on one GPU (SimComm): all `world` slabs of one 512^3
archive, every slab decoding the whole Huffman stream (decompress_slab) vs
the chunk-range split (decompress_slabs_split).  Prints wall time per full
decode of all slabs; the split's time is the sum of all ranks' work, so
world x (per-rank time) bounds a real N-GPU run from above.
Usage: split_probe.py [world] [shape]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2312_05492_b200 as P
from paper_2312_05492_b200 import distributed as D
from bench import smooth_field_gpu


def timed(fn, k=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k * 1e3


world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
shape = tuple(int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "512,512,512").split(","))
x = smooth_field_gpu(shape)
arch = P.compress_device(P.Grid(P.Dims(shape), x), 1e-3)
whole = P.decompress_device(arch).tensor
a = timed(lambda: D.decompress_simulated(arch, world))
b = timed(lambda: D.decompress_simulated(arch, world, split=True))
same = torch.equal(D.decompress_simulated(arch, world, split=True), whole)
print(f"{shape} world {world}: per-slab whole-stream decode {a:.2f} ms, chunk-range split "
      f"{b:.2f} ms (all slabs, one GPU), identical: {same}")
