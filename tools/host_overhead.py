"""Wall-clock split of one bench step: Grid() (range + sync) vs compress_device
vs decompress_device, against the GPU time of the same calls (CUDA events)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2312_05492_b200 as P
from bench import smooth_field_gpu
shape = (512, 512, 512)
x = smooth_field_gpu(shape)
dims = P.Dims(shape)
for _ in range(3):
    a = P.compress_device(P.Grid(dims, x), 1e-3); y = P.decompress_device(a)
torch.cuda.synchronize()
N = 20
tg = tc = td = 0.0
for _ in range(N):
    t0 = time.perf_counter(); g = P.Grid(dims, x); t1 = time.perf_counter()
    a = P.compress_device(g, 1e-3); t2 = time.perf_counter()
    y = P.decompress_device(a); torch.cuda.synchronize(); t3 = time.perf_counter()
    tg += t1 - t0; tc += t2 - t1; td += t3 - t2
print(f"Grid {1e3*tg/N:.3f} ms  compress_device {1e3*tc/N:.3f} ms  decompress_device {1e3*td/N:.3f} ms")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(10):
    a = P.compress_device(P.Grid(dims, x), 1e-3); y = P.decompress_device(a)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
