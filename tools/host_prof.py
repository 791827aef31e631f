import os, sys, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
import torch
import paper_2312_05492_b200 as P
from bench import smooth_field_gpu
shape=(32,32,32)
x = smooth_field_gpu(shape); dims=P.Dims(shape)
for _ in range(5):
    a = P.compress_device(P.Grid(dims, x), 1e-3); y=P.decompress_device(a)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(200):
    a = P.compress_device(P.Grid(dims, x), 1e-3)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
pr = cProfile.Profile(); pr.enable()
for _ in range(200):
    y = P.decompress_device(a)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
