"""One warm compress + decompress of the 512^3 bench field (for ncu launch lists)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2312_05492_b200 as P
from bench import smooth_field_gpu
shape = tuple(int(s) for s in (sys.argv[1] if len(sys.argv) > 1 else "512,512,512").split(","))
x = smooth_field_gpu(shape)
dims = P.Dims(shape)
for _ in range(2):
    a = P.compress_device(P.Grid(dims, x), 1e-3)
    y = P.decompress_device(a)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("timed")
a = P.compress_device(P.Grid(dims, x), 1e-3)
y = P.decompress_device(a)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("ok", len(a))
