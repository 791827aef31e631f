"""Root-side cost of the N-GPU compress (gather results -> concat -> pass-2)
at N=8 sizes, emulated on one GPU with compress_simulated (8 slabs of 512
planes of 512 x 512)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2312_05492_b200 as P
from paper_2312_05492_b200 import distributed as D
from bench import smooth_field_gpu
world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
shape = (512 * world, 512, 512)
x = smooth_field_gpu(shape)
orig = D.GpuSlabBackend.assemble
tt = {}
def timed(self, *a, **k):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = orig(self, *a, **k)
    torch.cuda.synchronize(); tt["assemble"] = time.perf_counter() - t0
    return r
D.GpuSlabBackend.assemble = timed
for _ in range(2):
    a = D.compress_simulated(x, world, 1e-3)
torch.cuda.synchronize(); t0 = time.perf_counter()
a = D.compress_simulated(x, world, 1e-3)
torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"world {world}: simulated compress {1e3*(t1-t0):.2f} ms (all slabs sequential), root assemble {1e3*tt['assemble']:.2f} ms, archive {len(a)} B")
