"""Kernel breakdown of the root-side assemble of the N-GPU compress (N=8 sizes
emulated on one GPU): torch.profiler over GpuSlabBackend.assemble."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2312_05492_b200 as P
from paper_2312_05492_b200 import distributed as D
from bench import smooth_field_gpu
world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
x = smooth_field_gpu((512 * world, 512, 512))
orig = D.GpuSlabBackend.assemble
state = {"prof": False}
def wrapped(self, *a, **k):
    if not state["prof"]:
        return orig(self, *a, **k)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as p:
        r = orig(self, *a, **k)
        torch.cuda.synchronize()
    print(p.key_averages().table(sort_by="cuda_time_total", row_limit=25))
    return r
D.GpuSlabBackend.assemble = wrapped
for _ in range(2):
    D.compress_simulated(x, world, 1e-3)
state["prof"] = True
D.compress_simulated(x, world, 1e-3)
