"""Host-side segments of a 512^3 compress_device step (Grid(), the libcszi
call that launches the graph, the ctl read-back including the GPU wait):
what the GPU waits on between steps."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import torch, ctypes
import paper_2312_05492_b200 as P
from paper_2312_05492_b200 import pipeline as PL, _lib
from bench import smooth_field_gpu
shape=(512,512,512)
x = smooth_field_gpu(shape); dims = P.Dims(shape)
for _ in range(5): P.compress_device(P.Grid(dims, x), 1e-3)
torch.cuda.synchronize()
lib = _lib.load()
# wrap the ctypes entry to time host-side segments
T = {}
def mark(k, t0):
    T[k] = T.get(k, 0.0) + time.perf_counter() - t0
orig_compress = lib.cszi_compress
orig_fetch = _lib.DeviceCtl.fetch
class Wrap:
    pass
def wrapped(*a):
    t0 = time.perf_counter(); r = orig_compress(*a); mark("cszi_compress (graph launch)", t0); return r
lib.cszi_compress = wrapped
def fetch(self):
    t0 = time.perf_counter(); r = orig_fetch(self); mark("fetch (incl. GPU wait)", t0); return r
_lib.DeviceCtl.fetch = fetch
N = 100
t_all = time.perf_counter()
for _ in range(N):
    t0 = time.perf_counter(); g = P.Grid(dims, x); mark("Grid()", t0)
    t0 = time.perf_counter(); a = P.compress_device(g, 1e-3); mark("compress_device total", t0)
torch.cuda.synchronize()
tot = time.perf_counter() - t_all
for k, v in T.items(): print(f"{k:32s} {1e6*v/N:8.1f} us")
print(f"{'per step wall':32s} {1e6*tot/N:8.1f} us")
