"""CPU time of the pieces of one compress_device / decompress_device call
(no syncs inside the measured pieces): where the GPU waits on the host."""
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2312_05492_b200 as P
from paper_2312_05492_b200 import _lib
from bench import smooth_field_gpu
x = smooth_field_gpu((512, 512, 512))
dims = P.Dims(x.shape)
lib = _lib.load()
acc = {}
def wrap(name):
    f = getattr(lib, name)
    def g(*a):
        t0 = time.perf_counter(); r = f(*a); acc[name] = acc.get(name, 0) + time.perf_counter() - t0
        return r
    g.argtypes = f.argtypes
    setattr(lib, name, g)
for nm in ("cszi_compress", "cszi_decompress", "cszi_range", "cszi_ctl_init"):
    wrap(nm)
for _ in range(3):
    a = P.compress_device(P.Grid(dims, x), 1e-3); P.decompress_device(a)
torch.cuda.synchronize(); acc.clear()
N = 20
tg = tc = td = 0
for _ in range(N):
    t0 = time.perf_counter(); g = P.Grid(dims, x); t1 = time.perf_counter()
    a = P.compress_device(g, 1e-3); t2 = time.perf_counter()
    y = P.decompress_device(a); torch.cuda.synchronize(); t3 = time.perf_counter()
    tg += t1 - t0; tc += t2 - t1; td += t3 - t2
print(f"wall: Grid {1e6*tg/N:.0f} us, compress_device {1e6*tc/N:.0f} us, decompress_device {1e6*td/N:.0f} us")
for k, v in acc.items():
    print(f"  CPU in {k}: {1e6*v/N:.1f} us per call")
