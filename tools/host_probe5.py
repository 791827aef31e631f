"""Host timeline of one bench step: where the GPU waits for Python.
Times (us, averaged) from compress_device entry to the cszi_compress call,
inside it, in ctl.fetch (sync), and the Grid() pieces."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2312_05492_b200 as P
from paper_2312_05492_b200 import _lib, pipeline
from bench import smooth_field_gpu
x = smooth_field_gpu((512, 512, 512))
dims = P.Dims(x.shape)
lib = _lib.load()
T = {}
def rec(k, v):
    T[k] = T.get(k, 0.0) + v
marks = {}
f_comp = lib.cszi_compress
def comp(*a):
    t0 = time.perf_counter(); marks["c0"] = t0
    r = f_comp(*a)
    marks["c1"] = time.perf_counter(); return r
comp.argtypes = f_comp.argtypes
lib.cszi_compress = comp
f_range = lib.cszi_scan_field
def rng(*a):
    marks["r0"] = time.perf_counter(); r = f_range(*a); marks["r1"] = time.perf_counter(); return r
rng.argtypes = f_range.argtypes
lib.cszi_scan_field = rng
orig_fetch = _lib.DeviceCtl.fetch
def fetch(self):
    t0 = time.perf_counter(); r = orig_fetch(self); rec("fetch(sync) total", time.perf_counter() - t0); return r
_lib.DeviceCtl.fetch = fetch
for _ in range(3):
    P.compress_device(P.Grid(dims, x), 1e-3)
torch.cuda.synchronize(); T.clear()
N = 30
for _ in range(N):
    t0 = time.perf_counter()
    g = P.Grid(dims, x)
    t1 = time.perf_counter()
    a = P.compress_device(g, 1e-3)
    t2 = time.perf_counter()
    rec("Grid: entry -> range call", marks["r0"] - t0)
    rec("Grid: range call -> return", t1 - marks["r1"])
    rec("compress: entry -> cszi_compress", marks["c0"] - t1)
    rec("compress: in cszi_compress", marks["c1"] - marks["c0"])
    rec("compress: cszi_compress -> return", t2 - marks["c1"])
    rec("step", t2 - t0)
for k, v in T.items():
    print(f"{k:40s} {1e6 * v / N:8.1f} us")
