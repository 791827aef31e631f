"""Micro-costs of the host layer: DeviceCtl(), ctl launches, fetch()."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2312_05492_b200 as P
from paper_2312_05492_b200 import _lib
from bench import smooth_field_gpu
x = smooth_field_gpu((512, 512, 512))
lib = _lib.load(); st = _lib.stream_ptr()
ctl = _lib.DeviceCtl()
def t(name, fn, n=200):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); print(f"{name:28s} {1e6*(time.perf_counter()-t0)/n:8.1f} us")
t("DeviceCtl()", lambda: _lib.DeviceCtl())
t("stream_ptr()", lambda: _lib.stream_ptr())
t("torch current_stream", lambda: torch.cuda.current_stream().cuda_stream)
t("current_device()", lambda: torch.cuda.current_device())
t("x.contiguous()", lambda: x.contiguous())
t("lib.load()", lambda: _lib.load())
t("P.Dims(shape)", lambda: P.Dims(x.shape))
t("_lib.ptr(x)", lambda: _lib.ptr(x))
t("ctl_init launch", lambda: lib.cszi_ctl_init(ctl.ptr, st))
t("fetch()", lambda: ctl.fetch())
t("stream.synchronize()", lambda: torch.cuda.current_stream().synchronize())
t("Grid(device) total", lambda: P.Grid(P.Dims(x.shape), x), 50)
g = P.Grid(P.Dims(x.shape), x)
t("compress_device", lambda: P.compress_device(g, 1e-3), 50)
a = P.compress_device(g, 1e-3)
t("decompress_device", lambda: P.decompress_device(a), 50)
