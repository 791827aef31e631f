"""CPU cost of the Python helpers on the compress critical path."""
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2312_05492_b200 as P
from paper_2312_05492_b200 import _lib, pipeline as PL
from paper_2312_05492_b200.tuning import compute_alpha
from paper_2312_05492_b200.predictor import default_layout
from bench import smooth_field_gpu
x = smooth_field_gpu((512, 512, 512))
dims = P.Dims(x.shape)
g = P.Grid(dims, x)
def t(name, fn, n=2000):
    t0 = time.perf_counter()
    for _ in range(n): fn()
    print(f"{name:34s} {1e6*(time.perf_counter()-t0)/n:7.2f} us")
t("compute_alpha(1e-3)", lambda: compute_alpha(1e-3))
t("default_layout(3)", lambda: default_layout(3))
t("thread_count(None)", lambda: PL.thread_count(None))
t("require_cuda()", lambda: _lib.require_cuda())
t("_lib.load()", lambda: _lib.load())
t("stream_ptr()", lambda: _lib.stream_ptr())
t("grid.tensor", lambda: g.tensor)
t("grid.dims.count", lambda: g.dims.count)
t("grid.is_device", lambda: g.is_device)
t("WS.get", lambda: _lib.WS.get(1000, "compress"))
t("_payload_buf(3MB)", lambda: PL._payload_buf(3 << 20))
lay = default_layout(3)
t("_compress_prep (hit)", lambda: PL._compress_prep(dims.extents, lay, True, 1e-3, 512, 1.5, None, None, False, False))
a = P.compress_device(g, 1e-3)
t("DeviceCtl()", lambda: _lib.DeviceCtl())
t("Grid(dims, x) [sync]", lambda: P.Grid(dims, x), 200)
t("compress_device [sync]", lambda: P.compress_device(g, 1e-3), 200)
