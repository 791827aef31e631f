"""e2e decompress(bytes) breakdown on the 512^3 bench field: the bench's
loop pattern against its parts (device decompress, range scan, pinned D2H)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2312_05492_b200 as P
from bench import smooth_field_gpu


def loop_ms(fn, k=10):
    out = fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        out = fn()
    torch.cuda.synchronize()
    del out
    return (time.perf_counter() - t0) / k * 1e3


shape = (512, 512, 512)
x = smooth_field_gpu(shape)
dims = P.Dims(shape)
pinned = torch.empty(shape, dtype=torch.float32, pin_memory=True)
pinned.copy_(x)
hg = P.Grid(dims, pinned.numpy())
blob = P.compress(hg, 1e-3)
print("decompress(bytes), bench loop  ms", loop_ms(lambda: P.decompress(blob)))
print("decompress_device(bytes)       ms", loop_ms(lambda: P.decompress_device(blob)))
y = P.decompress_device(blob).tensor.reshape(-1)
host = torch.empty(y.numel(), dtype=torch.float32, pin_memory=True)
print("D2H into one pinned buffer     ms", loop_ms(lambda: host.copy_(y, non_blocking=True)))
print("pinned alloc + D2H (loop)      ms",
      loop_ms(lambda: torch.empty(y.numel(), dtype=torch.float32, pin_memory=True)
              .copy_(y, non_blocking=True)))
print("compress(host grid), bench loop ms", loop_ms(lambda: P.compress(hg, 1e-3)))

# decompress() step by step (the same calls as pipeline.decompress)
from paper_2312_05492_b200 import _lib  # noqa: E402

lib = _lib.load()
for it in range(4):
    t0 = time.perf_counter()
    g = P.decompress_device(blob)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    yy = g.tensor.reshape(-1)
    ctl = _lib.DeviceCtl()
    st = _lib.stream_ptr()
    lib.cszi_ctl_init(ctl.ptr, st)
    lib.cszi_range(_lib.ptr(yy), yy.numel(), ctl.ptr, st)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    host = _lib.PINNED.get(4 * yy.numel()).view(torch.float32)
    t3 = time.perf_counter()
    host.copy_(yy, non_blocking=True)
    c = ctl.fetch()
    t4 = time.perf_counter()
    gg = P.Grid.wrap_host(g.dims, host.numpy())
    t5 = time.perf_counter()
    print(f"iter {it}: device {1e3*(t1-t0):.2f}  range {1e3*(t2-t1):.2f}  pool {1e3*(t3-t2):.2f}  "
          f"d2h+fetch {1e3*(t4-t3):.2f}  wrap {1e3*(t5-t4):.2f} ms", flush=True)
