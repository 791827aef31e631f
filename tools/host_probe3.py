import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_05492_b200 import _lib
lib = _lib.load(); st = _lib.stream_ptr(); ctl = _lib.DeviceCtl(); p = ctl.ptr
torch.cuda.synchronize()
for name, fn in [("ctypes cszi_launch_count", lambda: lib.cszi_launch_count()),
                 ("cszi_ctl_init (host only)", lambda: lib.cszi_ctl_init(p, st))]:
    t0 = time.perf_counter()
    for _ in range(200): fn()
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"{name:28s} host {1e6*(t1-t0)/200:7.1f} us/call, drain {1e6*(t2-t1):8.1f} us")
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
for _ in range(200): lib.cszi_ctl_init(p, st)
ev1.record(); torch.cuda.synchronize()
print("gpu time per ctl_init", ev0.elapsed_time(ev1) / 200 * 1000, "us")
x = torch.zeros(1024, device="cuda")
px = _lib.ptr(x)
for name, fn in [("cszi_range n=1024", lambda: lib.cszi_range(px, 1024, p, st)),
                 ("cszi_ctl_init again", lambda: lib.cszi_ctl_init(p, st))]:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200): fn()
    t1 = time.perf_counter(); torch.cuda.synchronize()
    print(f"{name:28s} host {1e6*(t1-t0)/200:7.1f} us/call")
