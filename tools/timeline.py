"""Device timeline of warm compress / decompress steps (torch.profiler /
CUPTI activity records): per-kernel start offset, duration and the idle gap
before it, so host time and launch gaps can be told apart from kernel time.
Usage: timeline.py [shape] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2312_05492_b200 as P
from bench import smooth_field_gpu


def main():
    shape = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "512,512,512").split(","))
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    x = smooth_field_gpu(shape)
    dims = P.Dims(shape)
    for _ in range(3):
        a = P.compress_device(P.Grid(dims, x), 1e-3)
        P.decompress_device(a)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(steps):
            a = P.compress_device(P.Grid(dims, x), 1e-3)
        torch.cuda.synchronize()
        for _ in range(steps):
            P.decompress_device(a)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    prev_end = None
    busy = 0.0
    rows = []
    for e in evs:
        s, d = e.time_range.start, e.time_range.end - e.time_range.start
        gap = 0.0 if prev_end is None else s - prev_end
        rows.append((s - t0, d, gap, e.name))
        busy += d
        prev_end = max(prev_end or 0, e.time_range.end)
    span = prev_end - t0
    for s, d, g, nm in rows:
        print(f"{s:10.1f} us  {d:8.1f} us  gap {g:7.1f}  {nm[:90]}")
    print(f"span {span:.1f} us, kernels+copies busy {busy:.1f} us, idle {span - busy:.1f} us "
          f"over {steps} compress + {steps} decompress steps")


if __name__ == "__main__":
    main()
