"""Host-path probe: bench-style compress / decompress step times (CUDA
events over a K-step loop, graphs on / off) against the sum of the kernel
times of one step, plus the pure host cost of one call on a tiny grid."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2312_05492_b200 as P
from bench import smooth_field_gpu


def loop_ms(fn, k=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


for shape in ((512, 512, 512), (32, 32, 32)):
    x = smooth_field_gpu(shape)
    dims = P.Dims(shape)
    a = P.compress_device(P.Grid(dims, x), 1e-3)
    c = loop_ms(lambda: P.compress_device(P.Grid(dims, x), 1e-3))
    d = loop_ms(lambda: P.decompress_device(a))
    t0 = time.perf_counter()
    for _ in range(30):
        P.compress_device(P.Grid(dims, x), 1e-3)
    tc = (time.perf_counter() - t0) / 30
    print(f"{shape}: compress step {c:.4f} ms  decompress step {d:.4f} ms  host wall/compress {1e3 * tc:.4f} ms",
          flush=True)
