"""Where the host-buffer decompress time goes (e2e leg of bench.py)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2312_05492_b200 as P
from bench import smooth_field_gpu
shape = (512, 512, 512)
x = smooth_field_gpu(shape)
blob = P.compress_device(P.Grid(P.Dims(shape), x), 1e-3).to_bytes()
for _ in range(3):
    g = P.decompress(blob)
torch.cuda.synchronize()
N = 10
t0 = time.perf_counter()
for _ in range(N):
    g = P.decompress(blob)
t1 = time.perf_counter()
print(f"decompress(bytes) {1e3*(t1-t0)/N:.2f} ms")
y = P.decompress_device(blob).tensor.reshape(-1)
torch.cuda.synchronize()
h = torch.empty(y.numel(), dtype=torch.float32, pin_memory=True)
for name, fn in [("pinned alloc", lambda: torch.empty(y.numel(), dtype=torch.float32, pin_memory=True)),
                 ("D2H pinned (reused)", lambda: h.copy_(y, non_blocking=False)),
                 ("decompress_device", lambda: P.decompress_device(blob))]:
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(N):
        r = fn()
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"{name} {1e3*(t1-t0)/N:.2f} ms")
pin = torch.empty(shape, dtype=torch.float32, pin_memory=True); pin.copy_(x)
for name, fn in [("H2D pinned", lambda: pin.to('cuda', non_blocking=True)),
                 ("compress(host pinned)", lambda: P.compress(P.Grid(P.Dims(shape), pin.numpy()), 1e-3))]:
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(N):
        r = fn()
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"{name} {1e3*(t1-t0)/N:.2f} ms")

# the bench's e2e loop pattern (events on the current stream, result kept alive)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for steps in (10, 50):
    torch.cuda.synchronize()
    ev0.record()
    t0 = time.perf_counter()
    for _ in range(steps):
        back = P.decompress(blob)
    ev1.record()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"bench-pattern decompress x{steps}: events {ev0.elapsed_time(ev1)/steps:.2f} ms, wall {1e3*(t1-t0)/steps:.2f} ms")
