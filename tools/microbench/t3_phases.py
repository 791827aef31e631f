"""Per-phase cycle split of k_t3_predict: setup, TMA wait, passes, epilogue
(cycles per tile and warp) and per interior pass.  Needs the instrumented
build in place of libcszi.so:
  make -C paper_2312_05492_b200/csrc EXTRA=-DT3_PROF OUT=../../tools/microbench/libcszi_prof.so
  (objects land in csrc/build: `make clean` before the normal build)
  cp tools/microbench/libcszi_prof.so paper_2312_05492_b200/libcszi.so"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2312_05492_b200 as P
from paper_2312_05492_b200 import _lib
from bench import smooth_field_gpu
shape = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "512,512,512").split(","))
x = smooth_field_gpu(shape)
for _ in range(2):
    P.compress_device(P.Grid(P.Dims(x.shape), x), 1e-3)
torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_ulonglong * 16)()
lib.cszi_t3_prof(buf)
P.compress_device(P.Grid(P.Dims(x.shape), x), 1e-3)
torch.cuda.synchronize()
lib.cszi_t3_prof(buf)
n = buf[4]
names = ["setup", "tma_wait", "passes", "epilogue"]
tot = sum(buf[i] for i in range(4))
for i, nm in enumerate(names):
    print(f"{nm:10s} {buf[i] / n:10.0f} cycles/tile  {100 * buf[i] / tot:5.1f}%")
print("tiles", n)
ni = ((shape[0] - 1) // 8) * ((shape[1] - 1) // 8) * ((shape[2] - 1) // 32)  # interior tiles
for lv in range(3):
    print("level s=%d:" % (4 >> lv), " ".join(f"{buf[6 + lv * 3 + i] / ni:8.0f}" for i in range(3)))

print("edge tiles", buf[5], "pass cycles per edge tile", buf[15] / max(buf[5], 1))
