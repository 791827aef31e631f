"""Per-call device time of decompress_device(arch) against the slab path
(decompress_device(arch, slab=(0, nz)) and half slabs) on one shape, and
whether the exact transfer-table retry (table_mode 1) fires.
Usage: slab_probe.py [shape]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2312_05492_b200 as P
from paper_2312_05492_b200 import pipeline
from bench import smooth_field_gpu


def ev_ms(fn, k=10):
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


def main():
    shape = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "449,449,235").split(","))
    x = smooth_field_gpu(shape)
    a = P.compress_device(P.Grid(P.Dims(shape), x), 1e-3)
    calls = []
    orig = pipeline._lib.DeviceCtl.fetch

    def fetch(self, _f=orig):
        c = _f(self)
        calls.append(int(c.scratch[1]))
        return c

    pipeline._lib.DeviceCtl.fetch = fetch
    nz = shape[0]
    for name, fn in (("whole", lambda: P.decompress_device(a)),
                     ("slab all", lambda: P.decompress_device(a, slab=(0, nz))),
                     ("slab lo", lambda: P.decompress_device(a, slab=(0, (nz // 16) * 8))),
                     ("slab hi", lambda: P.decompress_device(a, slab=((nz // 16) * 8, nz)))):
        calls.clear()
        ms = ev_ms(fn)
        print(f"{name:9s} {1e3 * ms:8.1f} us  fetches {len(calls)}  retry flags {sorted(set(calls))}",
              flush=True)
    pipeline._lib.DeviceCtl.fetch = orig


if __name__ == "__main__":
    main()
