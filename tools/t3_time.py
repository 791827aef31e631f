"""A/B timing of the tile kernels and the steps around them (CUDA events,
device-resident).  For each shape: predict kernel alone (cszi_predict after
the range / tuner), full compress_device and decompress_device steps, and
archive sha256 (to compare builds).  Usage: t3_time.py [shape ...]"""
import ctypes
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2312_05492_b200 as P
from paper_2312_05492_b200 import _lib
from paper_2312_05492_b200.predictor import default_layout, make_geom, make_params
from paper_2312_05492_b200.tuning import compute_alpha
from bench import smooth_field_gpu


def ev_ms(fn, k=20):
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
    shapes = sys.argv[1:] or ["512,512,512", "449,449,235", "33120,69,69", "256,384,384"]
    lib = _lib.load()
    for sh in shapes:
        shape = tuple(int(v) for v in sh.split(","))
        n = shape[0] * shape[1] * shape[2]
        x = smooth_field_gpu(shape)
        dims = P.Dims(shape)
        arch = P.compress_device(P.Grid(dims, x), 1e-3)
        sha = hashlib.sha256(arch.to_bytes()).hexdigest()[:16]
        geom = make_geom(shape, default_layout(3))
        st = _lib.stream_ptr()
        ctl = _lib.DeviceCtl()
        samples = torch.empty(_lib.SAMPLE_WORDS, dtype=torch.int32, device="cuda")
        params = make_params(3, True, 1e-3, 512, compute_alpha(1e-3), 8)
        lib.cszi_scan_field(_lib.ptr(x), n, ctl.ptr, st)
        lib.cszi_tune(_lib.ptr(x), ctypes.byref(geom), ctypes.byref(params), _lib.ptr(samples),
                      ctl.ptr, st)
        sym = torch.empty(n + 16, dtype=torch.int16, device="cuda")
        hist = torch.empty(1024, dtype=torch.int64, device="cuda")
        kp = ev_ms(lambda: lib.cszi_predict(_lib.ptr(x), ctypes.byref(geom), 512, 0, _lib.ptr(sym),
                                            _lib.ptr(hist), ctl.ptr, st))
        c = ev_ms(lambda: P.compress_device(P.Grid(dims, x), 1e-3))
        d = ev_ms(lambda: P.decompress_device(arch))
        # the same steps with the ctl read-back replaced by its known result:
        # the host runs ahead, so this is the device time of a step
        fetch = _lib.DeviceCtl.fetch
        memo = {}

        def fetch_memo(self, _f=fetch):
            k = id(_f)
            if k not in memo:
                memo[k] = _f(self)
            return memo[k]

        _lib.DeviceCtl.fetch = fetch_memo
        try:
            cg = ev_ms(lambda: P.compress_device(P.Grid(dims, x), 1e-3))
            memo.clear()
            dg = ev_ms(lambda: P.decompress_device(arch))
        finally:
            _lib.DeviceCtl.fetch = fetch
        y = P.decompress_device(arch).tensor
        dsha = hashlib.sha256(y.cpu().numpy().tobytes()).hexdigest()[:16]
        print(f"{sh:14s} predict {1e3 * kp:7.1f} us ({n / kp / 1e6:6.2f} Gpt/s)  compress {1e3 * c:7.1f} us"
              f"  decompress {1e3 * d:7.1f} us  (device-only {1e3 * cg:6.1f} / {1e3 * dg:6.1f})"
              f"  archive {sha}  field {dsha}", flush=True)
        del x, y, sym, arch
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
