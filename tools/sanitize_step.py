"""Small compress + decompress round trips for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): every product kernel path is
exercised on shapes that run in seconds under instrumentation.

  compute-sanitizer --tool racecheck python tools/sanitize_step.py
  CSZI_NO_TMA=1 compute-sanitizer --tool memcheck python tools/sanitize_step.py

Shapes: 41x30x37 (edge shell, unaligned pitch -> row staging), 9x9x33 (one
closed tile), 24x16x64 (TMA + non-R bitmap encoder), rank 1 / 2, a noisy
field at 1e-5 (dense packer, outliers), Lorenzo, and a sliced decompress.
Exits non-zero when a round trip misses the bound."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2312_05492_b200 as P


def field(shape, seed, noise=0.0):
    rng = np.random.default_rng(seed)
    g = np.meshgrid(*[np.linspace(0, 3, s) for s in shape], indexing="ij")
    f = sum(np.sin((i + 1.3) * a) for i, a in enumerate(g))
    if noise:
        f = f + rng.normal(0, noise, shape)
    return np.ascontiguousarray(f, dtype=np.float32)


def trip(data, eb, **kw):
    g = P.Grid(P.Dims(data.shape), torch.from_numpy(data).cuda())
    arch = P.compress_device(g, eb, **kw)
    y = P.decompress_device(arch).data
    eb_abs = P.parse_archive(arch.to_bytes()).eb_abs
    err = float(np.abs(y.astype(np.float64) - data).max())
    ok = err <= eb_abs
    print(f"{str(data.shape):18s} eb={eb:g} {kw} bytes={len(arch.to_bytes())} err={err:.3g} "
          f"bound={eb_abs:.3g} {'ok' if ok else 'FAIL'}", flush=True)
    return ok


def main():
    torch.cuda.set_device(0)
    ok = True
    ok &= trip(field((41, 30, 37), 1), 1e-3)
    ok &= trip(field((9, 9, 33), 2), 1e-3)
    ok &= trip(field((24, 16, 64), 3), 1e-3)
    ok &= trip(field((24, 16, 64), 4, noise=0.05), 1e-5)
    ok &= trip(field((300,), 5), 1e-3)
    ok &= trip(field((40, 50), 6), 1e-3)
    ok &= trip(field((17, 20, 23), 7), 1e-3, predictor="lorenzo")
    # sliced decompress (one z-slab)
    data = field((40, 16, 64), 8)
    g = P.Grid(P.Dims(data.shape), torch.from_numpy(data).cuda())
    arch = P.compress_device(g, 1e-3)
    whole = P.decompress_device(arch).data
    part = P.decompress_device(arch, slab=(8, 24))
    part = part.data if hasattr(part, "data") else part
    part = part.cpu().numpy() if isinstance(part, torch.Tensor) else np.asarray(part)
    same = np.array_equal(part.reshape(-1), whole[8:24].reshape(-1))
    print(f"slab (8, 24) equals whole planes: {same}", flush=True)
    ok &= same
    torch.cuda.synchronize()
    print("ALL OK" if ok else "FAILED")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
