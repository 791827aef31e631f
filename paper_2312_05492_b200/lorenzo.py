"""First-order Lorenzo predictor (mirrors ebcomp/lorenzo.py:22-53) on the GPU.

Raster-scan prediction from previously reconstructed neighbours (the signed
corner sum of the unit hypercube behind each point, out-of-grid neighbours
0), one global bound, no anchors -- the reference's comparison baseline.
The recurrence runs in libcszi (csrc/lorenzo.cu: anti-diagonal wavefronts of
tiles, bit-exact with the numba kernels of _kernels.py:104-215)."""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import Inconsistent
from .grid import Dims, Grid
from .predictor import QuantizedField, default_layout, make_geom

__all__ = ["lorenzo_predict_quantize", "lorenzo_reconstruct"]

_MAX_SYM = 0xFFFF  # symbols are uint16, 0xFFFF marks an outlier


def _geom(extents):
    return make_geom(extents, default_layout(len(extents)))


def lorenzo_predict_quantize(grid: Grid, eb: float, radius: int = 512) -> QuantizedField:
    """lorenzo.py:22-33: codes q (0 at outliers), outliers (flat index,
    original value), no anchors; eb is the absolute bound."""
    t = _lib.require_cuda()
    lib = _lib.load()
    R = int(radius)
    if R < 2:
        raise Inconsistent("quantizer radius must be at least 2")
    if 2 * R > 16384:
        raise NotImplementedError(f"quant_radius {R} exceeds the GPU codebook limit")
    grid.ensure_finite()
    x = grid.tensor.reshape(-1)
    n = grid.dims.count
    sym = t.empty(n + 16, dtype=t.int16, device="cuda")
    rec = t.empty(n, dtype=t.float32, device="cuda")
    ctl = _lib.DeviceCtl()
    geom = _geom(grid.dims.extents)
    _lib.check(lib.cszi_lorenzo_predict(_lib.ptr(x), ctypes.byref(geom), float(eb), R,
                                        _lib.ptr(sym), _lib.ptr(rec), ctl.ptr,
                                        _lib.stream_ptr()), "lorenzo_predict")
    s = sym[:n].to(t.int32) & 0xFFFF
    out = s == 0
    codes = t.where(out, t.zeros_like(s), s - R).cpu().numpy().astype(np.int32)
    oidx = t.nonzero(out).flatten()
    ovals = x[oidx].cpu().numpy()
    outliers = list(zip(oidx.cpu().numpy().tolist(), ovals.tolist()))
    return QuantizedField(codes=codes, outliers=outliers, anchors=[])


def lorenzo_reconstruct(field: QuantizedField, dims: Dims, eb: float) -> Grid:
    """lorenzo.py:36-53: replay the recurrence from codes and outliers."""
    t = _lib.require_cuda()
    lib = _lib.load()
    codes = np.ascontiguousarray(field.codes, dtype=np.int32).reshape(-1)
    if codes.size != dims.count:
        raise Inconsistent(f"{codes.size} codes for {dims.count} grid points")
    n = dims.count
    if field.outliers:
        oidx = np.asarray([i for i, _ in field.outliers], dtype=np.int64)
        oval = np.asarray([v for _, v in field.outliers], dtype=np.float32)
        if int(oidx.max()) >= n or int(oidx.min()) < -n:
            raise IndexError("outlier index out of bounds for the grid")
        oidx = np.where(oidx < 0, oidx + n, oidx)
        # the reference assigns through a boolean mask: the last value of a
        # repeated index wins; the device lookup needs a strictly increasing list
        order = np.argsort(oidx, kind="stable")
        oidx, oval = oidx[order], oval[order]
        keep = np.append(oidx[1:] != oidx[:-1], True)
        oidx, oval = oidx[keep], oval[keep]
    else:
        oidx = np.empty(0, dtype=np.int64)
        oval = np.empty(0, dtype=np.float32)
    # symbol = q + R with R large enough for every stored code
    qmax = int(np.abs(codes).max(initial=0))
    R = max(512, qmax + 1)
    if qmax + R >= _MAX_SYM:
        raise NotImplementedError(f"code magnitude {qmax} exceeds the uint16 symbol range")
    d_codes = t.from_numpy(codes).to("cuda")
    sym = (d_codes + R).to(t.int32)
    d_oidx = t.from_numpy(oidx).to("cuda")
    d_oval = t.from_numpy(oval).to("cuda")
    if oidx.size:
        sym[d_oidx] = _MAX_SYM
    sym16 = sym.to(t.int16)  # bit pattern: values < 2^16
    y = t.empty(n, dtype=t.float32, device="cuda")
    geom = _geom(dims.extents)
    _lib.check(lib.cszi_lorenzo_reconstruct(_lib.ptr(sym16), _lib.ptr(d_oidx), _lib.ptr(d_oval),
                                            int(oidx.size), ctypes.byref(geom), float(eb), R,
                                            _lib.ptr(y), _lib.stream_ptr()),
               "lorenzo_reconstruct")
    # Grid(dims, recon) of the reference: the finite scan runs on first use
    return Grid(dims, y.view(dims.extents))
