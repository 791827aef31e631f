"""Anchored multi-level interpolation predictor — host-side API.

Mirrors the public surface of ebcomp/predictor.py (layouts, configs, level
plans, the scalar semantic definitions ``quantize`` / ``spline_predict``)
while every grid-sized computation runs in libcszi on the GPU:

* ``compress_predict``   -> cszi_tune (config) + cszi_predict (fused
  G-Interp predict/quantize kernel, csrc/predict.cu)   predictor.py:395-420
* ``decompress_predict`` -> cszi_reconstruct (inverse interpolation)
                                                        predictor.py:423-465
* ``gather_anchors``     -> cszi_gather_anchors         predictor.py:250-256
"""

from __future__ import annotations

import ctypes
import functools
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import Inconsistent, InvalidStride, NoNeighbor
from .grid import Dims, Grid

NOTAKNOT = 0
NATURAL = 1

# predictor.py:62-69 weight vectors over offsets (-3s, -s, +s, +3s)
CUBIC_WEIGHTS = {
    NOTAKNOT: (-1.0 / 16.0, 9.0 / 16.0, 9.0 / 16.0, -1.0 / 16.0),
    NATURAL: (-3.0 / 40.0, 23.0 / 40.0, 23.0 / 40.0, -3.0 / 40.0),
}
QUAD_LEFT = (-1.0 / 8.0, 6.0 / 8.0, 3.0 / 8.0, 0.0)
QUAD_RIGHT = (0.0, 3.0 / 8.0, 6.0 / 8.0, -1.0 / 8.0)
LINEAR = (0.0, 0.5, 0.5, 0.0)
COPY = (0.0, 1.0, 0.0, 0.0)

_DEFAULT_STRIDE = {1: 512, 2: 16, 3: 8}
_DEFAULT_TILES = {1: (512,), 2: (16, 16), 3: (8, 8, 32)}


def _is_pow2(n: int) -> bool:
    return n >= 2 and (n & (n - 1)) == 0


@dataclass(frozen=True)
class ChunkLayout:
    """Anchor stride plus the super-chunk tile confining neighbour reads."""

    anchor_stride: int
    rank: int
    super_chunk_extents: tuple

    def __post_init__(self):
        if not _is_pow2(self.anchor_stride):
            raise InvalidStride(f"anchor stride {self.anchor_stride} is not a power of two")
        if len(self.super_chunk_extents) != self.rank:
            raise Inconsistent("super-chunk extents do not match rank")
        for e in self.super_chunk_extents:
            if e < self.anchor_stride or e % self.anchor_stride:
                raise Inconsistent(f"super-chunk extent {e} is not a multiple of the anchor stride")


@functools.lru_cache(maxsize=None)
def default_layout(rank: int) -> ChunkLayout:
    """Stride 8 / tiles (8,8,32) in 3D, 16 / (16,16) in 2D, 512 in 1D
    (frozen, so one shared instance per rank)."""
    return ChunkLayout(_DEFAULT_STRIDE[rank], rank, _DEFAULT_TILES[rank])


@dataclass(frozen=True)
class LevelStep:
    level: int
    stride: int
    eb: float


@dataclass(frozen=True)
class LevelPlan:
    levels: tuple
    global_eb: float
    alpha: float


def plan_levels(anchor_stride: int, eb: float, alpha: float) -> LevelPlan:
    """Per-level bounds eb / alpha**(level-1), coarsest first (predictor.py:122-136)."""
    if not _is_pow2(anchor_stride):
        raise InvalidStride(f"anchor stride {anchor_stride} is not a power of two")
    steps = []
    s = anchor_stride // 2
    while s >= 1:
        level = s.bit_length()
        steps.append(LevelStep(level=level, stride=s, eb=eb / alpha ** (level - 1)))
        s //= 2
    return LevelPlan(levels=tuple(steps), global_eb=eb, alpha=alpha)


@dataclass(frozen=True)
class PredictorConfig:
    layout: ChunkLayout
    alpha: float
    cubic_variant_per_dim: tuple
    dim_order: tuple
    eb_abs: float
    quant_radius: int = 512

    def __post_init__(self):
        rank = self.layout.rank
        if sorted(self.dim_order) != list(range(rank)):
            raise Inconsistent(f"dim_order {self.dim_order} is not a permutation")
        if len(self.cubic_variant_per_dim) != rank:
            raise Inconsistent("one cubic variant per dimension required")
        if self.quant_radius < 2:
            raise Inconsistent("quantizer radius must be at least 2")
        if not self.eb_abs > 0:
            raise Inconsistent("absolute error bound must be positive")


@dataclass(frozen=True, eq=False)
class QuantizedField:
    """Dense codes plus the sparse lossless side channels (predictor.py:160-171)."""

    codes: np.ndarray
    outliers: list
    anchors: list


@dataclass(frozen=True)
class Code:
    q: int


@dataclass(frozen=True)
class Outlier:
    pass


OUTLIER = Outlier()


def quantize(original: float, predicted: float, level_eb: float, radius: int):
    """Scalar semantic definition (predictor.py:187-198)."""
    t = (float(original) - float(predicted)) / (2.0 * float(level_eb))
    q = math.trunc(t + math.copysign(0.5, t))
    if abs(q) >= radius:
        return OUTLIER
    return Code(q)


def spline_predict(neighbors, cubic_variant: int = NOTAKNOT) -> float:
    """Scalar semantic definition (predictor.py:201-223)."""
    m3, m1, p1, p3 = (v is not None for v in neighbors)
    if not m1:
        raise NoNeighbor("the -s neighbor is required; traversal order guarantees it")
    if m3 and p1 and p3:
        w = CUBIC_WEIGHTS[cubic_variant]
    elif m3 and p1:
        w = QUAD_LEFT
    elif p1 and p3:
        w = QUAD_RIGHT
    elif p1:
        w = LINEAR
    else:
        w = COPY
    v = [0.0 if n is None else float(n) for n in neighbors]
    return ((w[0] * v[0] + w[1] * v[1]) + w[2] * v[2]) + w[3] * v[3]


# ---------------------------------------------------------------------------
# anchor lattice (predictor.py:230-256)
# ---------------------------------------------------------------------------

def _anchor_axis(extent: int, stride: int) -> np.ndarray:
    coords = list(range(0, extent, stride))
    if coords[-1] != extent - 1:
        coords.append(extent - 1)
    return np.asarray(coords, dtype=np.int64)


def _anchor_coords(extents, stride: int):
    return tuple(_anchor_axis(e, stride) for e in extents)


def count_anchors(dims: Dims, stride: int) -> int:
    """Anchor count without touching data (closed-form per axis)."""
    n = 1
    for e in dims.extents:
        k = (e + stride - 1) // stride
        if (k - 1) * stride != e - 1:
            k += 1
        n *= k
    return n


def anchor_flat_indices(extents, stride: int) -> np.ndarray:
    mesh = np.meshgrid(*_anchor_coords(extents, stride), indexing="ij")
    return np.ravel_multi_index(mesh, extents).ravel()


# ---------------------------------------------------------------------------
# geometry helpers shared with the pipeline
# ---------------------------------------------------------------------------

def make_geom(extents, layout: ChunkLayout) -> _lib.Geom:
    rank = len(extents)
    pad = 3 - rank
    g = _lib.Geom()
    g.rank = rank
    ext = (1,) * pad + tuple(int(e) for e in extents)
    til = (1,) * pad + tuple(int(t) for t in layout.super_chunk_extents)
    for a in range(3):
        g.ext[a] = ext[a]
        g.tile[a] = til[a]
    g.stride = int(layout.anchor_stride)
    return g


def nlevels(stride: int) -> int:
    return int(stride).bit_length() - 1


def alpha_powers(alpha: float, stride: int) -> list:
    """alpha ** (level - 1) for level = 1..log2(S) — CPython float pow, as
    plan_levels evaluates it."""
    return [alpha ** k for k in range(nlevels(stride))]


def make_params(rank: int, mode_rel: bool, eb: float, radius: int, alpha: float,
                stride: int, variants=None, dim_order=None, exact: bool = False) -> _lib.Params:
    pad = 3 - rank
    p = _lib.Params()
    p.mode_rel = 1 if mode_rel else 0
    p.radius = int(radius)
    p.eb = float(eb)
    p.have_alpha = 1
    p.alpha = float(alpha)
    for k, v in enumerate(alpha_powers(float(alpha), stride)):
        p.alpha_pow[k] = v
    if variants is not None:
        p.have_variants = 1
        for d, v in enumerate(variants):
            p.variant[pad + d] = int(v)
    if dim_order is not None:
        p.have_order = 1
        for i, d in enumerate(dim_order):
            p.order[i] = pad + int(d)
    p.exact = 1 if exact else 0
    return p


def ctl_variants(c: _lib.Ctl, rank: int) -> tuple:
    pad = 3 - rank
    return tuple(int(c.variant[pad + d]) for d in range(rank))


def ctl_order(c: _lib.Ctl, rank: int) -> tuple:
    pad = 3 - rank
    return tuple(int(c.order[i]) - pad for i in range(rank))


# ---------------------------------------------------------------------------
# level execution (predictor.py:264-392): the fine-grained per-level API
# ---------------------------------------------------------------------------

@dataclass
class Compress:
    """Quantize against ``source`` while reconstructing (predictor.py:264-271).
    Arrays are numpy (updated in place after the GPU pass) or CUDA tensors
    (updated in HBM)."""

    source: object
    codes: object
    is_outlier: object
    anchor_block: object


@dataclass
class Decompress:
    """Reconstruct from stored codes and outlier values (predictor.py:274-281)."""

    codes: object
    is_outlier: object
    outlier_values: object
    anchor_block: object


def _dev(a, dtype):
    """(CUDA tensor view, write-back numpy array or None) for a level operand."""
    t = _lib.torch()
    if isinstance(a, t.Tensor):
        if not a.is_cuda or not a.is_contiguous():
            raise ValueError("device operands must be contiguous CUDA tensors")
        if dtype == np.bool_:
            return a.view(t.uint8), None
        return a, None
    arr = np.asarray(a)
    host = np.ascontiguousarray(arr, dtype=dtype)
    d = t.from_numpy(host.view(np.uint8) if dtype == np.bool_ else host).cuda()
    return d, arr


def interpolate_level(recon, level: LevelStep, config: PredictorConfig, mode,
                      threads: int = 1) -> None:
    """Run one level's per-dimension passes on the GPU (predictor.py:367-392);
    ``recon`` must hold lattice 2s.  Same point sets, arithmetic and anchor
    restores as the reference; numpy operands are written back in place."""
    t = _lib.require_cuda()
    lib = _lib.load()
    extents = tuple(int(e) for e in (recon.shape if hasattr(recon, "shape") else ()))
    rank = len(extents)
    if rank != config.layout.rank:
        raise Inconsistent("recon rank does not match the layout")
    d_rec, h_rec = _dev(recon, np.float32)
    comp = isinstance(mode, Compress)
    if not comp and not isinstance(mode, Decompress):
        raise TypeError("mode must be Compress or Decompress")
    d_codes, h_codes = _dev(mode.codes, np.int32)
    d_out, h_out = _dev(mode.is_outlier, np.bool_)
    d_anc, _ = _dev(mode.anchor_block, np.float32)
    d_src = _dev(mode.source, np.float32)[0] if comp else None
    d_oval = None if comp else _dev(mode.outlier_values, np.float32)[0]
    geom = make_geom(extents, config.layout)
    pad = 3 - rank
    var = (ctypes.c_int32 * 3)(*((0,) * pad + tuple(int(v) for v in config.cubic_variant_per_dim)))
    order = (ctypes.c_int32 * 3)(*(tuple(pad + int(d) for d in config.dim_order) + (0,) * pad))
    _lib.check(lib.cszi_interp_level(
        _lib.ptr(d_rec), _lib.ptr(d_src) if comp else None, _lib.ptr(d_codes), _lib.ptr(d_out),
        None if comp else _lib.ptr(d_oval), _lib.ptr(d_anc), ctypes.byref(geom),
        int(level.stride), float(level.eb), var, order, int(config.quant_radius),
        0 if comp else 1, _lib.stream_ptr()), "interp_level")
    if h_rec is not None:
        h_rec[...] = d_rec.cpu().numpy().reshape(h_rec.shape)
    if comp:
        if h_codes is not None:
            h_codes[...] = d_codes.cpu().numpy().reshape(h_codes.shape)
        if h_out is not None:
            h_out[...] = d_out.cpu().numpy().view(np.bool_).reshape(h_out.shape)


# ---------------------------------------------------------------------------
# GPU-backed predictor API
# ---------------------------------------------------------------------------

def _run_predict(grid: Grid, config: PredictorConfig, exact: bool = False):
    """cszi_tune (explicit config) + cszi_predict -> (sym uint16 tensor, hist, ctl)."""
    t = _lib.require_cuda()
    lib = _lib.load()
    grid.ensure_finite()
    x = grid.tensor
    rank = grid.dims.rank
    geom = make_geom(grid.dims.extents, config.layout)
    params = make_params(rank, False, config.eb_abs, config.quant_radius, config.alpha,
                         config.layout.anchor_stride, config.cubic_variant_per_dim,
                         config.dim_order, exact)
    ctl = _lib.DeviceCtl()
    st = _lib.stream_ptr()
    n = grid.dims.count
    sym = t.empty(n + 16, dtype=t.int16, device="cuda")
    hist = t.empty(2 * config.quant_radius, dtype=t.int64, device="cuda")
    _lib.check(lib.cszi_ctl_init(ctl.ptr, st), "ctl_init")
    samples = t.empty(_lib.SAMPLE_WORDS, dtype=t.int32, device="cuda")
    _lib.check(lib.cszi_tune(_lib.ptr(x), ctypes.byref(geom), ctypes.byref(params),
                             _lib.ptr(samples), ctl.ptr, st), "tune")
    _lib.check(lib.cszi_predict(_lib.ptr(x), ctypes.byref(geom), config.quant_radius,
                                1 if exact else 0, _lib.ptr(sym), _lib.ptr(hist), ctl.ptr, st),
               "predict")
    return sym[:n], hist, ctl, x


def compress_predict(grid: Grid, config: PredictorConfig, threads: int = 1) -> QuantizedField:
    """Predict/quantize every non-anchor point on the GPU (predictor.py:395-420)."""
    sym_t, _, ctl, x = _run_predict(grid, config)
    c = ctl.fetch()
    if c.flags & _lib.F_EB_NONPOSITIVE:
        raise Inconsistent("absolute error bound must be positive")
    sym = sym_t.view(dtype=sym_t.dtype).cpu().numpy().view(np.uint16).astype(np.int32)
    R = config.quant_radius
    out_mask = sym == 0
    codes = sym - R
    codes[out_mask] = 0
    data = grid.values
    oidx = np.nonzero(out_mask)[0]
    outliers = list(zip(oidx.tolist(), data[oidx].tolist()))
    return QuantizedField(codes=codes, outliers=outliers,
                          anchors=gather_anchors(grid, config.layout.anchor_stride))


def gather_anchors(grid: Grid, stride: int):
    """(flat index, value) for every anchor, ascending flat index, gathered on the GPU."""
    t = _lib.require_cuda()
    lib = _lib.load()
    extents = grid.dims.extents
    layout = ChunkLayout(stride, grid.dims.rank, (stride,) * grid.dims.rank)
    geom = make_geom(extents, layout)
    na = count_anchors(grid.dims, stride)
    out = t.empty(na, dtype=t.float32, device="cuda")
    _lib.check(lib.cszi_gather_anchors(_lib.ptr(grid.tensor), ctypes.byref(geom), _lib.ptr(out),
                                       _lib.stream_ptr()), "gather_anchors")
    vals = out.cpu().numpy()
    idx = anchor_flat_indices(extents, stride)
    return list(zip(idx.tolist(), vals.tolist()))


def decompress_predict(field: QuantizedField, config: PredictorConfig, dims: Dims,
                       threads: int = 1) -> Grid:
    """Replay the prediction from codes on the GPU (predictor.py:423-465)."""
    t = _lib.require_cuda()
    lib = _lib.load()
    extents = dims.extents
    codes = np.ascontiguousarray(field.codes, dtype=np.int32).ravel()
    if codes.size != dims.count:
        raise Inconsistent(f"{codes.size} codes for {dims.count} grid points")
    stride = config.layout.anchor_stride
    expected = anchor_flat_indices(extents, stride)
    got = np.asarray([i for i, _ in field.anchors], dtype=np.int64) if field.anchors else \
        np.empty(0, dtype=np.int64)
    if not np.array_equal(got, expected):
        raise Inconsistent("anchor indices do not match the lattice for these dims")
    R = config.quant_radius
    sym = (codes.astype(np.int64) + R)
    if sym.min(initial=0) < 0 or sym.max(initial=0) >= 2 * R:
        raise NotImplementedError("codes outside (-R, R) are not representable as symbols")
    sym = sym.astype(np.uint16)
    if field.outliers:
        oidx = np.asarray([i for i, _ in field.outliers], dtype=np.int64)
        oval = np.asarray([v for _, v in field.outliers], dtype=np.float32)
        order = np.argsort(oidx, kind="stable")
        oidx, oval = oidx[order], oval[order]
        sym[oidx] = 0xFFFF
    else:
        oidx = np.zeros(1, dtype=np.int64)
        oval = np.zeros(1, dtype=np.float32)
    n_out = len(field.outliers)
    anchors = np.asarray([v for _, v in field.anchors], dtype=np.float32)
    d_sym = t.from_numpy(sym.view(np.int16)).cuda()
    d_anc = t.from_numpy(anchors).cuda()
    d_oidx = t.from_numpy(oidx.astype(np.int64)).cuda()
    d_oval = t.from_numpy(oval).cuda()
    y = t.empty(dims.count, dtype=t.float32, device="cuda")
    geom = make_geom(extents, config.layout)
    plan = plan_levels(stride, config.eb_abs, config.alpha)
    leb = (ctypes.c_double * _lib.MAX_LEVELS)(*[s.eb for s in plan.levels])
    rank = dims.rank
    pad = 3 - rank
    var = (ctypes.c_int32 * 3)(*((0,) * pad + tuple(int(v) for v in config.cubic_variant_per_dim)))
    order = (ctypes.c_int32 * 3)(*(tuple(pad + int(d) for d in config.dim_order) + (0,) * pad))
    _lib.check(lib.cszi_reconstruct(_lib.ptr(d_sym), _lib.ptr(d_anc), _lib.ptr(d_oidx),
                                    _lib.ptr(d_oval), n_out, ctypes.byref(geom), R, leb,
                                    len(plan.levels), var, order, _lib.ptr(y),
                                    _lib.stream_ptr()), "reconstruct")
    return Grid(dims, y.cpu().numpy())
