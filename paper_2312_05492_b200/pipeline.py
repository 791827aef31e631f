"""End-to-end compression pipeline — the drop-in boundary.

``compress(grid, eb, ...) -> bytes`` and ``decompress(data) -> Grid`` keep the
signatures, defaults, error classes and archive bytes of
ebcomp/pipeline.py:66-204.  One call = one stream-ordered sequence of
libcszi kernels on the current CUDA stream (range -> tune -> fused
predict/quantize/histogram -> anchors -> codebook -> Huffman encode ->
section assembly -> pass-2 encode), then a single device->host read of the
control record and the payload.  ``compress_device`` / ``decompress_device``
are the same path without the host copies (inputs and outputs stay in HBM).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._keys import key_to_float
from .archive import (
    EB_ABS,
    EB_REL,
    HEADER_SIZE,
    PREDICTOR_INTERP,
    PREDICTOR_LORENZO,
    pack_header,
    unpack_header,
)
from .errors import (
    Corrupt,
    EmptyHistogram,
    Inconsistent,
    LengthMismatch,
    LengthOverflow,
    MalformedSection,
    NonFiniteValue,
    TruncatedStream,
)
from .grid import Dims, Grid
from .pass2 import DEFAULT_CODEC, lookup
from .predictor import (
    ChunkLayout,
    count_anchors,
    ctl_order,
    ctl_variants,
    default_layout,
    make_geom,
    make_params,
    plan_levels,
)
from .tuning import compute_alpha

__all__ = ["compress", "decompress", "compress_device", "decompress_device", "thread_count",
           "DeviceArchive"]

_MODE_IDS = {"abs": EB_ABS, "rel": EB_REL}
_MAX_BINS = 16384


def thread_count(threads=None) -> int:
    """Explicit argument, else EBCOMP_THREADS, else 1 (pipeline.py:49-56).

    The GPU path is byte-identical for every value; the count is accepted for
    API compatibility only."""
    if threads is not None:
        return max(1, int(threads))
    try:
        return max(1, int(os.environ.get("EBCOMP_THREADS", "1")))
    except ValueError:
        return 1


@dataclass
class DeviceArchive:
    """An archive whose payload stays in device memory."""

    header: bytes
    payload: object  # CUDA uint8 tensor (payload_len bytes) or host bytes

    def __len__(self) -> int:
        return HEADER_SIZE + int(len(self.payload) if isinstance(self.payload, bytes)
                                 else self.payload.numel())

    def to_bytes(self) -> bytes:
        if isinstance(self.payload, bytes):
            return self.header + self.payload
        t = _lib.torch()
        n = self.payload.numel()
        host = _lib.PINNED.get(n)
        if n:
            host.copy_(self.payload, non_blocking=True)
            t.cuda.current_stream().synchronize()
        return self.header + host.numpy().tobytes()


def _payload_buf(nbytes: int):
    """A fresh payload buffer per call (the returned DeviceArchive owns it;
    torch's caching allocator makes this cheap)."""
    t = _lib.require_cuda()
    return t.empty(int(nbytes), dtype=t.uint8, device="cuda")


_caps_hint = {}


def _caps_for(n: int, worst: bool) -> _lib.Caps:
    c = _lib.Caps()
    if worst:
        c.bits_cap = (4 * n + 64 + 15) & ~15
        c.outlier_cap = n + 16
    else:
        c.bits_cap = ((n * 10) // 8 + 65536 + 15) & ~15
        c.outlier_cap = n // 32 + 4096
    return c


_prep_cache = {}


def _compress_prep(extents, layout, rel, eb, R, a, variants, dim_order, exact, worst):
    """(params, geom, caps, workspace bytes, payload capacity) of a compress
    call, memoised: the structs are read-only inputs of cszi_compress, and
    building them sits between the caller and the first kernel launch."""
    key = (extents, layout.anchor_stride, rel, eb, R, a, variants, dim_order, exact, worst)
    hit = _prep_cache.get(key)
    if hit is not None:
        return hit
    lib = _lib.load()
    rank = len(extents)
    params = make_params(rank, rel, eb, R, a, layout.anchor_stride, variants, dim_order, exact)
    geom = make_geom(extents, layout)
    n = 1
    for e in extents:
        n *= e
    caps = _caps_for(n, worst)
    ws_bytes = int(lib.cszi_compress_workspace_size(ctypes.byref(geom), R, ctypes.byref(caps)))
    pcap = int(lib.cszi_payload_capacity(ctypes.byref(geom), R, ctypes.byref(caps)))
    if len(_prep_cache) > 256:
        _prep_cache.clear()
    hit = (params, geom, caps, ws_bytes, pcap)
    _prep_cache[key] = hit
    return hit


def compress_device(grid: Grid, eb: float, mode: str = "rel", predictor: str = "interp",
                    pass2: bool = True, pass2_codec: int = DEFAULT_CODEC, alpha: float = None,
                    variants=None, dim_order=None, quant_radius: int = 512,
                    threads: int = None, exact: bool = False) -> DeviceArchive:
    """compress() with the payload left in device memory."""
    if mode not in _MODE_IDS:
        raise ValueError(f"unknown error-bound mode {mode!r}")
    if not eb > 0:
        raise ValueError("error bound must be positive")
    thread_count(threads)
    if predictor == "lorenzo":
        return _compress_lorenzo(grid, eb, mode, pass2, pass2_codec, quant_radius)
    if predictor != "interp":
        raise ValueError(f"unknown predictor {predictor!r}")
    rank = grid.dims.rank
    layout = default_layout(rank)
    if variants is not None:
        variants = tuple(int(v) for v in variants)
        if len(variants) != rank:
            raise Inconsistent("one cubic variant per dimension required")
    if dim_order is not None:
        dim_order = tuple(int(d) for d in dim_order)
        if sorted(dim_order) != list(range(rank)):
            raise Inconsistent(f"dim_order {dim_order} is not a permutation")
    R = int(quant_radius)
    if R < 2:
        raise Inconsistent("quantizer radius must be at least 2")
    if 2 * R > _MAX_BINS:
        raise NotImplementedError(f"quant_radius {R} exceeds the GPU codebook limit")
    codec_enc = None
    if pass2 and pass2_codec != DEFAULT_CODEC:
        codec_enc = lookup(pass2_codec)[0]

    t = _lib.require_cuda()
    lib = _lib.load()
    st = _lib.stream_ptr()
    x = grid.tensor
    n = grid.dims.count
    # The range / finite scan runs inside every call (a device Grid may have
    # been updated in place since construction; the reference recomputes
    # value_range per compress, tuning.py:46), with a per-call ctl record.
    range_done = False
    ctl = _lib.DeviceCtl()
    if alpha is not None:
        a = float(alpha)
    elif mode == "rel":
        a = compute_alpha(float(eb))
    else:
        # abs mode: alpha follows eb / range (tuning.py:102-104); alpha ** k is
        # CPython pow, so the range comes back to the host first.
        if not range_done:
            _lib.check(lib.cszi_ctl_init(ctl.ptr, st), "ctl_init")
            _lib.check(lib.cszi_range(_lib.ptr(x), n, ctl.ptr, st), "range")
            range_done = True
        c0 = ctl.fetch()
        if c0.first_nonfinite != 2**64 - 1:
            raise NonFiniteValue(int(c0.first_nonfinite))
        rng = key_to_float(c0.vmax_key) - key_to_float(c0.vmin_key)
        eb_abs = float(eb)
        a = compute_alpha(eb_abs / rng if rng > 0 else eb_abs)
    dev_pass2 = 1 if (pass2 and codec_enc is None) else 0
    worst = _caps_hint.get(n, False)
    while True:
        params, geom, caps, ws_bytes, pcap = _compress_prep(
            grid.dims.extents, layout, mode == "rel", float(eb), R, a, variants, dim_order,
            bool(exact), worst)
        ws = _lib.WS.get(ws_bytes, "compress")
        # the graph writes a per-stream staging buffer (stable pointers: a
        # fresh capacity-sized buffer per call gave the replayed graph a new
        # argument set whenever the allocator handed out another address);
        # the archive gets its own exact-length copy below
        pay = _lib.WS.get(pcap, "payload")
        _lib.check(lib.cszi_compress(_lib.ptr(x), ctypes.byref(geom), ctypes.byref(params),
                                     ctypes.byref(caps), dev_pass2, 1 if range_done else 0,
                                     _lib.ptr(pay), _lib.ptr(ws), ws.numel(), ctl.ptr, st),
                   "compress")
        c = ctl.fetch()
        if c.flags & _lib.F_CAPACITY and not worst:
            worst = True
            _caps_hint[n] = True
            range_done = True  # ctl keeps the range of x
            continue
        break
    if c.flags & _lib.F_NONFINITE:
        raise NonFiniteValue(int(c.first_nonfinite))
    grid._mark_finite()
    if c.flags & _lib.F_EB_NONPOSITIVE:
        raise Inconsistent("absolute error bound must be positive")
    if c.flags & _lib.F_EMPTY_HISTOGRAM:
        raise EmptyHistogram("cannot build a codebook from all-zero counts")
    if c.flags & _lib.F_LENGTH_OVERFLOW:
        raise LengthOverflow("a symbol would need more than 32 bits")
    if c.flags & _lib.F_CAPACITY:
        raise RuntimeError("compress: output capacity exceeded at worst-case sizing")
    na = count_anchors(grid.dims, layout.anchor_stride)
    sec = (4 * na, 2 * R, (int(c.bits) + 7) // 8, 8 + 12 * int(c.n_outliers))
    payload = pay[: int(c.payload_len)].clone()  # stream-ordered before the next call's graph
    if codec_enc is not None:
        raw = payload.cpu().numpy().tobytes()
        payload = bytes(codec_enc(raw))
    plen = len(payload) if isinstance(payload, bytes) else payload.numel()
    header = pack_header(rank, PREDICTOR_INTERP, _MODE_IDS[mode], bool(pass2), int(pass2_codec),
                         ctl_variants(c, rank), ctl_order(c, rank), R, layout.anchor_stride,
                         grid.dims.extents, float(eb), float(c.eb_abs), a, sec, plen)
    return DeviceArchive(header=header, payload=payload)


def _compress_lorenzo(grid: Grid, eb: float, mode: str, pass2: bool, pass2_codec: int,
                      quant_radius: int) -> DeviceArchive:
    """pipeline.py:123-150: value_range -> eb_abs -> the Lorenzo recurrence
    -> sections (no anchors) -> pass-2, one libcszi call on the GPU."""
    R = int(quant_radius)
    if R < 2:
        raise Inconsistent("quantizer radius must be at least 2")
    if 2 * R > _MAX_BINS:
        raise NotImplementedError(f"quant_radius {R} exceeds the GPU codebook limit")
    codec_enc = None
    if pass2 and pass2_codec != DEFAULT_CODEC:
        codec_enc = lookup(pass2_codec)[0]
    _lib.require_cuda()
    lib = _lib.load()
    st = _lib.stream_ptr()
    x = grid.tensor
    n = grid.dims.count
    rank = grid.dims.rank
    geom = make_geom(grid.dims.extents, default_layout(rank))
    ctl = _lib.DeviceCtl()
    dev_pass2 = 1 if (pass2 and codec_enc is None) else 0
    worst = _caps_hint.get(("lz", n), False)
    while True:
        caps = _caps_for(n, worst)
        ws = _lib.WS.get(int(lib.cszi_compress_lorenzo_workspace_size(ctypes.byref(geom), R,
                                                                      ctypes.byref(caps))),
                         "compress_lz")
        pay = _payload_buf(int(lib.cszi_payload_capacity(ctypes.byref(geom), R,
                                                         ctypes.byref(caps))))
        _lib.check(lib.cszi_compress_lorenzo(_lib.ptr(x), ctypes.byref(geom),
                                             1 if mode == "rel" else 0, float(eb), R,
                                             ctypes.byref(caps), dev_pass2, _lib.ptr(pay),
                                             _lib.ptr(ws), ws.numel(), ctl.ptr, st),
                   "compress_lorenzo")
        c = ctl.fetch()
        if c.flags & _lib.F_CAPACITY and not worst:
            worst = True
            _caps_hint[("lz", n)] = True
            continue
        break
    if c.flags & _lib.F_NONFINITE:
        raise NonFiniteValue(int(c.first_nonfinite))
    grid._mark_finite()
    if c.flags & _lib.F_EMPTY_HISTOGRAM:
        raise EmptyHistogram("cannot build a codebook from all-zero counts")
    if c.flags & _lib.F_LENGTH_OVERFLOW:
        raise LengthOverflow("a symbol would need more than 32 bits")
    if c.flags & _lib.F_CAPACITY:
        raise RuntimeError("compress: output capacity exceeded at worst-case sizing")
    sec = (0, 2 * R, (int(c.bits) + 7) // 8, 8 + 12 * int(c.n_outliers))
    payload = pay[: int(c.payload_len)]
    if codec_enc is not None:
        payload = bytes(codec_enc(payload.cpu().numpy().tobytes()))
    plen = len(payload) if isinstance(payload, bytes) else payload.numel()
    header = pack_header(rank, PREDICTOR_LORENZO, _MODE_IDS[mode], bool(pass2), int(pass2_codec),
                         (0,) * rank, tuple(range(rank)), R, 0, grid.dims.extents, float(eb),
                         float(c.eb_abs), 1.0, sec, plen)
    return DeviceArchive(header=header, payload=payload)


def compress(grid: Grid, eb: float, mode: str = "rel", predictor: str = "interp",
             pass2: bool = True, pass2_codec: int = DEFAULT_CODEC, alpha: float = None,
             variants=None, dim_order=None, quant_radius: int = 512,
             threads: int = None) -> bytes:
    """Compress a grid to archive bytes (pipeline.py:66-156), on the GPU."""
    return compress_device(grid, eb, mode, predictor, pass2, pass2_codec, alpha, variants,
                           dim_order, quant_radius, threads).to_bytes()


# ---------------------------------------------------------------------------
# decompress
# ---------------------------------------------------------------------------

def _layout_for(rank: int, stride: int) -> ChunkLayout:
    """pipeline.py:159-163."""
    default = default_layout(rank)
    if stride == default.anchor_stride:
        return default
    return ChunkLayout(anchor_stride=stride, rank=rank, super_chunk_extents=(stride,) * rank)


def _split_input(data):
    """-> (header bytes, device payload tensor or None, host payload bytes or None, total)."""
    t = _lib.torch()
    if isinstance(data, DeviceArchive):
        if isinstance(data.payload, bytes):
            return data.header, None, data.payload, len(data)
        return data.header, data.payload, None, len(data)
    if isinstance(data, t.Tensor):
        d = data.view(t.uint8).reshape(-1)
        head = d[:HEADER_SIZE].cpu().numpy().tobytes()
        return head, d[HEADER_SIZE:], None, d.numel()
    b = bytes(data)
    return b[:HEADER_SIZE], None, b[HEADER_SIZE:], len(b)


def _host_checks(h, dims: Dims):
    """Checks the reference performs on the host side, in its order, returning
    the first failure (exception instance) or None plus the layout."""
    if h.predictor != PREDICTOR_INTERP:
        return Corrupt(f"unknown predictor id {h.predictor}"), None
    try:
        layout = _layout_for(h.rank, h.anchor_stride)
    except Exception as e:  # InvalidStride / Inconsistent
        return e, None
    expected = count_anchors(dims, h.anchor_stride)
    if h.sec_lens[0] % 4:
        return ValueError("buffer size must be a multiple of element size"), None
    if h.sec_lens[0] // 4 != expected:
        return MalformedSection(
            f"anchor section holds {h.sec_lens[0] // 4} values, lattice needs {expected}"
        ), None
    if sorted(h.dim_order) != list(range(h.rank)):
        return Inconsistent(f"dim_order {h.dim_order} is not a permutation"), None
    if h.quant_radius < 2:
        return Inconsistent("quantizer radius must be at least 2"), None
    if not h.eb_abs > 0:
        return Inconsistent("absolute error bound must be positive"), None
    if any(v not in (0, 1) for v in h.variants):
        return KeyError(next(v for v in h.variants if v not in (0, 1))), None
    if 2 * h.quant_radius > _MAX_BINS:
        return NotImplementedError(f"quant_radius {h.quant_radius} exceeds the GPU limit"), None
    return None, layout


def _raise_device_flags(c, n: int) -> None:
    f = c.flags
    if f & _lib.F_P2_CORRUPT:
        raise Corrupt("literal run overruns the encoded stream")
    if f & _lib.F_P2_LENGTH:
        raise LengthMismatch("sections total does not match the header")
    if f & _lib.F_LENGTH_OVERFLOW:
        raise LengthOverflow("stored code length exceeds 32 bits")
    if f & _lib.F_TRUNCATED:
        raise TruncatedStream(f"bitstream ended before {n} codes were decoded")
    if f & (_lib.F_OUTLIER_COUNT | _lib.F_OUTLIER_ORDER):
        raise MalformedSection("outlier section is malformed")


def _validate_only(h, d_payload, dev_pass2: bool, dims: Dims, host_err) -> None:
    """Slow path for archives that fail a host-side check: reproduce the
    errors the reference raises before reaching that check, then raise it."""
    from .huffman import Codebook, decode_device, _canonical_tables
    from .pass2 import decode_device as p2_decode

    t = _lib.torch()
    raw_len = sum(h.sec_lens)
    if dev_pass2:
        raw, m = p2_decode(d_payload, d_payload.numel())
        if m != raw_len:
            raise LengthMismatch(f"sections total {m} bytes, header says {raw_len}")
    else:
        raw = d_payload
    s0, s1, s2, s3 = h.sec_lens
    if s1 != 2 * h.quant_radius:
        raise MalformedSection(f"codebook holds {s1} lengths for radius {h.quant_radius}")
    lengths = raw[s0:s0 + s1].cpu().numpy()
    if lengths.size and int(lengths.max()) > 32:
        raise LengthOverflow("stored code length exceeds 32 bits")
    _, tables = _canonical_tables(lengths)
    out = t.empty(max(dims.count, 1), dtype=t.int32, device="cuda")
    decode_device(raw[s0 + s1:s0 + s1 + s2], s2, dims.count, h.quant_radius, tables, out,
                  int(lengths.max(initial=1)) or 1)
    from .archive import expand_outliers

    expand_outliers(raw[s0 + s1 + s2:s0 + s1 + s2 + s3].cpu().numpy().tobytes())
    raise host_err


def decompress_device(data, threads: int = None, slab=None):
    """decompress() returning a Grid whose data stays in device memory.

    Extension (multi-GPU): ``slab=(z0, z1)`` decodes only the
    z-slab shard [z0, z1) of a 3-D default-layout archive -- the Huffman
    stream is synchronised over its whole length but only the slab's symbol
    window (plus the closing halo plane) is decoded -- and returns the
    (z1 - z0, ny, nx) float32 CUDA tensor of those planes."""
    thread_count(threads)
    t = _lib.require_cuda()
    lib = _lib.load()
    head, d_payload, h_payload, total = _split_input(data)
    key = (head, total, None if slab is None else (int(slab[0]), int(slab[1])))
    plan = _dplan_cache.get(key)
    if plan is not None:
        # a header seen before: every host-side check passed and the launch
        # arguments are known (they depend on the header and length alone;
        # only archives with the built-in pass-2 codec or none are cached)
        if d_payload is None:
            d_payload = _lib.to_device_u8(h_payload)
        return _decompress_launch(lib, t, d_payload, *plan)
    h = unpack_header(head, total)
    dev_pass2 = bool(h.pass2)
    if h.pass2 and h.pass2_codec != DEFAULT_CODEC:
        dec = lookup(h.pass2_codec)[1]
        if h_payload is None:
            h_payload = d_payload.cpu().numpy().tobytes()
        h_payload = bytes(dec(h_payload))
        d_payload = None
        dev_pass2 = False
    if d_payload is None:
        d_payload = _lib.to_device_u8(h_payload)
    raw_len = sum(h.sec_lens)
    if dev_pass2 and raw_len > 128 * d_payload.numel():
        # a zero-run control byte expands to at most 128 bytes (pass2.py:30-67):
        # a header claiming more cannot match, so fail before sizing buffers
        raise LengthMismatch(f"sections total {raw_len} bytes exceeds what a "
                             f"{d_payload.numel()}-byte pass-2 stream can hold")
    if not dev_pass2 and d_payload.numel() != raw_len:
        raise LengthMismatch(f"sections total {d_payload.numel()} bytes, header says {raw_len}")
    dims = Dims(h.extents)
    n = dims.count
    if h.predictor == PREDICTOR_LORENZO:
        if slab is not None:
            raise NotImplementedError("slab decompress needs an interp archive")
        return _decompress_lorenzo(h, d_payload, dev_pass2, dims)
    host_err, layout = _host_checks(h, dims)
    if host_err is None and h.sec_lens[1] != 2 * h.quant_radius:
        host_err = MalformedSection(
            f"codebook holds {h.sec_lens[1]} lengths for radius {h.quant_radius}")
    if host_err is not None:
        _validate_only(h, d_payload, dev_pass2, dims, host_err)
    geom = make_geom(h.extents, layout)
    out_n = n
    if slab is not None:
        z0, z1 = (int(v) for v in slab)
        if h.rank != 3 or layout.anchor_stride != 8 or layout.super_chunk_extents != (8, 8, 32):
            raise NotImplementedError("slab decompress needs a 3-D default-layout archive")
        nz = h.extents[0]
        if not (0 <= z0 < z1 <= nz) or z0 % 8 or (z1 % 8 and z1 != nz):
            # a slab is a run of whole 8-plane tiles: its last tile's closing
            # plane (z1, or nz - 1) is decoded as the halo; an unaligned z1
            # would cut a tile the reconstructor stores in full
            raise ValueError(f"slab [{z0}, {z1}) must start and end on anchor planes "
                             f"(multiples of 8, or {nz}) inside [0, {nz}]")
        geom.slab[0], geom.slab[1] = z0, z1
        out_n = (z1 - z0) * h.extents[1] * h.extents[2]
    plan = plan_levels(layout.anchor_stride, h.eb_abs, h.alpha)
    leb = (ctypes.c_double * _lib.MAX_LEVELS)(*[s.eb for s in plan.levels])
    pad = 3 - h.rank
    var = (ctypes.c_int32 * 3)(*((0,) * pad + h.variants))
    order = (ctypes.c_int32 * 3)(*(tuple(pad + d for d in h.dim_order) + (0,) * pad))
    sec = (ctypes.c_uint64 * 4)(*h.sec_lens)
    R = h.quant_radius
    plen = d_payload.numel()
    ws_bytes = int(lib.cszi_decompress_workspace_size(ctypes.byref(geom), R, sec, plen))
    shape = None if slab is None else (slab[1] - slab[0], h.extents[1], h.extents[2])
    args = (dev_pass2, sec, geom, R, leb, len(plan.levels), var, order, ws_bytes, out_n, n, dims,
            shape)
    if h.pass2_codec == DEFAULT_CODEC or not h.pass2:
        if len(_dplan_cache) > 256:
            _dplan_cache.clear()
        _dplan_cache[key] = args
    return _decompress_launch(lib, t, d_payload, *args)


_dplan_cache = {}


def _decompress_launch(lib, t, d_payload, dev_pass2, sec, geom, R, leb, nlev, var, order,
                       ws_bytes, out_n, n, dims, shape):
    """cszi_decompress with prepared arguments; device flags -> exceptions."""
    y = t.empty(out_n, dtype=t.float32, device="cuda")
    ctl = _lib.DeviceCtl()
    st = _lib.stream_ptr()
    plen = d_payload.numel()
    ws = _lib.WS.get(ws_bytes, "decompress")
    for table_mode in (0, 1):
        _lib.check(lib.cszi_decompress(_lib.ptr(d_payload), plen, 1 if dev_pass2 else 0, sec,
                                       ctypes.byref(geom), R, leb, nlev, var, order,
                                       table_mode, _lib.ptr(y), _lib.ptr(ws), ws.numel(),
                                       ctl.ptr, st), "decompress")
        c = ctl.fetch()
        if table_mode == 0 and c.scratch[1] != 0:
            continue
        break
    _raise_device_flags(c, n)
    if c.flags & _lib.F_OUTLIER_INDEX:
        raise IndexError("outlier index out of bounds for the grid")
    if shape is not None:
        return y.view(*shape)
    return Grid.wrap_device(dims, y)


def _decompress_lorenzo(h, d_payload, dev_pass2: bool, dims: Dims) -> Grid:
    """pipeline.py:172-179, 202-203: codebook, Huffman decode, outliers, then
    the Lorenzo replay (lorenzo.py:36-53) on the GPU."""
    lib = _lib.load()
    t = _lib.torch()
    n = dims.count
    if h.sec_lens[1] != 2 * h.quant_radius:
        raise MalformedSection(
            f"codebook holds {h.sec_lens[1]} lengths for radius {h.quant_radius}")
    if h.quant_radius < 2 or 2 * h.quant_radius > _MAX_BINS:
        raise NotImplementedError(f"quant_radius {h.quant_radius} is not supported on the GPU")
    geom = make_geom(h.extents, default_layout(h.rank))
    sec = (ctypes.c_uint64 * 4)(*h.sec_lens)
    R = h.quant_radius
    y = t.empty(n, dtype=t.float32, device="cuda")
    ctl = _lib.DeviceCtl()
    st = _lib.stream_ptr()
    plen = d_payload.numel()
    ws = _lib.WS.get(int(lib.cszi_decompress_workspace_size(ctypes.byref(geom), R, sec, plen)),
                     "decompress")
    for table_mode in (0, 1):
        _lib.check(lib.cszi_decompress_lorenzo(_lib.ptr(d_payload), plen, 1 if dev_pass2 else 0,
                                               sec, ctypes.byref(geom), R, float(h.eb_abs),
                                               table_mode, _lib.ptr(y), _lib.ptr(ws), ws.numel(),
                                               ctl.ptr, st), "decompress_lorenzo")
        c = ctl.fetch()
        if table_mode == 0 and c.scratch[1] != 0:
            continue
        break
    _raise_device_flags(c, n)
    if c.flags & _lib.F_OUTLIER_INDEX:
        raise IndexError("outlier index out of bounds for the grid")
    return Grid.wrap_device(dims, y)


def decompress(data: bytes, threads: int = None) -> Grid:
    """Decode archive bytes back to a grid (pipeline.py:166-204), on the GPU.

    The reference wraps the result in Grid(), whose finite scan raises
    NonFiniteValue for NaN/Inf outlier or anchor values of a crafted archive;
    that scan runs on the device here before the pinned device->host copy.
    Large 3-D archives are reconstructed z-slab by z-slab, each slab's copy
    to the host running on a copy stream under the next slab's kernels."""
    thread_count(threads)
    t = _lib.require_cuda()
    head, d_payload, h_payload, total = _split_input(data)
    plan = _pipeline_slabs(unpack_header(head, total)) if total >= HEADER_SIZE else None
    if plan is None:
        g = decompress_device(data, threads)
        y = g.tensor.reshape(-1)
        bounds, plane = [(0, 1)], y.numel()
        parts = [y]
    else:
        # one upload of the payload, then one decompress_device per slab
        dims, bounds, plane = plan
        if d_payload is None:
            d_payload = _lib.to_device_u8(h_payload)
        arch = DeviceArchive(header=head, payload=d_payload)
        parts = None
    lib = _lib.load()
    ctl = _lib.DeviceCtl()
    st = _lib.stream_ptr()
    _lib.check(lib.cszi_ctl_init(ctl.ptr, st), "ctl_init")
    n = bounds[-1][1] * plane
    host = _lib.PINNED.get(4 * n).view(t.float32)
    main = t.cuda.current_stream()
    cs = _copy_stream()
    for i, (z0, z1) in enumerate(bounds):
        y = parts[i] if parts is not None else \
            decompress_device(arch, slab=(z0, z1)).reshape(-1)
        _lib.check(lib.cszi_range(_lib.ptr(y), y.numel(), ctl.ptr, st), "range")
        done = t.cuda.Event()
        done.record(main)
        cs.wait_event(done)
        with t.cuda.stream(cs):
            host[z0 * plane:z1 * plane].copy_(y, non_blocking=True)
        y.record_stream(cs)
    c = ctl.fetch()  # synchronises the compute stream
    cs.synchronize()
    if c.first_nonfinite != 2**64 - 1:
        raise NonFiniteValue(int(c.first_nonfinite))
    if plan is None:
        return Grid.wrap_host(g.dims, host.numpy())
    return Grid.wrap_host(dims, host.numpy())


_PIPE_MIN_VALUES = 1 << 25  # 128 MB: smaller fields copy back in well under a millisecond
_PIPE_SLABS = 4
_copy_streams = {}


def _copy_stream():
    t = _lib.torch()
    dev = _lib.current_device()
    s = _copy_streams.get(dev)
    if s is None:
        s = _copy_streams[dev] = t.cuda.Stream(device=dev)
    return s


def _pipeline_slabs(h):
    """(dims, z-slab bounds, plane size) when decompress() can pipeline the
    archive by slabs (3-D interp archive, default layout, built-in pass-2
    codec or none, large enough), else None."""
    if h.predictor != PREDICTOR_INTERP or h.rank != 3 or h.anchor_stride != 8:
        return None
    if h.pass2 and h.pass2_codec != DEFAULT_CODEC:
        return None
    nz, ny, nx = h.extents
    if nz * ny * nx < _PIPE_MIN_VALUES or nz < 8 * _PIPE_SLABS:
        return None
    from .distributed import slab_bounds

    bounds = [b for b in slab_bounds(nz, _PIPE_SLABS) if b[1] > b[0]]
    return Dims(h.extents), bounds, ny * nx
