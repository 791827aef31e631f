"""Canonical Huffman coding of quantization codes (mirrors ebcomp/huffman.py).

Every stage runs in libcszi on the GPU (csrc/huffman.cu):
histogram -> cszi_histogram_i32, code lengths + canonical words ->
cszi_codebook / cszi_canonical, encode -> cszi_huff_encode_i32 (one
MSB-first stream, tile offsets by decoupled look-back), decode ->
cszi_huff_decode_i32 (self-synchronising chunked decode of the single
index-free stream; exact transfer-table fallback when chunks do not
resynchronise).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import EmptyHistogram, LengthOverflow, OutOfRange, TruncatedStream, UnknownSymbol

__all__ = [
    "MAX_CODE_LENGTH",
    "Histogram",
    "Codebook",
    "build_histogram",
    "build_codebook",
    "huffman_encode",
    "huffman_decode",
]

MAX_CODE_LENGTH = 32

# csrc/huffman.cu DecTables layout
_DT_LUT = 0
_DT_FIRST_CODE = 4096 * 4
_DT_FIRST_INDEX = _DT_FIRST_CODE + 33 * 8
_DT_COUNTS = _DT_FIRST_INDEX + 33 * 4
_DT_MAXLEN = _DT_COUNTS + 33 * 4
_DT_SORTED = _DT_MAXLEN + 8


@dataclass(frozen=True, eq=False)
class Histogram:
    """Symbol counts indexed by shifted code q + R."""

    counts: np.ndarray

    @property
    def num_bins(self) -> int:
        return int(self.counts.shape[0])

    @property
    def radius(self) -> int:
        return self.num_bins // 2

    @property
    def total(self) -> int:
        return int(self.counts.sum())


def build_histogram(codes, radius: int) -> Histogram:
    """Count codes into 2*radius bins on the GPU (huffman.py:60-74)."""
    t = _lib.require_cuda()
    lib = _lib.load()
    arr = np.ascontiguousarray(codes, dtype=np.int32).ravel()
    hist = t.zeros(2 * radius, dtype=t.int64, device="cuda")
    ctl = _lib.DeviceCtl()
    st = _lib.stream_ptr()
    _lib.check(lib.cszi_ctl_init(ctl.ptr, st), "ctl_init")
    if arr.size:
        d = t.from_numpy(arr).cuda()
        _lib.check(lib.cszi_histogram_i32(_lib.ptr(d), arr.size, radius, _lib.ptr(hist),
                                          ctl.ptr, st), "histogram")
    c = ctl.fetch()
    if c.flags & _lib.F_OUT_OF_RANGE:
        bad = arr[(arr <= -radius) | (arr >= radius)]
        raise OutOfRange(f"code {int(bad[0])} outside (-{radius}, {radius})")
    return Histogram(counts=hist.cpu().numpy().astype(np.int64))


def _canonical_tables(lengths: np.ndarray):
    """cszi_canonical: words + decode tables for stored lengths."""
    t = _lib.require_cuda()
    lib = _lib.load()
    nb = int(lengths.size)
    d_len = t.from_numpy(np.ascontiguousarray(lengths, dtype=np.uint8)).cuda()
    words = t.zeros(max(nb, 1), dtype=t.int32, device="cuda")
    tables = t.zeros(int(lib.cszi_dec_tables_size(nb)), dtype=t.uint8, device="cuda")
    ctl = _lib.DeviceCtl()
    st = _lib.stream_ptr()
    _lib.check(lib.cszi_ctl_init(ctl.ptr, st), "ctl_init")
    _lib.check(lib.cszi_canonical(_lib.ptr(d_len), nb, _lib.ptr(words), _lib.ptr(tables),
                                  ctl.ptr, st), "canonical")
    c = ctl.fetch()
    if c.flags & _lib.F_LENGTH_OVERFLOW:
        raise LengthOverflow("stored code length exceeds 32 bits")
    return words, tables


@dataclass(frozen=True, eq=False)
class Codebook:
    """Canonical codes plus the derived decoder tables (huffman.py:105-160)."""

    code_lengths: np.ndarray
    words: np.ndarray = field(repr=False, default=None)
    first_code: np.ndarray = field(repr=False, default=None)
    first_index: np.ndarray = field(repr=False, default=None)
    length_counts: np.ndarray = field(repr=False, default=None)
    sorted_symbols: np.ndarray = field(repr=False, default=None)

    @property
    def num_symbols(self) -> int:
        return int(self.code_lengths.shape[0])

    @property
    def radius(self) -> int:
        return self.num_symbols // 2

    def kraft_sum(self) -> float:
        used = self.code_lengths[self.code_lengths > 0].astype(np.float64)
        return float(np.sum(2.0 ** -used))

    @staticmethod
    def from_lengths(code_lengths) -> "Codebook":
        """Rebuild canonical codes and decode tables from lengths (GPU)."""
        lens = np.ascontiguousarray(code_lengths, dtype=np.uint8)
        if lens.size and int(lens.max()) > MAX_CODE_LENGTH:
            raise LengthOverflow("stored code length exceeds 32 bits")
        words, tables = _canonical_tables(lens)
        raw = tables.cpu().numpy()
        fc = raw[_DT_FIRST_CODE:_DT_FIRST_INDEX].view(np.uint64).astype(np.int64)
        fi = raw[_DT_FIRST_INDEX:_DT_COUNTS].view(np.uint32).astype(np.int64)
        lc = raw[_DT_COUNTS:_DT_MAXLEN].view(np.uint32).astype(np.int64)
        ncoded = int(lc.sum())
        ss = raw[_DT_SORTED:_DT_SORTED + 2 * ncoded].view(np.uint16).astype(np.int64)
        # first_code / first_index are only defined where a length is used
        fc = np.where(lc > 0, fc, 0)
        fi_ref = np.zeros(33, dtype=np.int64)
        fi_ref[lc > 0] = fi[lc > 0]
        return Codebook(
            code_lengths=lens,
            words=words.cpu().numpy().view(np.uint32)[: lens.size].copy(),
            first_code=fc,
            first_index=fi_ref,
            length_counts=lc,
            sorted_symbols=ss,
        )


def build_codebook(hist: Histogram) -> Codebook:
    """Code lengths with (freq, min symbol) tie-breaks, canonical words (GPU)."""
    t = _lib.require_cuda()
    lib = _lib.load()
    counts = np.ascontiguousarray(hist.counts, dtype=np.int64)
    nb = counts.size
    d_cnt = t.from_numpy(counts).cuda()
    d_len = t.zeros(max(nb, 1), dtype=t.uint8, device="cuda")
    d_words = t.zeros(max(nb, 1), dtype=t.int32, device="cuda")
    ctl = _lib.DeviceCtl()
    st = _lib.stream_ptr()
    _lib.check(lib.cszi_ctl_init(ctl.ptr, st), "ctl_init")
    _lib.check(lib.cszi_codebook(_lib.ptr(d_cnt), nb, _lib.ptr(d_len), _lib.ptr(d_words),
                                 ctl.ptr, st), "codebook")
    c = ctl.fetch()
    if c.flags & _lib.F_EMPTY_HISTOGRAM:
        raise EmptyHistogram("cannot build a codebook from all-zero counts")
    if c.flags & _lib.F_LENGTH_OVERFLOW:
        raise LengthOverflow(f"a symbol would need more than {MAX_CODE_LENGTH} bits")
    return Codebook.from_lengths(d_len.cpu().numpy()[:nb])


def huffman_encode(codes, codebook: Codebook) -> tuple:
    """Pack codes MSB-first on the GPU; returns (padded bytes, exact bit count)."""
    t = _lib.require_cuda()
    lib = _lib.load()
    arr = np.ascontiguousarray(codes, dtype=np.int32).ravel()
    if arr.size == 0:
        return b"", 0
    R = codebook.radius
    maxlen = int(codebook.code_lengths.max(initial=1)) or 1
    cap = ((arr.size * maxlen + 7) // 8 + 64) & ~15
    d_codes = t.from_numpy(arr).cuda()
    d_len = t.from_numpy(np.ascontiguousarray(codebook.code_lengths, dtype=np.uint8)).cuda()
    d_words = t.from_numpy(np.ascontiguousarray(codebook.words, dtype=np.uint32).view(np.int32)).cuda()
    out = t.zeros(cap, dtype=t.uint8, device="cuda")
    ws = _lib.WS.get(int(lib.cszi_huff_encode_workspace_size(arr.size)), "huff_enc")
    ctl = _lib.DeviceCtl()
    st = _lib.stream_ptr()
    _lib.check(lib.cszi_ctl_init(ctl.ptr, st), "ctl_init")
    _lib.check(lib.cszi_huff_encode_i32(_lib.ptr(d_codes), arr.size, R, _lib.ptr(d_len),
                                        _lib.ptr(d_words), _lib.ptr(out), cap, _lib.ptr(ws),
                                        ctl.ptr, st), "huffman_encode")
    c = ctl.fetch()
    if c.flags & _lib.F_UNKNOWN_SYMBOL:
        syms = arr.astype(np.int64) + R
        bad = (syms < 0) | (syms >= codebook.num_symbols)
        bad |= ~bad & (codebook.code_lengths[np.clip(syms, 0, codebook.num_symbols - 1)] == 0)
        raise UnknownSymbol(f"code {int(arr[np.argmax(bad)])} has no codebook entry")
    nbits = int(c.bits)
    return out[: (nbits + 7) // 8].cpu().numpy().tobytes(), nbits


def decode_device(d_stream, nbytes: int, n: int, radius: int, d_tables, out, max_len: int):
    """Decode n int32 codes into `out` (CUDA tensor); raises TruncatedStream."""
    lib = _lib.load()
    ctl = _lib.DeviceCtl()
    st = _lib.stream_ptr()
    for table_mode in (0, 1):
        ws = _lib.WS.get(int(lib.cszi_huff_decode_workspace_size(nbytes, table_mode)), "huff_dec")
        _lib.check(lib.cszi_ctl_init(ctl.ptr, st), "ctl_init")
        _lib.check(lib.cszi_huff_decode_i32(_lib.ptr(d_stream), nbytes, n, radius,
                                            _lib.ptr(d_tables), _lib.ptr(out), table_mode,
                                            max_len, _lib.ptr(ws), ctl.ptr, st),
                   "huffman_decode")
        c = ctl.fetch()
        if table_mode == 0 and c.scratch[1] != 0:
            continue  # chunks did not resynchronise: exact table decode
        break
    if c.flags & _lib.F_TRUNCATED:
        raise TruncatedStream(f"bitstream ended before {n} codes were decoded")


def huffman_decode(stream: bytes, codebook: Codebook, n: int) -> np.ndarray:
    """Decode exactly n codes on the GPU; inverse of huffman_encode."""
    t = _lib.require_cuda()
    if n == 0:
        return np.empty(0, dtype=np.int32)
    _, tables = _canonical_tables(np.ascontiguousarray(codebook.code_lengths, dtype=np.uint8))
    d_stream = _lib.to_device_u8(stream)
    out = t.empty(n, dtype=t.int32, device="cuda")
    maxlen = int(codebook.code_lengths.max(initial=1)) or 1
    decode_device(d_stream, len(stream), n, codebook.radius, tables, out, maxlen)
    return out.cpu().numpy()
