"""ctypes binding of libcszi.so (include/cszi.h) plus device-buffer plumbing.

The shared library is the product: every compute stage of the compress /
decompress path runs in it on the GPU.  This module fails loudly when the
library is missing or no CUDA device is present — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import sys
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CSZI_LIB") or os.path.join(_HERE, "libcszi.so")  # override: A/B runs
CSRC = os.path.join(_HERE, "csrc")

MAX_LEVELS = 16
SAMPLE_WORDS = 64 * 3 * 5

# status codes (include/cszi.h)
OK = 0
E_NONFINITE = -1
E_INCONSISTENT = -2
E_LENGTH_OVERFLOW = -3
E_EMPTY_HISTOGRAM = -4
E_TRUNCATED = -5
E_CORRUPT = -6
E_MALFORMED = -7
E_UNKNOWN_SYMBOL = -8
E_OUT_OF_RANGE = -9
E_LENGTH_MISMATCH = -10
E_INVALID_ARG = -20
E_UNSUPPORTED = -21
E_CAPACITY = -22
E_CUDA = -30

# ctl flag bits
F_NONFINITE = 1 << 0
F_EB_NONPOSITIVE = 1 << 1
F_LENGTH_OVERFLOW = 1 << 2
F_EMPTY_HISTOGRAM = 1 << 3
F_TRUNCATED = 1 << 4
F_P2_CORRUPT = 1 << 5
F_P2_LENGTH = 1 << 6
F_OUTLIER_COUNT = 1 << 7
F_OUTLIER_ORDER = 1 << 8
F_OUTLIER_INDEX = 1 << 9
F_CAPACITY = 1 << 10
F_UNKNOWN_SYMBOL = 1 << 11
F_OUT_OF_RANGE = 1 << 31


class Geom(ctypes.Structure):
    _fields_ = [
        ("rank", ctypes.c_int32),
        ("pad_", ctypes.c_int32),
        ("ext", ctypes.c_int64 * 3),
        ("stride", ctypes.c_int64),
        ("tile", ctypes.c_int64 * 3),
        ("slab", ctypes.c_int64 * 2),
    ]


class Params(ctypes.Structure):
    _fields_ = [
        ("mode_rel", ctypes.c_int32),
        ("radius", ctypes.c_int32),
        ("eb", ctypes.c_double),
        ("have_alpha", ctypes.c_int32),
        ("have_variants", ctypes.c_int32),
        ("have_order", ctypes.c_int32),
        ("pad_", ctypes.c_int32),
        ("alpha", ctypes.c_double),
        ("alpha_pow", ctypes.c_double * MAX_LEVELS),
        ("variant", ctypes.c_int32 * 3),
        ("order", ctypes.c_int32 * 3),
        ("exact", ctypes.c_int32),
        ("pad2_", ctypes.c_int32),
    ]


class Caps(ctypes.Structure):
    _fields_ = [("bits_cap", ctypes.c_uint64), ("outlier_cap", ctypes.c_uint64)]


class Ctl(ctypes.Structure):
    _fields_ = [
        ("vmin_key", ctypes.c_uint32),
        ("vmax_key", ctypes.c_uint32),
        ("first_nonfinite", ctypes.c_uint64),
        ("vmin", ctypes.c_double),
        ("vmax", ctypes.c_double),
        ("rng", ctypes.c_double),
        ("eb_abs", ctypes.c_double),
        ("alpha", ctypes.c_double),
        ("level_eb", ctypes.c_double * MAX_LEVELS),
        ("inv_e2", ctypes.c_double * MAX_LEVELS),
        ("err_sum", (ctypes.c_double * 2) * 3),
        ("sample_count", ctypes.c_int64 * 3),
        ("variant", ctypes.c_int32 * 3),
        ("order", ctypes.c_int32 * 3),
        ("nlev", ctypes.c_int32),
        ("radius", ctypes.c_int32),
        ("bits", ctypes.c_uint64),
        ("n_outliers", ctypes.c_uint64),
        ("raw_len", ctypes.c_uint64),
        ("payload_len", ctypes.c_uint64),
        ("decoded_symbols", ctypes.c_uint64),
        ("flags", ctypes.c_uint32),
        ("max_len", ctypes.c_uint32),
        ("scratch", ctypes.c_uint64 * 8),
    ]


CTL_BYTES = ctypes.sizeof(Ctl)

# symbol table: name -> (restype, argtypes)
_vp = ctypes.c_void_p
_u64 = ctypes.c_uint64
_i32 = ctypes.c_int32
_u32 = ctypes.c_uint32
_SIGS = {
    "cszi_version": (ctypes.c_char_p, []),
    "cszi_abi_sizes": (None, [_vp]),
    "cszi_launch_count": (_u64, []),
    "cszi_compress_workspace_size": (_u64, [_vp, _i32, _vp]),
    "cszi_payload_capacity": (_u64, [_vp, _i32, _vp]),
    "cszi_compress": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _u64, _vp, _vp]),
    "cszi_decompress_workspace_size": (_u64, [_vp, _i32, _vp, _u64]),
    "cszi_decompress": (
        ctypes.c_int,
        [_vp, _u64, _i32, _vp, _vp, _i32, _vp, _i32, _vp, _vp, _i32, _vp, _vp, _u64, _vp, _vp],
    ),
    "cszi_compress_lorenzo_workspace_size": (_u64, [_vp, _i32, _vp]),
    "cszi_compress_lorenzo": (
        ctypes.c_int,
        [_vp, _vp, _i32, ctypes.c_double, _i32, _vp, _i32, _vp, _vp, _u64, _vp, _vp],
    ),
    "cszi_decompress_lorenzo": (
        ctypes.c_int,
        [_vp, _u64, _i32, _vp, _vp, _i32, ctypes.c_double, _i32, _vp, _vp, _u64, _vp, _vp],
    ),
    "cszi_lorenzo_predict": (ctypes.c_int, [_vp, _vp, ctypes.c_double, _i32, _vp, _vp, _vp, _vp]),
    "cszi_lorenzo_reconstruct": (
        ctypes.c_int, [_vp, _vp, _vp, _u64, _vp, ctypes.c_double, _i32, _vp, _vp]
    ),
    "cszi_ctl_init": (ctypes.c_int, [_vp, _vp]),
    "cszi_ctl_fetch": (ctypes.c_int, [_vp, _vp, _vp]),
    "cszi_range": (ctypes.c_int, [_vp, _u64, _vp, _vp]),
    "cszi_scan_field": (ctypes.c_int, [_vp, _u64, _vp, _vp]),
    "cszi_tune": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "cszi_predict": (ctypes.c_int, [_vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp]),
    "cszi_reconstruct": (
        ctypes.c_int, [_vp, _vp, _vp, _vp, _u64, _vp, _i32, _vp, _i32, _vp, _vp, _vp, _vp]
    ),
    "cszi_gather_anchors": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "cszi_interp_level": (
        ctypes.c_int,
        [_vp, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_int64, ctypes.c_double, _vp, _vp, _i32, _i32,
         _vp],
    ),
    "cszi_slab_anchor_count": (_u64, [_vp]),
    "cszi_shard_scan": (ctypes.c_int, [_vp, _u64, _u64, _vp, _vp, _vp, _vp, _vp]),
    "cszi_shard_set_range": (ctypes.c_int, [_vp, _vp, _vp]),
    "cszi_shard_piece_bits": (ctypes.c_int, [_vp, _vp, _i32, _vp, _vp]),
    "cszi_shard_counts": (ctypes.c_int, [_vp, _vp, _vp]),
    "cszi_decompress_prologue": (ctypes.c_int, [_vp, _u64, _i32, _vp, _vp, _i32, _vp, _u64, _vp,
                                                _vp]),
    "cszi_huff_chunks": (_u64, [_u64]),
    "cszi_p2d_chunks": (_u64, [_u64]),
    "cszi_p2d_resolve_scratch_size": (_u64, [_u64]),
    "cszi_p2d_tables": (ctypes.c_int, [_vp, _u64, _u64, _u64, _vp, _vp, _vp]),
    "cszi_p2d_resolve": (ctypes.c_int, [_vp, _vp, _u64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "cszi_p2d_expand": (ctypes.c_int, [_vp, _u64, _vp, _vp, _vp, _u64, _u64, _vp, _u64, _vp,
                                       _vp]),
    "cszi_decompress_raw_offset": (_u64, [_vp, _i32, _vp, _u64]),
    "cszi_decompress_prologue_raw": (ctypes.c_int, [_u64, _vp, _vp, _i32, _vp, _u64, _vp, _vp]),
    "cszi_find_cuts": (ctypes.c_int, [_vp, _u64, _u64, _vp, _vp]),
    "cszi_decompress_sync_range": (ctypes.c_int, [_vp, _u64, _i32, _vp, _vp, _i32, _u64, _u64,
                                                  _u64, _vp, _vp, _vp, _vp, _vp, _u64, _vp, _vp]),
    "cszi_decompress_write_window": (ctypes.c_int, [_vp, _u64, _i32, _vp, _vp, _i32, _vp, _vp,
                                                    _vp, _vp, _u64, _vp, _vp]),
    "cszi_decompress_epilogue": (ctypes.c_int, [_vp, _u64, _i32, _vp, _vp, _i32, _vp, _i32, _vp,
                                                _vp, _vp, _vp, _u64, _vp, _vp]),
    "cszi_shard_assemble": (ctypes.c_int, [_i32, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp,
                                           _vp, _i32, _vp, _u64, _vp, _vp, _u64, _vp, _vp]),
    "cszi_sample_gather": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "cszi_tune_from_samples": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "cszi_encode_sym_workspace_size": (_u64, [_u64]),
    "cszi_encode_sym": (
        ctypes.c_int,
        [_vp, _u64, _i32, _vp, _vp, _vp, _u64, _vp, _u64, _vp, _vp, _u64, _vp, _vp, _vp],
    ),
    "cszi_encode_sym_at": (
        ctypes.c_int,
        [_vp, _u64, _i32, _vp, _vp, _vp, _u64, ctypes.c_uint32, _vp, _u64, _vp, _vp, _u64, _vp,
         _vp, _vp],
    ),
    "cszi_encode_sym_nz": (
        ctypes.c_int,
        [_vp, _u64, _i32, _vp, _vp, _vp, _u64, ctypes.c_uint32, _vp, _u64, _vp, _vp, _u64, _vp,
         _vp, _vp, _vp, _vp],
    ),
    "cszi_predict_nz": (ctypes.c_int, [_vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "cszi_concat_bits": (ctypes.c_int, [_vp, _u64, _vp, _u64, _vp]),
    "cszi_pack_outliers": (ctypes.c_int, [_vp, _vp, _u64, _vp, _vp]),
    "cszi_histogram_i32": (ctypes.c_int, [_vp, _u64, _i32, _vp, _vp, _vp]),
    "cszi_codebook": (ctypes.c_int, [_vp, _u32, _vp, _vp, _vp, _vp]),
    "cszi_dec_tables_size": (_u64, [_u32]),
    "cszi_canonical": (ctypes.c_int, [_vp, _u32, _vp, _vp, _vp, _vp]),
    "cszi_huff_encode_workspace_size": (_u64, [_u64]),
    "cszi_huff_encode_i32": (ctypes.c_int, [_vp, _u64, _i32, _vp, _vp, _vp, _u64, _vp, _vp, _vp]),
    "cszi_huff_decode_workspace_size": (_u64, [_u64, _i32]),
    "cszi_huff_decode_i32": (
        ctypes.c_int, [_vp, _u64, _u64, _i32, _vp, _vp, _i32, _i32, _vp, _vp, _vp]
    ),
    "cszi_pass2_encode_workspace_size": (_u64, [_u64]),
    "cszi_pass2_encode": (ctypes.c_int, [_vp, _vp, _u64, _vp, _vp, _vp, _vp]),
    "cszi_pass2_decode_workspace_size": (_u64, [_u64]),
    "cszi_pass2_decode": (ctypes.c_int, [_vp, _u64, _vp, _u64, _i32, _vp, _vp, _vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def build(force: bool = False) -> None:
    """Compile libcszi.so in-tree for sm_100a (nvcc; cross-compiles without a GPU)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", CSRC, "-j8"], check=True)


def load():
    """Load libcszi.so and bind every entry point of include/cszi.h."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with paper_2312_05492_b200._lib.build() "
                    "(there is no CPU fallback)"
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            sizes = (ctypes.c_uint64 * 4)()
            lib.cszi_abi_sizes(sizes)
            mine = (ctypes.sizeof(Geom), ctypes.sizeof(Params), ctypes.sizeof(Caps), CTL_BYTES)
            if tuple(sizes) != mine:
                raise ImportError(f"cszi ABI mismatch: library {tuple(sizes)} vs binding {mine}")
            _lib = lib
    return _lib


# ---------------------------------------------------------------------------
# device plumbing (torch: allocator, streams)
# ---------------------------------------------------------------------------

_T = None
_CUDA_OK = False
_GET_RAW = None


def torch():
    global _T
    if _T is None:
        import torch as _t

        _T = _t
    return _T


def require_cuda():
    """torch, after checking once that a CUDA device is usable (every entry
    point calls this first: there is no CPU fallback)."""
    global _CUDA_OK, _GET_RAW
    t = torch()
    if not _CUDA_OK:
        if not t.cuda.is_available():
            raise RuntimeError(
                "paper_2312_05492_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists"
            )
        t.cuda.init()
        _GET_RAW = getattr(t._C, "_cuda_getCurrentRawStream", None)
        _CUDA_OK = True
    return t


def current_device() -> int:
    """torch.cuda.current_device() without its per-call lazy-init checks."""
    return require_cuda()._C._cuda_getDevice()


def _raw_stream() -> int:
    """Handle of the current CUDA stream of the current device (the raw
    accessor is ~10x cheaper than torch.cuda.current_stream())."""
    t = require_cuda()
    dev = t._C._cuda_getDevice()
    return _GET_RAW(dev) if _GET_RAW is not None else t.cuda.current_stream(dev).cuda_stream


def stream_ptr():
    return ctypes.c_void_p(_raw_stream())


def ptr(tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(tensor.data_ptr())


class Workspace:
    """Grow-only scratch buffers (uint8 torch tensors) keyed by (device,
    stream, purpose).  Calls on one stream are ordered, so they may share a
    buffer; calls on different streams get different buffers (a buffer
    allocated and used on one stream only is also safe to free and regrow:
    the caching allocator reuses it in that stream's order)."""

    def __init__(self):
        self._bufs = {}

    def get(self, nbytes: int, key: str = "ws"):
        t = require_cuda()
        dev = t._C._cuda_getDevice()
        k = (dev, _raw_stream(), key)
        buf = self._bufs.get(k)
        if buf is None or buf.numel() < nbytes:
            self._bufs[k] = None
            buf = t.empty(max(int(nbytes), 256), dtype=t.uint8, device=f"cuda:{dev}")
            self._bufs[k] = buf
        return buf


WS = Workspace()


class PinnedPool:
    """Pinned host buffers for results handed to the caller (decompress()
    output grids, archive bytes).  A buffer is reused once nothing outside
    the pool shares its storage (numpy arrays and views made from it hold
    the storage, so a Grid still held by the caller keeps its buffer).
    torch's caching host allocator does not reliably reuse 0.5 GB blocks,
    and a fresh cudaHostAlloc of that size costs ~80 ms.  Reuse is safe:
    every user synchronises its stream before handing the buffer out."""

    def __init__(self, per_size: int = 4):
        self._free = {}
        self._per = per_size
        self._lock = threading.Lock()

    def get(self, nbytes: int):
        t = require_cuda()
        nbytes = max(int(nbytes), 1)
        with self._lock:
            bufs = self._free.setdefault(nbytes, [])
            use = getattr(t._C, "_storage_Use_Count", None)
            for b in bufs:
                # the pool's tensor + the temporary storage object: nobody else
                if use is not None and use(b.untyped_storage()._cdata) == 2:
                    return b
            b = t.empty(nbytes, dtype=t.uint8, pin_memory=True)
            if len(bufs) < self._per:
                bufs.append(b)
            return b


PINNED = PinnedPool()


class DeviceCtl:
    """A device-resident cszi_ctl plus a pinned host mirror.

    The buffer pairs are recycled through a pool keyed by (device, stream):
    a call's first launch waits on the host allocating them otherwise.  A
    recycled pair is reused on the same stream only, so stream order keeps
    its previous user's kernels ahead of the new user's."""

    _pool = {}
    _pool_lock = threading.Lock()

    def __init__(self):
        t = require_cuda()
        self._key = (t._C._cuda_getDevice(), _raw_stream())
        with DeviceCtl._pool_lock:
            free = DeviceCtl._pool.get(self._key)
            pair = free.pop() if free else None
        if pair is None:
            pair = (t.empty(CTL_BYTES, dtype=t.uint8, device="cuda"),
                    t.empty(CTL_BYTES, dtype=t.uint8, pin_memory=True))
        self.dev, self.host = pair
        self._ptr = ctypes.c_void_p(self.dev.data_ptr())
        self._hptr = self.host.data_ptr()

    def __del__(self):
        try:
            with DeviceCtl._pool_lock:
                free = DeviceCtl._pool.setdefault(self._key, [])
                if len(free) < 64:
                    free.append((self.dev, self.host))
        except Exception:  # interpreter shutdown
            pass

    @property
    def ptr(self):
        return self._ptr

    def fetch(self) -> Ctl:
        """Copy back (stream-ordered) and synchronise; returns a Ctl struct."""
        check(load().cszi_ctl_fetch(self._ptr, ctypes.c_void_p(self._hptr), stream_ptr()),
              "ctl_fetch")
        return Ctl.from_buffer_copy(ctypes.string_at(self._hptr, CTL_BYTES))


def check(rc: int, what: str) -> None:
    if rc == OK:
        return
    if rc == E_UNSUPPORTED:
        raise NotImplementedError(f"{what}: configuration not supported by the sm_100a kernels")
    if rc == E_CUDA:
        raise RuntimeError(f"{what}: CUDA launch failure")
    raise RuntimeError(f"{what}: libcszi status {rc}")


def to_device_u8(data) -> "object":
    """bytes / numpy uint8 / torch tensor -> contiguous uint8 CUDA tensor."""
    t = require_cuda()
    if isinstance(data, t.Tensor):
        if data.dtype != t.uint8:
            data = data.view(t.uint8)
        return data.contiguous().cuda()
    if isinstance(data, np.ndarray):
        arr = np.ascontiguousarray(data).view(np.uint8).reshape(-1)
    else:
        # bytearray keeps the buffer writable (torch.from_numpy rejects
        # read-only memory with a warning); one host copy of the payload
        arr = np.frombuffer(bytearray(data), dtype=np.uint8)
    out = t.empty(max(arr.size, 1), dtype=t.uint8, device="cuda")
    if arr.size:
        if not arr.flags.writeable:
            arr = arr.copy()
        out[: arr.size].copy_(t.from_numpy(arr), non_blocking=False)
    return out[: arr.size] if arr.size else out[:0]
