"""Second lossless pass over the serialized sections (mirrors ebcomp/pass2.py).

Codec id 0 — the zero-run codec — runs on the GPU (csrc/pass2.cu):
runs of >= 2 zero bytes become controls 127 + min(128, run); every other
byte travels in literal chunks [len-1][<= 128 bytes].  Other ids are the
reference's plugin API: Python callables registered at runtime.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import Corrupt

__all__ = ["pass2_encode", "pass2_decode", "register_pass2_codec", "DEFAULT_CODEC"]

DEFAULT_CODEC = 0


def encode_device(d_in, n: int, out=None):
    """Zero-run encode of the first n bytes of a CUDA uint8 tensor.

    Returns (encoded CUDA tensor, encoded length)."""
    t = _lib.require_cuda()
    lib = _lib.load()
    cap = n + n // 128 + 16
    if out is None or out.numel() < cap:
        out = t.empty(cap, dtype=t.uint8, device="cuda")
    ws = _lib.WS.get(int(lib.cszi_pass2_encode_workspace_size(n)), "p2_enc")
    d_n = t.tensor([n], dtype=t.int64, device="cuda")
    ctl = _lib.DeviceCtl()
    st = _lib.stream_ptr()
    _lib.check(lib.cszi_ctl_init(ctl.ptr, st), "ctl_init")
    _lib.check(lib.cszi_pass2_encode(_lib.ptr(d_in), _lib.ptr(d_n), n, _lib.ptr(out),
                                     _lib.ptr(ws), ctl.ptr, st), "pass2_encode")
    c = ctl.fetch()
    return out, int(c.payload_len)


def decode_device(d_in, n: int, expected=None):
    """Zero-run decode of n bytes (CUDA tensor) -> (decoded CUDA tensor, length).

    With ``expected`` the output buffer is sized for it and a size mismatch
    is reported by the returned length; otherwise the size pass runs first."""
    t = _lib.require_cuda()
    lib = _lib.load()
    ws = _lib.WS.get(int(lib.cszi_pass2_decode_workspace_size(n)), "p2_dec")
    ctl = _lib.DeviceCtl()
    st = _lib.stream_ptr()
    if expected is None:
        _lib.check(lib.cszi_ctl_init(ctl.ptr, st), "ctl_init")
        _lib.check(lib.cszi_pass2_decode(_lib.ptr(d_in), n, None, 0, 0, _lib.ptr(ws), ctl.ptr,
                                         st), "pass2_decode(size)")
        c = ctl.fetch()
        if c.flags & _lib.F_P2_CORRUPT:
            raise Corrupt("literal run overruns the encoded stream")
        expected = int(c.raw_len)
    out = t.empty(max(int(expected), 1), dtype=t.uint8, device="cuda")
    _lib.check(lib.cszi_ctl_init(ctl.ptr, st), "ctl_init")
    _lib.check(lib.cszi_pass2_decode(_lib.ptr(d_in), n, _lib.ptr(out), int(expected), 1,
                                     _lib.ptr(ws), ctl.ptr, st), "pass2_decode")
    c = ctl.fetch()
    if c.flags & _lib.F_P2_CORRUPT:
        raise Corrupt("literal run overruns the encoded stream")
    return out, int(c.raw_len)


def _zero_run_encode(data: bytes) -> bytes:
    if not data:
        return b""
    d_in = _lib.to_device_u8(data)
    out, m = encode_device(d_in, len(data))
    return out[:m].cpu().numpy().tobytes()


def _zero_run_decode(data: bytes) -> bytes:
    if not data:
        return b""
    d_in = _lib.to_device_u8(data)
    out, m = decode_device(d_in, len(data))
    return out[:m].cpu().numpy().tobytes()


_REGISTRY = {DEFAULT_CODEC: (_zero_run_encode, _zero_run_decode)}


def register_pass2_codec(codec_id: int, encode, decode) -> None:
    """Register an alternative pass-2 codec under a nonzero id (pass2.py:92-96)."""
    if not 0 < codec_id < 256:
        raise ValueError("codec id must be in [1, 255]")
    _REGISTRY[codec_id] = (encode, decode)


def lookup(codec_id: int):
    try:
        return _REGISTRY[codec_id]
    except KeyError:
        raise Corrupt(f"pass-2 codec {codec_id} is not registered") from None


def pass2_encode(data: bytes, codec: int = DEFAULT_CODEC) -> bytes:
    return lookup(codec)[0](data)


def pass2_decode(data: bytes, codec: int = DEFAULT_CODEC) -> bytes:
    return lookup(codec)[1](data)
