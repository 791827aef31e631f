"""Order-preserving float32 keys used by the device range reduction."""

import struct


def key_to_float(k: int) -> float:
    """Inverse of csrc/common.cuh float_key: key -> float32 value as a float."""
    b = (k & 0x7FFFFFFF) if (k & 0x80000000) else (~k & 0xFFFFFFFF)
    return struct.unpack("<f", struct.pack("<I", b))[0]


def float_to_key(f: float) -> int:
    b = struct.unpack("<I", struct.pack("<f", f))[0]
    return (~b & 0xFFFFFFFF) if (b & 0x80000000) else (b | 0x80000000)
