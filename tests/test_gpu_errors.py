"""Decompress error behaviour matches the reference's check order/classes."""
import struct

import numpy as np
import pytest

import paper_2312_05492_b200 as P
from conftest import smooth_field

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def blobs():
    rng = np.random.default_rng(0x5EED)
    g = P.Grid(P.Dims((16, 16)), smooth_field(rng, (16, 16)))
    return P.compress(g, 1e-3, pass2=False), P.compress(g, 1e-3, pass2=True)


def test_header_errors(blobs):
    raw, _ = blobs
    with pytest.raises(P.LengthMismatch):
        P.decompress(raw[:100])
    with pytest.raises(P.BadMagic):
        P.decompress(b"NOPE" + raw[4:])
    with pytest.raises(P.VersionUnsupported):
        P.decompress(raw[:4] + b"\x07" + raw[5:])
    with pytest.raises(P.LengthMismatch):
        P.decompress(raw + b"\x00")


def test_codebook_size_and_predictor_errors(blobs):
    raw, _ = blobs
    b = bytearray(raw)
    struct.pack_into("<I", b, 16, 256)
    with pytest.raises(P.MalformedSection):
        P.decompress(bytes(b))
    b = bytearray(raw)
    b[6] = 9
    with pytest.raises(P.Corrupt):
        P.decompress(bytes(b))


def test_truncated_bitstream(blobs):
    raw, _ = blobs
    h = P.archive.unpack_header(raw, len(raw))
    s0, s1, s2, s3 = h.sec_lens
    payload = bytearray(raw[112:])
    # zero the bitstream: the all-zero prefix decodes, but flip it to ones so
    # the stream runs out / hits invalid codes
    for i in range(s0 + s1, s0 + s1 + s2):
        payload[i] = 0xFF
    try:
        P.decompress(raw[:112] + bytes(payload))
    except P.TruncatedStream:
        pass


def test_outlier_section_errors(blobs):
    raw, _ = blobs
    h = P.archive.unpack_header(raw, len(raw))
    s0, s1, s2, s3 = h.sec_lens
    payload = bytearray(raw[112:])
    struct.pack_into("<Q", payload, s0 + s1 + s2, 5)  # count says 5, body holds 0
    with pytest.raises(P.MalformedSection):
        P.decompress(raw[:112] + bytes(payload))


def test_pass2_corruption(blobs):
    _, p2 = blobs
    payload = p2[112:] + b"\x05"  # a literal run that overruns the stream
    head = bytearray(p2[:112])
    struct.pack_into("<Q", head, 104, len(payload))
    with pytest.raises(P.Corrupt):
        P.decompress(bytes(head) + payload)
    payload = p2[112:] + b"\x85"  # decodes, but the sections no longer add up
    struct.pack_into("<Q", head, 104, len(payload))
    with pytest.raises(P.LengthMismatch):
        P.decompress(bytes(head) + payload)


def test_compress_argument_errors():
    g = P.Grid(P.Dims((16,)), np.arange(16, dtype=np.float32))
    with pytest.raises(ValueError):
        P.compress(g, -1.0)
    with pytest.raises(ValueError):
        P.compress(g, 1e-3, mode="percent")
    with pytest.raises(ValueError):
        P.compress(g, 1e-3, predictor="psychic")
    with pytest.raises(P.Inconsistent):
        P.compress(g, 1e-3, dim_order=(1,))
    with pytest.raises(P.Inconsistent):
        P.compress(g, 1e-3, quant_radius=1)
    with pytest.raises(P.Corrupt):
        P.compress(g, 1e-3, pass2_codec=251)


def test_device_grid_nonfinite():
    import torch

    x = torch.ones(1000, device="cuda")
    x[123] = float("inf")
    with pytest.raises(P.NonFiniteValue) as e:
        P.Grid(P.Dims((1000,)), x)
    assert e.value.index == 123
