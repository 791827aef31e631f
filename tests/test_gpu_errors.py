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
    # the device grid defers its finite scan to first use (grid.py:60-62)
    g = P.Grid(P.Dims((1000,)), x)
    for use in (lambda: P.compress_device(g, 1e-3), lambda: g.data, g.ensure_finite,
                lambda: P.value_range(g)):
        with pytest.raises(P.NonFiniteValue) as e:
            use()
        assert e.value.index == 123
    # abs mode reads the range back before anything else
    with pytest.raises(P.NonFiniteValue):
        P.compress(P.Grid(P.Dims((1000,)), x), 1e-3, mode="abs")


def test_pass2_section_lengths_beyond_expansion_rejected(blobs):
    """A header whose section lengths exceed what the pass-2 stream could
    expand to fails with LengthMismatch before any buffer is sized."""
    _, p2 = blobs
    b = bytearray(p2)
    # sec_lens live at offset 64 (<4s6B3B3B2I3Q3d then 5Q): inflate the bitstream
    off = struct.calcsize("<4s6B3B3B2I3Q3d") + 16
    struct.pack_into("<Q", b, off, 1 << 40)
    with pytest.raises(P.LengthMismatch):
        P.decompress(bytes(b))


def test_slab_end_must_be_tile_aligned():
    import torch

    rng = np.random.default_rng(5)
    data = smooth_field(rng, (40, 16, 32))
    arch = P.compress_device(P.Grid(P.Dims(data.shape), torch.from_numpy(data).cuda()), 1e-3)
    with pytest.raises(ValueError):
        P.decompress_device(arch, slab=(0, 12))
    with pytest.raises(ValueError):
        P.decompress_device(arch, slab=(4, 16))
    whole = P.decompress_device(arch).tensor
    assert torch.equal(P.decompress_device(arch, slab=(8, 16)), whole[8:16])
    assert torch.equal(P.decompress_device(arch, slab=(32, 40)), whole[32:40])


def test_device_grid_updated_in_place_is_rescanned():
    """A device Grid aliases its tensor; compress sees in-place updates (the
    reference recomputes the range per call)."""
    import torch

    rng = np.random.default_rng(6)
    data = smooth_field(rng, (24, 16, 32))
    x = torch.from_numpy(data).cuda()
    g = P.Grid(P.Dims(data.shape), x)
    a0 = P.compress(g, 1e-3)
    x.mul_(3.0)
    a1 = P.compress(g, 1e-3)
    assert a1 == P.compress(P.Grid(P.Dims(data.shape), data * np.float32(3.0)), 1e-3)
    assert a1 != a0
    x[3, 4, 5] = float("nan")
    with pytest.raises(P.NonFiniteValue):
        P.compress(g, 1e-3)
