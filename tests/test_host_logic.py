"""Host-side logic of the drop-in API (no GPU): header layout, tuner
decisions, level plans, lattice counts, scalar semantic definitions."""
import math
import struct

import numpy as np
import pytest

import paper_2312_05492_b200 as P
from paper_2312_05492_b200 import archive as A
from paper_2312_05492_b200._keys import float_to_key, key_to_float


def test_header_layout_offsets():
    h = A.pack_header(3, 0, 1, True, 0, (0, 1, 0), (1, 0, 2), 512, 8, (64, 65, 66), 1e-3,
                      4.9e-3, 1.5, (10, 20, 30, 40), 77)
    assert len(h) == A.HEADER_SIZE == 112
    assert h[:4] == b"CSZI" and h[4] == 1 and h[5] == 3
    assert struct.unpack_from("<I", h, 16)[0] == 512
    assert struct.unpack_from("<I", h, 20)[0] == 8
    assert struct.unpack_from("<3Q", h, 24) == (64, 65, 66)
    assert struct.unpack_from("<3d", h, 48) == (1e-3, 4.9e-3, 1.5)
    assert struct.unpack_from("<5Q", h, 72) == (10, 20, 30, 40, 77)
    hd = A.unpack_header(h + b"\0" * 77, 112 + 77)
    assert hd.extents == (64, 65, 66) and hd.variants == (0, 1, 0) and hd.dim_order == (1, 0, 2)


def test_header_checks():
    h = A.pack_header(2, 0, 1, False, 0, (0, 0), (0, 1), 512, 16, (4, 4), 1e-3, 1e-3, 1.5,
                      (0, 0, 0, 0), 0)
    with pytest.raises(P.LengthMismatch):
        A.unpack_header(h[:50], 50)
    with pytest.raises(P.BadMagic):
        A.unpack_header(b"XXXX" + h[4:], 112)
    with pytest.raises(P.VersionUnsupported):
        A.unpack_header(h[:4] + b"\x02" + h[5:], 112)
    with pytest.raises(P.Corrupt):
        A.unpack_header(h[:5] + b"\x04" + h[6:], 112)
    with pytest.raises(P.LengthMismatch):
        A.unpack_header(h + b"\0", 113)


def test_outlier_section_roundtrip_and_checks():
    pairs = [(3, 1.5), (10, -2.25), (2 ** 40, 0.125)]
    sec = A.compact_outliers(pairs)
    assert len(sec) == 8 + 12 * 3
    assert A.expand_outliers(sec) == pairs
    with pytest.raises(P.MalformedSection):
        A.expand_outliers(sec[:7])
    with pytest.raises(P.MalformedSection):
        A.expand_outliers(sec[:-1])
    with pytest.raises(P.MalformedSection):
        A.expand_outliers(A.compact_outliers([(5, 1.0), (5, 2.0)]))


def test_alpha_map_knots_and_midpoints():
    for rel, a in ((1e-1, 2.0), (1e-2, 1.75), (1e-3, 1.5), (1e-4, 1.25), (1e-5, 1.0)):
        assert P.compute_alpha(rel) == a
        assert abs(P.compute_alpha(float(np.nextafter(rel, 0.0))) - a) <= 1e-12
    assert P.compute_alpha(1.0) == 2.0 and P.compute_alpha(1e-9) == 1.0
    assert P.compute_alpha(5.5e-3) == pytest.approx(1.625)


def test_plan_levels():
    plan = P.plan_levels(8, 1e-2, 1.5)
    assert [(s.level, s.stride) for s in plan.levels] == [(3, 4), (2, 2), (1, 1)]
    assert plan.levels[0].eb == 1e-2 / 1.5 ** 2 and plan.levels[2].eb == 1e-2
    for s in (2, 4, 16, 512):
        assert len(P.plan_levels(s, 1.0, 1.25).levels) == s.bit_length() - 1
    with pytest.raises(P.InvalidStride):
        P.plan_levels(12, 1.0, 1.5)


def test_lattice_counts():
    assert P.count_anchors(P.Dims((512, 512, 512)), 8) == 65 ** 3
    assert P.count_anchors(P.Dims((20,)), 8) == 4
    assert P.count_anchors(P.Dims((5, 5)), 8) == 4
    assert P.count_anchors(P.Dims((1,)), 8) == 1


def test_layout_and_config_validation():
    assert P.default_layout(3) == P.ChunkLayout(8, 3, (8, 8, 32))
    with pytest.raises(P.Inconsistent):
        P.ChunkLayout(8, 1, (12,))
    lay = P.ChunkLayout(8, 2, (16, 16))
    with pytest.raises(P.Inconsistent):
        P.PredictorConfig(lay, 1.5, (0, 0), (0, 0), 1e-3)
    with pytest.raises(P.Inconsistent):
        P.PredictorConfig(lay, 1.5, (0, 0), (0, 1), 0.0)


def test_scalar_semantics():
    assert P.quantize(1.05, 1.0, 0.01, 512) == P.Code(3)
    assert P.quantize(1.5, 1.0, 0.125, 512) == P.Code(2)
    assert P.quantize(0.5, 1.0, 0.125, 512) == P.Code(-2)
    assert P.quantize(2.0, 0.0, 0.5, 2) is P.OUTLIER
    assert P.spline_predict([-5.0, -1.0, 3.0, 7.0]) == 1.0
    assert P.spline_predict([None, -1.0, 3.0, None]) == 1.0
    assert P.spline_predict([None, -1.0, None, None]) == -1.0
    with pytest.raises(P.NoNeighbor):
        P.spline_predict([1.0, None, 1.0, 1.0])


def test_thread_count(monkeypatch):
    monkeypatch.delenv("EBCOMP_THREADS", raising=False)
    assert P.thread_count() == 1 and P.thread_count(4) == 4 and P.thread_count(0) == 1
    monkeypatch.setenv("EBCOMP_THREADS", "3")
    assert P.thread_count() == 3
    monkeypatch.setenv("EBCOMP_THREADS", "soup")
    assert P.thread_count() == 1


def test_float_keys_order():
    vals = [-math.inf, -3.5, -1e-30, -0.0, 0.0, 1e-40, 2.0, 3e38]
    keys = [float_to_key(np.float32(v)) for v in vals]
    assert keys == sorted(keys)
    for v in (-3.5, 0.0, 2.0, 1e-40):
        assert key_to_float(float_to_key(np.float32(v))) == float(np.float32(v))


def test_grid_host_semantics():
    g = P.Grid(P.Dims((2, 3)), np.arange(6, dtype=np.float32))
    assert g.data.shape == (2, 3) and g.values.tolist() == [0, 1, 2, 3, 4, 5]
    with pytest.raises(P.SizeMismatch):
        P.Grid(P.Dims((2, 3)), np.arange(5, dtype=np.float32))
    bad = np.ones(6, dtype=np.float32)
    bad[4] = np.nan
    with pytest.raises(P.NonFiniteValue) as e:
        P.Grid(P.Dims((6,)), bad)
    assert e.value.index == 4
    assert P.Grid(P.Dims((1,)), [-0.0]) != P.Grid(P.Dims((1,)), [0.0])
    with pytest.raises(ValueError):
        P.Dims((0, 3))
