"""Parity of the alternative code paths inside the sm_100a kernels against the
CPU oracle (test infrastructure): TMA vs manual tile staging, interior vs
edge-shell tiles of the warp-per-tile predictor, the sparse vs dense Huffman
packer, and the exact-quantiser / outlier fix-up paths of the walks."""
import os

import numpy as np
import pytest

import paper_2312_05492_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _smooth(shape, seed=0, noise=0.0):
    g = [np.arange(s, dtype=np.float64) / max(s, 1) for s in shape]
    z, y, x = np.meshgrid(*g, indexing="ij")
    d = np.sin(2 * np.pi * 2 * z) + 0.7 * np.cos(2 * np.pi * 3 * y) + 0.5 * np.sin(3 * np.pi * x)
    if noise:
        d = d + np.random.default_rng(seed).normal(0.0, noise, size=shape)
    return d.astype(np.float32)


def _round_trip_equals_oracle(data, eb, **kw):
    blob = P.compress(P.Grid(P.Dims(data.shape), data), eb, **kw)
    ref = O.compress(data, eb, **kw)
    assert blob == ref
    out = P.decompress(blob)
    assert out.data.tobytes() == O.decompress(ref).tobytes()
    return blob


@pytest.mark.parametrize("shape", [(9, 9, 33), (8, 8, 32), (17, 2, 70), (2, 33, 97),
                                   (25, 17, 65), (16, 24, 64)])
def test_tile_shell_shapes(shape):
    # (9, 9, 33): one interior tile; (8, 8, 32): a single edge tile (closing
    # planes outside the grid); extents 2 and odd x exercise the shell logic
    data = _smooth(shape, noise=0.01)
    for eb in (1e-2, 1e-4):
        _round_trip_equals_oracle(data, eb)


def test_tma_and_manual_staging_identical():
    data = _smooth((40, 72, 96), noise=0.02)  # nx % 8 == 0: TMA by default
    blob = _round_trip_equals_oracle(data, 1e-3)
    os.environ["CSZI_NO_TMA"] = "1"
    try:
        blob2 = P.compress(P.Grid(P.Dims(data.shape), data), 1e-3)
        out2 = P.decompress(blob2)
    finally:
        del os.environ["CSZI_NO_TMA"]
    assert blob2 == blob
    assert out2.data.tobytes() == O.decompress(blob).tobytes()


@pytest.mark.parametrize("shape", [(40, 33, 69), (27, 18, 235), (17, 9, 33)])
def test_row_staging_unaligned_pitch(shape):
    """Row pitch not a multiple of 16 bytes: row-wise asynchronous staging
    (prefetched across tiles) against the oracle, at several eb."""
    data = _smooth(shape, noise=0.02)
    for eb in (1e-2, 1e-3, 1e-5):
        _round_trip_equals_oracle(data, eb)


def test_sparse_and_dense_huffman_packers():
    # smooth at 1e-3: almost every code is R (sparse packer); noisy at 1e-5:
    # most codes are not (dense packer)
    _round_trip_equals_oracle(_smooth((64, 64, 64)), 1e-3)
    _round_trip_equals_oracle(_smooth((48, 40, 64), seed=3, noise=0.05), 1e-5)


def test_outlier_heavy_and_exact_paths():
    data = _smooth((33, 40, 64), seed=5, noise=0.3)
    blob = _round_trip_equals_oracle(data, 1e-6)  # most points are outliers
    assert len(P.parse_archive(blob).outliers) > 8
    _round_trip_equals_oracle(data, 1e-3, mode="abs", quant_radius=4)  # |q| >= R often
    _round_trip_equals_oracle(data, 1e-3, quant_radius=7)  # odd R: bitstream not word-aligned
    g = P.Grid(P.Dims(data.shape), data)
    a = P.compress_device(g, 1e-4, exact=True).to_bytes()
    assert a == O.compress(data, 1e-4)


@pytest.mark.parametrize("shape", [(37, 21, 64), (9, 15, 96), (70, 8, 32)])
def test_nonr_bitmap_encoder(shape):
    # nx % 32 == 0: the predictor writes the non-R bitmap and the sparse
    # stream is encoded from it; partial z / y tiles take the edge epilogue
    data = _smooth(shape, seed=7, noise=0.001)
    data[shape[0] // 2, 3, 5] = 40.0  # one outlier
    for eb in (1e-3, 1e-2):
        _round_trip_equals_oracle(data, eb)


def test_bitmap_encoder_many_outliers():
    # sparse stream (R = "0") with thousands of outliers spread over the
    # super-chunks: outlier order and values come from the bitmap path
    data = _smooth((64, 64, 96), seed=9)
    flat = data.reshape(-1)
    flat[::97] = 1000.0
    flat[5000:5400] = -1000.0  # a dense run: super-chunk with > 256 non-R symbols
    blob = _round_trip_equals_oracle(data, 1e-3, mode="abs")
    sec = P.parse_archive(blob).outliers  # u64 count + 12-byte records
    assert int.from_bytes(sec[:8], "little") > 2000


def test_bitmap_and_full_scan_encoders_identical():
    # CSZI_NO_NZ=1 turns the predictor's non-R bitmap off: the sparse stream
    # then comes from the full-symbol packer; both must give the same bytes
    data = _smooth((40, 48, 64), seed=4, noise=0.002)
    data.reshape(-1)[::211] = 50.0
    ref = _round_trip_equals_oracle(data, 1e-3)
    os.environ["CSZI_NO_NZ"] = "1"
    try:
        blob = P.compress(P.Grid(P.Dims(data.shape), data), 1e-3)
    finally:
        del os.environ["CSZI_NO_NZ"]
    assert blob == ref
