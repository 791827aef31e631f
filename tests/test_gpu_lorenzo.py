"""GPU Lorenzo predictor (csrc/lorenzo.cu) against the reference's own
archives (tests/golden/lorenzo.npz) and against the CPU oracle at sizes the
golden set does not reach."""
import os

import numpy as np
import pytest

import paper_2312_05492_b200 as P
from conftest import KINDS
from oracle import oracle as O

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "lorenzo.npz")
CASES = [("rel", 1e-3, True), ("abs", 1e-2, False), ("rel", 1e-5, True), ("rel", 1e-1, True)]


@pytest.fixture(scope="module")
def lz():
    return np.load(GOLD)


def test_gpu_lorenzo_archives_match_reference(lz):
    i = 0
    while f"f{i}" in lz:
        data = lz[f"f{i}"]
        g = P.Grid(P.Dims(data.shape), data)
        for ci, (mode, eb, p2) in enumerate(CASES):
            blob = P.compress(g, eb, mode=mode, predictor="lorenzo", pass2=p2)
            assert blob == lz[f"a{i}_{ci}"].tobytes(), (i, data.shape, mode, eb)
            back = P.decompress(lz[f"a{i}_{ci}"].tobytes())
            assert back.data.tobytes() == lz[f"d{i}_{ci}"].tobytes(), (i, ci)
        i += 1
    assert i == 10


@pytest.mark.parametrize("shape", [(200, 150, 96), (33, 290, 65), (1500, 900), (100000,)])
def test_gpu_lorenzo_vs_oracle_larger(shape):
    rng = np.random.default_rng(len(shape) * 7 + shape[0])
    data = KINDS[shape[0] % 2](rng, shape)
    for mode, eb in (("rel", 1e-3), ("rel", 1e-5)):
        blob = P.compress(P.Grid(P.Dims(shape), data), eb, mode=mode, predictor="lorenzo")
        assert blob == O.compress_lorenzo(data, eb, mode=mode), (shape, eb)
        back = P.decompress(blob).data
        assert back.tobytes() == O.decompress(blob).tobytes()
        eb_abs = P.parse_archive(blob).eb_abs
        assert float(np.abs(back.astype(np.float64) - data).max()) <= eb_abs


def test_gpu_lorenzo_fine_api_vs_oracle():
    rng = np.random.default_rng(11)
    for shape in ((57,), (20, 37), (9, 14, 40)):
        data = KINDS[1](rng, shape)
        data.reshape(-1)[5] = np.float32(1e5)
        f = P.lorenzo_predict_quantize(P.Grid(P.Dims(shape), data), 1e-4)
        codes, is_out = O.lorenzo_predict(data, 1e-4)
        assert np.array_equal(np.asarray(f.codes), codes)
        assert [i for i, _ in f.outliers] == np.nonzero(is_out)[0].tolist()
        assert f.anchors == []
        g = P.lorenzo_reconstruct(f, P.Dims(shape), 1e-4)
        outval = np.zeros(data.size, dtype=np.float32)
        outval[is_out.astype(bool)] = data.reshape(-1)[is_out.astype(bool)]
        ref = O.lorenzo_reconstruct(codes, is_out, outval, shape, 1e-4)
        assert g.data.tobytes() == ref.tobytes()
