"""Oracle vs the reference package itself, on fresh random inputs (build
container only: skipped where /root/reference is absent)."""
import importlib
import os
import sys

import numpy as np
import pytest

from conftest import KINDS, REFERENCE_SRC
from oracle import oracle as O

pytestmark = pytest.mark.skipif(not os.path.isdir(REFERENCE_SRC), reason="reference not mounted")


@pytest.fixture(scope="module")
def ebcomp():
    sys.path.insert(0, REFERENCE_SRC)
    try:
        return importlib.import_module("ebcomp")
    finally:
        sys.path.remove(REFERENCE_SRC)


def test_random_archives_identical(ebcomp):
    rng = np.random.default_rng(99)
    for i in range(60):
        rank = i % 3 + 1
        shape = tuple(int(rng.integers(1, 36)) for _ in range(rank))
        data = KINDS[i % 4](rng, shape)
        g = ebcomp.Grid(ebcomp.Dims(shape), data)
        for mode, eb, p2 in (("rel", 1e-3, True), ("abs", 1e-2, False), ("rel", 1e-5, True)):
            ref = ebcomp.compress(g, eb, mode=mode, pass2=p2)
            assert O.compress(data, eb, mode=mode, pass2=p2) == ref, (shape, mode, eb)
            assert O.decompress(ref).tobytes() == ebcomp.decompress(ref).data.tobytes()


def test_codebook_and_stream_identical(ebcomp):
    from ebcomp.huffman import build_codebook, build_histogram, huffman_encode

    rng = np.random.default_rng(7)
    for k in (1, 2, 5, 40, 300, 1000):
        codes = rng.integers(-min(k, 511), min(k, 511) + 1, size=5000).astype(np.int32)
        book = build_codebook(build_histogram(codes, 512))
        cb = O.canonical(O.code_lengths(O.histogram(codes, 512)))
        assert np.array_equal(cb.lengths, book.code_lengths)
        assert O.huffman_encode(codes, cb, 512)[0] == huffman_encode(codes, book)[0]


def test_pass2_identical(ebcomp):
    rng = np.random.default_rng(3)
    for n in (0, 1, 2, 129, 1000, 70000):
        data = bytes((rng.random(n) < 0.6).astype(np.uint8) * rng.integers(1, 255, n).astype(np.uint8))
        assert O.pass2_encode(data) == ebcomp.pass2_encode(data)
