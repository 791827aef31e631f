"""The CPU oracle's Lorenzo restatement (oracle/cszi_oracle.c orc_lorenzo)
against archives and decompressed bytes written by the reference itself
(tests/golden/make_golden_lorenzo.py)."""
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "lorenzo.npz")
CASES = [("rel", 1e-3, True), ("abs", 1e-2, False), ("rel", 1e-5, True), ("rel", 1e-1, True)]


@pytest.fixture(scope="module")
def lz():
    return np.load(GOLD)


def fields(lz):
    i = 0
    while f"f{i}" in lz:
        yield i, lz[f"f{i}"]
        i += 1


def test_oracle_lorenzo_archives_match_reference(lz):
    n = 0
    for i, data in fields(lz):
        for ci, (mode, eb, p2) in enumerate(CASES):
            blob = O.compress_lorenzo(data, eb, mode=mode, pass2=p2)
            assert blob == lz[f"a{i}_{ci}"].tobytes(), (i, data.shape, mode, eb)
            n += 1
    assert n == 40


def test_oracle_lorenzo_decompression_matches_reference(lz):
    for i, data in fields(lz):
        for ci in range(len(CASES)):
            back = O.decompress(lz[f"a{i}_{ci}"].tobytes())
            assert back.tobytes() == lz[f"d{i}_{ci}"].tobytes(), (i, ci)
