"""Bit-exact parity at every single-GPU BASELINE.json config, pinned to the
REFERENCE's own archives.

tests/golden/large.json holds, per config, the sha256 of the reference's
archive and decompressed bytes (written by tests/golden/make_golden_large.py,
which runs ebcomp on the same numpy-generated field).  Here the field is
regenerated, its digest checked, and the CUDA path's archive and decompressed
field must hash identically: codes, outliers, histogram, codebook, bitstream
and pass-2 bytes are all inside the archive digest.

Covers the dense packer (hurricane / miranda at 1e-5: 10^5+ outliers), the
non-TMA staging path (nx = 235, 69: row pitch not a multiple of 16 bytes),
abs mode, the noisy §8(d) variant and the 8 RTM snapshot phases.
"""
import hashlib
import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from fields import CONFIGS, make_input  # noqa: E402

import paper_2312_05492_b200 as P  # noqa: E402

with open(os.path.join(HERE, "golden", "large.json")) as _f:
    GOLD = json.load(_f)

NAMES = [c["name"] for c in CONFIGS if c["name"] in GOLD]


def _sha(b) -> str:
    return hashlib.sha256(bytes(b)).hexdigest()


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_config_archive_equals_reference(name):
    import torch

    cfg = next(c for c in CONFIGS if c["name"] == name)
    gold = GOLD[name]
    data = make_input(cfg)
    assert _sha(data.tobytes()) == gold["input_sha256"], "input generator drifted"
    x = torch.from_numpy(data).cuda()
    g = P.Grid(P.Dims(data.shape), x)
    arch = P.compress_device(g, cfg["eb"], mode=cfg.get("mode", "rel"))
    blob = arch.to_bytes()
    assert len(blob) == gold["archive_bytes"]
    assert _sha(blob) == gold["archive_sha256"]
    y = P.decompress_device(arch)
    host = y.tensor.cpu().numpy()
    assert _sha(host.tobytes()) == gold["decompressed_sha256"]
    eb_abs = P.parse_archive(blob).eb_abs
    assert float(np.abs(host.astype(np.float64) - data.astype(np.float64)).max()) <= eb_abs
    # the host-bytes API gives the same archive
    if data.nbytes <= 200 << 20:
        assert _sha(P.compress(P.Grid(P.Dims(data.shape), data), cfg["eb"],
                               mode=cfg.get("mode", "rel"))) == gold["archive_sha256"]
