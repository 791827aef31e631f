"""The oracle pinned to the reference at BASELINE sizes (CPU): the oracle's
archive and decompressed bytes hash to the digests the reference itself wrote
(tests/golden/large.json).  A subset keeps the CPU suite short; set
CSZI_ORACLE_ALL=1 for every config."""
import hashlib
import json
import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from fields import BY_NAME, make_input  # noqa: E402

from oracle import oracle as O  # noqa: E402

with open(os.path.join(HERE, "golden", "large.json")) as _f:
    GOLD = json.load(_f)

SUBSET = ("hurricane_1e-05", "rtm_snap3", "miranda_noisy_1e-4", "hurricane_abs_1e-3")
NAMES = sorted(GOLD) if os.environ.get("CSZI_ORACLE_ALL") else list(SUBSET)


@pytest.mark.parametrize("name", NAMES)
def test_oracle_matches_reference_digest(name):
    cfg = BY_NAME[name]
    g = GOLD[name]
    data = make_input(cfg)
    assert hashlib.sha256(data.tobytes()).hexdigest() == g["input_sha256"]
    blob = O.compress(data, cfg["eb"], mode=cfg.get("mode", "rel"), threads=os.cpu_count())
    assert len(blob) == g["archive_bytes"]
    assert hashlib.sha256(blob).hexdigest() == g["archive_sha256"]
    back = O.decompress(blob, threads=os.cpu_count())
    assert hashlib.sha256(back.tobytes()).hexdigest() == g["decompressed_sha256"]
