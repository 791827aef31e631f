"""Golden archive digests at the BASELINE.json sizes, written by the REFERENCE.

    NUMBA_CACHE_DIR=/tmp/numba python tests/golden/make_golden_large.py

Runs ebcomp.compress / ebcomp.decompress (the reference package under
/root/reference, build container only) on every single-GPU config that
BASELINE.json names and records, per config, the sha256 of the input field,
of the reference's archive and of its decompressed bytes, plus the archive
length and section sizes.  The fields are generated with numpy from the
SURVEY §8(d) formulas (``fields.py``, shared with the GPU tests), so the GPU box
regenerates bit-identical inputs (the input digest is checked first).

Output: tests/golden/large.json (tiny; committed).  tests/test_gpu_configs.py
compares the CUDA path's archive / decompressed digests against it, which
pins GPU == reference directly at full size (not only via the oracle).
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")
import ebcomp  # noqa: E402  (the reference)

from fields import CONFIGS, make_input  # noqa: E402


def sha(b) -> str:
    return hashlib.sha256(bytes(b)).hexdigest()


def main():
    only = set(sys.argv[1:])
    path = os.path.join(HERE, "large.json")
    out = {}
    if os.path.exists(path):
        with open(path) as f:
            out = json.load(f)
    threads = min(8, os.cpu_count() or 1)
    for cfg in CONFIGS:
        name = cfg["name"]
        if only and name not in only:
            continue
        data = make_input(cfg)
        t0 = time.time()
        g = ebcomp.Grid(ebcomp.Dims(data.shape), data)
        blob = ebcomp.compress(g, cfg["eb"], mode=cfg.get("mode", "rel"), threads=threads)
        t1 = time.time()
        back = ebcomp.decompress(blob, threads=threads)
        t2 = time.time()
        arc = ebcomp.parse_archive(blob)
        out[name] = {
            "shape": list(data.shape),
            "eb": cfg["eb"],
            "input_sha256": sha(data.tobytes()),
            "archive_sha256": sha(blob),
            "archive_bytes": len(blob),
            "decompressed_sha256": sha(back.data.tobytes()),
            "n_outliers": int.from_bytes(arc.outliers[:8], "little"),
            "bitstream_bytes": len(arc.bitstream),
            "reference_s": [round(t1 - t0, 2), round(t2 - t1, 2)],
        }
        print(name, out[name], flush=True)
        with open(path, "w") as f:
            json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
