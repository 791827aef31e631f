"""Golden fixtures for the Lorenzo predictor, written by the REFERENCE
package itself (build container only):

    python tests/golden/make_golden_lorenzo.py

tests/golden/lorenzo.npz holds seeded fields (ranks 1-3, smooth / noisy /
constant / spiky), ebcomp.compress(..., predictor="lorenzo") archives for
several bounds, modes and pass-2 settings, and ebcomp.decompress bytes.
They pin the oracle (tests/test_oracle_golden.py) and the GPU path
(tests/test_gpu_lorenzo.py) without /root/reference at run time."""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import ebcomp  # noqa: E402  (the reference)

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import make_field  # noqa: E402

SHAPES = [(300,), (1,), (2000,), (25, 31), (1, 40), (64, 64), (11, 13, 17), (9, 9, 9),
          (40, 24, 70), (17, 65, 33)]
KINDS = ["smooth", "noisy", "constant", "affine"]
CASES = [("rel", 1e-3, True), ("abs", 1e-2, False), ("rel", 1e-5, True), ("rel", 1e-1, True)]


def main():
    rng = np.random.default_rng(2024)
    out = {}
    k = 0
    for si, shape in enumerate(SHAPES):
        kind = KINDS[si % len(KINDS)]
        data = make_field(rng, shape, kind)
        if si % 3 == 2:  # a few spikes -> outliers
            flat = data.reshape(-1)
            for j in rng.integers(0, flat.size, size=3):
                flat[j] = np.float32(1e4)
        out[f"f{si}"] = data
        g = ebcomp.Grid(ebcomp.Dims(shape), data)
        for ci, (mode, eb, p2) in enumerate(CASES):
            blob = ebcomp.compress(g, eb, mode=mode, predictor="lorenzo", pass2=p2)
            out[f"a{si}_{ci}"] = np.frombuffer(blob, dtype=np.uint8)
            out[f"d{si}_{ci}"] = ebcomp.decompress(blob).data.reshape(-1).view(np.uint8)
            k += 1
    np.savez_compressed(os.path.join(HERE, "lorenzo.npz"), **out)
    print(f"{k} archives")


if __name__ == "__main__":
    main()
