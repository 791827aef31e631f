"""Generate the golden fixtures from the REFERENCE package (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden.npz: seeded input fields and the reference's own
archives / decompressed bytes for them, plus sinusoid_64 archives.  The
fixtures pin both the oracle (tests/test_oracle_golden.py, CPU) and the GPU
path (tests/test_gpu_parity.py) without /root/reference at run time.
"""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import ebcomp  # noqa: E402  (the reference)

HERE = os.path.dirname(os.path.abspath(__file__))


def smooth(rng, shape):
    axes = np.indices(shape).astype(np.float64)
    out = np.zeros(shape)
    for ax, coord in enumerate(axes):
        for _ in range(int(rng.integers(1, 4))):
            freq = rng.uniform(0.5, 3.0) / max(shape[ax], 2)
            out += rng.uniform(0.3, 1.0) * np.sin(2 * np.pi * freq * coord + rng.uniform(0, 6.283))
    return out


def make_field(rng, shape, kind):
    if kind == "smooth":
        return smooth(rng, shape).astype(np.float32)
    if kind == "noisy":
        return (smooth(rng, shape) + rng.normal(0, 0.2, shape)).astype(np.float32)
    if kind == "constant":
        return np.full(shape, np.float32(rng.uniform(-5, 5)), dtype=np.float32)
    axes = np.indices(shape).astype(np.float64)
    out = np.full(shape, rng.uniform(-1, 1))
    for c in axes:
        out = out + rng.uniform(-0.5, 0.5) * c
    return out.astype(np.float32)


def sinusoid_64():
    n = 64
    z, y, x = np.mgrid[0:n, 0:n, 0:n].astype(np.float64)
    f = (np.sin(2 * np.pi * z * 2.0 / n) + 0.7 * np.cos(2 * np.pi * y * 3.0 / n)
         + 0.5 * np.sin(2 * np.pi * x * 1.5 / n) + 0.3 * np.sin(2 * np.pi * (z + y + x) / n))
    return f.astype(np.float32)


def main():
    rng = np.random.default_rng(20231205)
    kinds = ("smooth", "noisy", "constant", "affine")
    settings = (("rel", 1e-3, True), ("abs", 1e-2, True), ("rel", 1e-5, True), ("rel", 1e-2, False))
    out = {}
    cases = []
    shapes = [(9,), (7,), (600,), (1100,), (5, 9), (40, 31), (17, 33), (1, 50), (9, 9, 9),
              (5, 7, 9), (2, 3, 4), (9, 1, 9), (17, 20, 23), (24, 17, 33), (1, 30, 40),
              (33, 9, 8), (20, 20, 70), (41, 12, 13)]
    for i, shape in enumerate(shapes):
        kind = kinds[i % 4]
        data = make_field(rng, shape, kind)
        out[f"in_{i}"] = data
        g = ebcomp.Grid(ebcomp.Dims(shape), data)
        for j, (mode, eb, p2) in enumerate(settings):
            blob = ebcomp.compress(g, eb, mode=mode, pass2=p2)
            back = ebcomp.decompress(blob)
            out[f"arc_{i}_{j}"] = np.frombuffer(blob, dtype=np.uint8)
            out[f"dec_{i}_{j}"] = back.data
            cases.append((i, j, mode, eb, p2, kind, shape))
    s64 = sinusoid_64()
    g = ebcomp.Grid(ebcomp.Dims(s64.shape), s64)
    for eb, p2 in ((1e-3, True), (1e-2, True), (1e-4, True), (1e-3, False)):
        blob = ebcomp.compress(g, eb, pass2=p2)
        out[f"s64_{eb:g}_{int(p2)}"] = np.frombuffer(blob, dtype=np.uint8)
    out["s64_input_sha"] = np.frombuffer(hashlib.sha256(s64.tobytes()).digest(), dtype=np.uint8)
    # overrides: alpha / variants / dim_order / radius
    d = make_field(rng, (19, 23, 29), "smooth")
    out["ovr_in"] = d
    g = ebcomp.Grid(ebcomp.Dims(d.shape), d)
    out["ovr_arc_0"] = np.frombuffer(ebcomp.compress(g, 1e-3, alpha=1.25, variants=(1, 0, 1),
                                                     dim_order=(2, 0, 1)), dtype=np.uint8)
    out["ovr_arc_1"] = np.frombuffer(ebcomp.compress(g, 1e-4, quant_radius=64), dtype=np.uint8)
    out["ovr_arc_2"] = np.frombuffer(ebcomp.compress(g, 1e-3, mode="abs", quant_radius=3),
                                     dtype=np.uint8)
    meta = np.array([f"{i}|{j}|{m}|{eb!r}|{int(p)}|{k}|{','.join(map(str, s))}"
                     for i, j, m, eb, p, k, s in cases])
    out["meta"] = meta
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("cases", len(cases), "bytes", os.path.getsize(os.path.join(HERE, "golden.npz")))


if __name__ == "__main__":
    main()
