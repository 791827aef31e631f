"""Synthetic inputs of the BASELINE.json configs, numpy only.

Shared by tests/golden/make_golden_large.py (which runs the reference on them
in the build container) and the GPU config tests (which regenerate them on
the B200 box and check the input digest before comparing archives).
"""
import numpy as np


def smooth(shape, phase=0.0):
    """f = sin(2pi 2z/nz) + 0.7 cos(2pi 3y/ny) + 0.5 sin(2pi 1.5x/nx)
    + 0.3 sin(2pi (z/nz + y/ny + x/nx)), each argument shifted by ``phase``;
    float64 math, cast to float32.  Same expression order as
    oracle.smooth_field and bench.smooth_field_gpu."""
    nz, ny, nx = shape
    z, y, x = np.meshgrid(np.arange(nz, dtype=np.float64), np.arange(ny, dtype=np.float64),
                          np.arange(nx, dtype=np.float64), indexing="ij", sparse=True)
    f = (np.sin(2 * np.pi * z * 2.0 / nz + phase)
         + 0.7 * np.cos(2 * np.pi * y * 3.0 / ny + phase)
         + 0.5 * np.sin(2 * np.pi * x * 1.5 / nx + phase)
         + 0.3 * np.sin(2 * np.pi * (z / nz + y / ny + x / nx) + phase))
    return f.astype(np.float32)


def noisy(shape, sigma=0.01):
    """The §8(d) noisy variant: smooth + N(0, sigma) from default_rng(0x5EED)."""
    rng = np.random.default_rng(0x5EED)
    f = smooth(shape).astype(np.float64) + rng.normal(0.0, sigma, shape)
    return f.astype(np.float32)


def make_input(cfg):
    shape = tuple(cfg["shape"])
    if cfg.get("kind", "smooth") == "noisy":
        return noisy(shape, cfg.get("sigma", 0.01))
    return smooth(shape, cfg.get("phase", 0.0))


def _cfg(name, shape, eb, **kw):
    d = {"name": name, "shape": list(shape), "eb": eb}
    d.update(kw)
    return d


# every single-GPU shape / eb that BASELINE.json lists (configs[1..4])
CONFIGS = (
    [_cfg("nyx512_1e-3", (512, 512, 512), 1e-3), _cfg("nyx512_1e-4", (512, 512, 512), 1e-4)]
    + [_cfg(f"miranda_{eb:g}", (256, 384, 384), eb) for eb in (1e-2, 1e-3, 1e-4, 1e-5)]
    + [_cfg(f"hurricane_{eb:g}", (100, 500, 500), eb) for eb in (1e-2, 1e-3, 1e-4, 1e-5)]
    + [_cfg(f"rtm_snap{k}", (449, 449, 235), 1e-3, phase=2 * np.pi * k / 8) for k in range(8)]
    + [_cfg("qmcpack_1e-3", (33120, 69, 69), 1e-3),
       _cfg("miranda_noisy_1e-4", (256, 384, 384), 1e-4, kind="noisy"),
       _cfg("hurricane_abs_1e-3", (100, 500, 500), 1e-3, mode="abs")]
)

BY_NAME = {c["name"]: c for c in CONFIGS}
