"""n > 2^32: the 64-bit path (SURVEY §7 hard part 6, §8 J3).

A 1040 x 2048 x 2048 float32 field (4.36e9 values, 17.4 GB) compressed as one
grid on one GPU must give the same archive bytes as the same field split into
8 z-slabs (each slab < 2^32 values, stitched by the multi-GPU path on one
device), decompress within the bound, and decode any z-slab identically to the
matching planes of the whole field.  No CPU oracle can run at this size, so
parity here is the size-independent property "whole == sharded" plus the
bound; both paths are pinned to the oracle at smaller sizes elsewhere."""
import math

import pytest

import paper_2312_05492_b200 as P
from paper_2312_05492_b200 import distributed as D

pytestmark = pytest.mark.gpu

SHAPE = (1040, 2048, 2048)


def _field(torch, shape, chunk=16):
    """SURVEY §8d smooth field, generated plane-chunk by plane-chunk."""
    nz, ny, nx = shape
    out = torch.empty(shape, dtype=torch.float32, device="cuda")
    y = torch.arange(ny, dtype=torch.float64, device="cuda").view(1, ny, 1)
    x = torch.arange(nx, dtype=torch.float64, device="cuda").view(1, 1, nx)
    tp = 2 * math.pi
    fy = 0.7 * torch.cos(tp * y * 3.0 / ny)
    fx = 0.5 * torch.sin(tp * x * 1.5 / nx)
    for za in range(0, nz, chunk):
        zb = min(nz, za + chunk)
        z = torch.arange(za, zb, dtype=torch.float64, device="cuda").view(-1, 1, 1)
        f = torch.sin(tp * z * 2.0 / nz) + fy + fx + 0.3 * torch.sin(tp * (z / nz + y / ny + x / nx))
        out[za:zb] = f.to(torch.float32)
    return out


def _max_err(torch, x, y, chunk=32):
    m = 0.0
    for za in range(0, x.shape[0], chunk):
        d = (x[za:za + chunk].double() - y[za:za + chunk].double()).abs().max().item()
        m = max(m, d)
    return m


def test_more_than_2pow32_values_whole_equals_sharded():
    import torch

    free, _ = torch.cuda.mem_get_info()
    if free < 100 * (1 << 30):
        pytest.skip("needs ~100 GB of free device memory")
    x = _field(torch, SHAPE)
    n = x.numel()
    assert n > (1 << 32)
    arch = P.compress_device(P.Grid(P.Dims(SHAPE), x), 1e-3)
    blob = arch.to_bytes()
    h = P.parse_archive(blob)
    assert h.extents[:3] == SHAPE
    y = P.decompress_device(arch).tensor
    assert _max_err(torch, x, y) <= h.eb_abs
    # one z-slab of the decompressed field, decoded on its own
    z0, z1 = D.slab_bounds(SHAPE[0], 8)[7]
    part = P.decompress_device(arch, slab=(z0, z1))
    assert torch.equal(part, y[z0:z1])
    del y, part
    torch.cuda.empty_cache()
    # the same field as 8 z-slabs (each < 2^32 values) stitched into one archive
    sim = D.compress_simulated(x, 8, 1e-3)
    assert sim.to_bytes() == blob
