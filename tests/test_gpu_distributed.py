"""GPU-count determinism: z-slab sharded compression of one
field over 1..8 simulated ranks on one GPU produces the byte-identical archive
of single-GPU compress (and of the oracle)."""
import numpy as np
import pytest

import paper_2312_05492_b200 as P
from paper_2312_05492_b200.distributed import compress_simulated, slab_bounds
from conftest import noisy_field, smooth_field
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape", [(64, 40, 70), (41, 30, 37), (57, 33, 47), (112, 56, 58), (9, 20, 33),
                                   (73, 40, 64), (40, 24, 96)])  # nx % 32 == 0: bitmap slab encodes
def test_slab_sharding_is_byte_identical(shape):
    import torch

    rng = np.random.default_rng(sum(shape))
    data = (smooth_field if shape[0] % 2 else noisy_field)(rng, shape)
    ref = O.compress(data, 1e-3)
    single = P.compress(P.Grid(P.Dims(shape), data), 1e-3)
    assert single == ref
    x = torch.from_numpy(data).cuda()
    for world in (1, 2, 3, 5, 8):
        arch = compress_simulated(x, world, 1e-3)
        assert arch.to_bytes() == ref, (shape, world, slab_bounds(shape[0], world))


def test_slab_sharding_modes_and_outliers():
    import torch

    rng = np.random.default_rng(3)
    data = noisy_field(rng, (48, 36, 40))
    x = torch.from_numpy(data).cuda()
    for mode, eb, p2 in (("abs", 1e-2, True), ("rel", 1e-5, False), ("rel", 1e-2, True)):
        ref = O.compress(data, eb, mode=mode, pass2=p2)
        for world in (2, 4):
            assert compress_simulated(x, world, eb, mode=mode, pass2=p2).to_bytes() == ref


@pytest.mark.parametrize("shape,world", [((64, 48, 64), 2), ((41, 30, 37), 4), ((100, 64, 96), 8),
                                         ((17, 24, 40), 3)])
def test_sharded_decompress_equals_whole(shape, world):
    """Each slab decoded from the one archive (symbol window + halo plane)
    matches the corresponding planes of the whole-grid decompression."""
    import torch

    from paper_2312_05492_b200.distributed import decompress_simulated

    rng = np.random.default_rng(7)
    data = noisy_field(rng, shape)
    for eb in (1e-3, 1e-5):
        blob = O.compress(data, eb)
        whole = P.decompress_device(blob).tensor
        parts = decompress_simulated(blob, world)
        assert torch.equal(parts.view(-1), whole.reshape(-1))
        arch = P.compress_device(P.Grid(P.Dims(shape), torch.from_numpy(data).cuda()), eb)
        assert torch.equal(decompress_simulated(arch, world).view(-1), whole.reshape(-1))


def test_phase_packed_pieces_odd_radius():
    """Odd R leaves the bitstream section unaligned: the root shifts the
    phase-packed pieces instead of OR-ing words; bytes still match."""
    import torch

    rng = np.random.default_rng(11)
    data = noisy_field(rng, (40, 24, 48))
    x = torch.from_numpy(data).cuda()
    for R in (7, 512):
        ref = O.compress(data, 1e-3, quant_radius=R)
        for world in (2, 3, 5):
            assert compress_simulated(x, world, 1e-3, quant_radius=R).to_bytes() == ref
