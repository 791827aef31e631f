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
        # the Huffman synchronisation split by chunk ranges across the slabs
        assert torch.equal(decompress_simulated(arch, world, split=True).view(-1),
                           whole.reshape(-1))


@pytest.mark.parametrize("shape,world,eb", [((64, 64, 64), 2, 1e-3), ((96, 40, 64), 8, 1e-5),
                                            ((256, 128, 128), 4, 1e-4), ((9, 16, 32), 3, 1e-3)])
def test_split_decompress_ranges(shape, world, eb):
    """decompress_slabs_split: each slab synchronises only its chunk range of
    the Huffman stream (records all-gathered, entries repaired), then writes
    and reconstructs its own planes -- bit-identical to the single-rank
    slab decode; the split path is taken (not the fallback)."""
    import torch

    from paper_2312_05492_b200.distributed import SimComm, decompress_slabs_split, slab_bounds

    rng = np.random.default_rng(11)
    data = noisy_field(rng, shape)
    arch = P.compress_device(P.Grid(P.Dims(shape), torch.from_numpy(data).cuda()), eb)
    whole = P.decompress_device(arch).tensor
    bounds = slab_bounds(shape[0], world)
    got = decompress_slabs_split(arch, [(r, z0, z1) for r, (z0, z1) in enumerate(bounds)],
                                 SimComm(world), world)
    assert got is not None
    for (z0, z1, y), (b0, b1) in zip(got, bounds):
        assert (z0, z1) == (b0, b1)
        assert torch.equal(y.reshape(-1), whole[z0:z1].reshape(-1))


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


def test_snapshot_batch_is_byte_identical():
    """A batch of snapshots (RTM x 8 style: the §8d field with a phase per
    snapshot) compressed with one collective per stage for the whole batch:
    every archive equals single-GPU compress of that snapshot."""
    import math

    import torch

    from paper_2312_05492_b200.distributed import compress_simulated_batch

    shape = (45, 33, 40)
    snaps = [O.smooth_field(shape, phase=2 * math.pi * k / 8) for k in range(8)]
    refs = [P.compress(P.Grid(P.Dims(shape), d), 1e-3) for d in snaps]
    xs = [torch.from_numpy(d).cuda() for d in snaps]
    for world in (1, 2, 3, 6):
        archs = compress_simulated_batch(xs, world, 1e-3)
        assert [a.to_bytes() for a in archs] == refs, world


def _torchcomm_worker(rank, world, port, data, out_path):
    """One rank of a real torch.distributed run (gloo process group, both
    ranks on cuda:0): GpuSlabBackend + TorchComm end to end."""
    import os

    import torch
    import torch.distributed as dist

    from paper_2312_05492_b200.distributed import (TorchComm, compress_sharded,
                                                   compress_sharded_batch, decompress_sharded,
                                                   decompress_slabs_split, slab_bounds)

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nz = data.shape[0]
        z0, z1 = slab_bounds(nz, world)[rank]
        x = torch.from_numpy(data[z0:min(z1 + 1, nz)].copy()).cuda()
        arch = compress_sharded(x, data.shape, z0, z1, 1e-3)
        # the same with pass-2 encoded per slab (forced on this small field)
        from paper_2312_05492_b200 import distributed as D

        D.PASS2_SPLIT_MIN_BYTES = 0
        arch_p2 = compress_sharded(x, data.shape, z0, z1, 1e-3)
        D.PASS2_SPLIT_MIN_BYTES = 48 << 20
        if rank == 0:
            assert arch_p2.to_bytes() == arch.to_bytes()
        batch = compress_sharded_batch([x, x * 2.0], data.shape, z0, z1, 1e-3)
        blob = arch.to_bytes() if rank == 0 else None
        # every rank decodes its slab of the one archive
        obj = [blob]
        dist.broadcast_object_list(obj, src=0)
        _, _, ys = decompress_sharded(obj[0])
        parts = [None] * world
        dist.all_gather_object(parts, ys.cpu().numpy())
        # the chunk-range split of the Huffman synchronisation over TorchComm
        got = decompress_slabs_split(obj[0], [(rank, z0, z1)], TorchComm(), world)
        assert got is not None and torch.equal(got[0][2], ys)
        D.P2D_SPLIT_MIN_BYTES = 0  # and with the pass-2 decode split too
        got = decompress_slabs_split(obj[0], [(rank, z0, z1)], TorchComm(), world)
        assert got is not None and torch.equal(got[0][2], ys)
        if rank == 0:
            np.savez(out_path, blob=np.frombuffer(blob, dtype=np.uint8),
                     b0=np.frombuffer(batch[0].to_bytes(), dtype=np.uint8),
                     b1=np.frombuffer(batch[1].to_bytes(), dtype=np.uint8),
                     dec=np.concatenate(parts, 0))
    finally:
        dist.destroy_process_group()


def test_torchcomm_gpu_backend_two_processes(tmp_path):
    """The real combination: two processes, TorchComm over a
    gloo group, GpuSlabBackend on the GPU -> the single-GPU archive bytes;
    sharded decompress -> the whole-grid decompression."""
    import socket

    import torch.multiprocessing as mp

    rng = np.random.default_rng(21)
    data = noisy_field(rng, (40, 24, 64))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "r0.npz")
    mp.start_processes(_torchcomm_worker, args=(2, port, data, out), nprocs=2, join=True,
                       start_method="spawn")
    r = np.load(out)
    ref = P.compress(P.Grid(P.Dims(data.shape), data), 1e-3)
    assert r["blob"].tobytes() == ref
    assert r["b0"].tobytes() == ref
    assert r["b1"].tobytes() == P.compress(P.Grid(P.Dims(data.shape), data * np.float32(2.0)),
                                           1e-3)
    assert r["dec"].tobytes() == P.decompress(ref).data.tobytes()


@pytest.mark.parametrize("shape,world", [((64, 48, 64), 2), ((100, 64, 96), 8), ((41, 30, 40), 3),
                                         ((256, 96, 128), 4)])
def test_distributed_pass2_is_byte_identical(shape, world, monkeypatch):
    """Pass-2 encoded where the pieces live (cut after zero runs, prefixes
    borrowed from the next slab, root tail + outliers): the archive equals
    single-GPU compress, single snapshots and a batch."""
    import torch

    from paper_2312_05492_b200 import distributed as D

    monkeypatch.setattr(D, "PASS2_SPLIT_MIN_BYTES", 0)
    calls = []
    orig = D._pass2_split
    monkeypatch.setattr(D, "_pass2_split", lambda *a: calls.append(1) or orig(*a))
    rng = np.random.default_rng(5)
    for eb in (1e-3, 1e-5):
        data = smooth_field(rng, shape) if eb == 1e-3 else noisy_field(rng, shape)
        x = torch.from_numpy(data).cuda()
        ref = P.compress(P.Grid(P.Dims(shape), data), eb)
        assert D.compress_simulated(x, world, eb).to_bytes() == ref
        batch = D.compress_simulated_batch([x, x * 1.5], world, eb)
        assert batch[0].to_bytes() == ref
        assert batch[1].to_bytes() == P.compress(P.Grid(P.Dims(shape), data * np.float32(1.5)),
                                                 eb)
    assert calls


@pytest.mark.parametrize("shape,world,eb", [((64, 64, 64), 2, 1e-3), ((96, 40, 64), 8, 1e-5),
                                            ((256, 128, 128), 4, 1e-4), ((41, 30, 37), 3, 1e-3)])
def test_split_decompress_with_split_pass2(shape, world, eb, monkeypatch):
    """The pass-2 decode split as well (tables per rank, all-gathered; each
    slab expands only the raw ranges it reads): still bit-identical."""
    import torch

    from paper_2312_05492_b200 import distributed as D

    monkeypatch.setattr(D, "P2D_SPLIT_MIN_BYTES", 0)
    made = []
    orig = D._split_pass2_decode
    monkeypatch.setattr(D, "_split_pass2_decode", lambda *a: made.append(1) or orig(*a))
    rng = np.random.default_rng(13)
    data = noisy_field(rng, shape)
    arch = P.compress_device(P.Grid(P.Dims(shape), torch.from_numpy(data).cuda()), eb)
    whole = P.decompress_device(arch).tensor
    bounds = D.slab_bounds(shape[0], world)
    got = D.decompress_slabs_split(arch, [(r, z0, z1) for r, (z0, z1) in enumerate(bounds)],
                                   D.SimComm(world), world)
    assert got is not None and made
    for (z0, z1, y), (b0, b1) in zip(got, bounds):
        assert torch.equal(y.reshape(-1), whole[z0:z1].reshape(-1))
