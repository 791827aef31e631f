"""Multi-process (gloo, world 2 and 3) check of the z-slab orchestration:
collectives, slab partition, bit/outlier offsets, root assembly.  The
per-slab compute comes from an oracle-backed backend (CPU), so this runs
without a GPU; the GPU backend is covered by tests/test_gpu_distributed.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_05492_b200 import distributed as D
from paper_2312_05492_b200._keys import float_to_key


class OracleSlabBackend:
    """Slab stages from the oracle's full-field results (test-only)."""

    def __init__(self, full: np.ndarray, eb: float, mode: str):
        from oracle import oracle as O

        self.O = O
        self.full = full
        self.cfg = O.select_config(full, mode, eb)
        self.codes, self.is_out, _ = O.predict(full, self.cfg)
        self.plane = full.shape[1] * full.shape[2]

    def range_keys(self, s):
        own = self.full[s.z0:s.z1]
        lo = float_to_key(np.float32(own.min())) if own.size else 0xFFFFFFFF
        hi = float_to_key(np.float32(own.max())) if own.size else 0
        return torch.tensor([lo, -hi, D.INT64_MAX], dtype=torch.int64)

    def set_range(self, s, k):
        s.scratch["range"] = k.clone()

    def samples(self, s):
        # owned sample values only (the packed layout of k_sample_gather)
        v = np.zeros(64 * 3 * 5, dtype=np.int32)
        ext = self.full.shape
        per = [self.O.sample_axis(e) for e in ext]
        pts = [p if p else [e // 2] for p, e in zip(per, ext)]
        mesh = np.meshgrid(*pts, indexing="ij")
        for p, point in enumerate(zip(*(m.ravel() for m in mesh))):
            for d in range(3):
                if not per[d]:
                    continue
                for k, off in enumerate((-3, -1, 1, 3, 0)):
                    c = list(point)
                    c[d] += off
                    if s.z0 <= c[0] < s.z1:
                        v[(p * 3 + d) * 5 + k] = np.float32(self.full[tuple(c)]).view(np.int32)
        return torch.from_numpy(v)

    def tune(self, s, samples, alpha):
        s.scratch["samples"] = samples.clone()
        assert alpha == self.cfg.alpha

    def predict(self, s):
        c = self.codes.reshape(self.full.shape)[s.z0:s.z1].ravel()
        o = self.is_out.reshape(self.full.shape)[s.z0:s.z1].ravel()
        s.scratch["c"], s.scratch["o"] = c, o
        return torch.from_numpy(self.O.histogram(c, self.cfg.quant_radius))

    def codebook(self, s, hist):
        s.scratch["book"] = self.O.canonical(self.O.code_lengths(hist.numpy()))

    def encode(self, s):
        stream, nbits = self.O.huffman_encode(s.scratch["c"], s.scratch["book"], 512)
        oidx = np.nonzero(s.scratch["o"])[0] + s.z0 * self.plane
        s.scratch.update(stream=stream, nbits=nbits, oidx=oidx)
        return torch.tensor([nbits, oidx.size], dtype=torch.int64)

    def anchors(self, s):
        ax = [np.asarray(self.O.anchor_axis(e, 8)) for e in self.full.shape]
        az = ax[0][(ax[0] >= s.z0) & (ax[0] < s.z1)]
        return torch.from_numpy(np.ascontiguousarray(self.full[np.ix_(az, ax[1], ax[2])]).ravel())

    def pieces(self, s, counts):
        b = torch.from_numpy(np.frombuffer(s.scratch["stream"], dtype=np.uint8).copy())
        oidx = torch.from_numpy(s.scratch["oidx"].astype(np.int64))
        oval = torch.from_numpy(self.full.ravel()[s.scratch["oidx"]].astype(np.float32))
        return b, oidx, oval

    def assemble(self, s0, anchors, bits, nbits, oidx, oval, pass2, alpha):
        total = sum(nbits)
        out = np.zeros((total + 7) // 8 + 1, dtype=np.uint8)
        off = 0
        for piece, nb in zip(bits, nbits):  # bit-shift concatenation
            p = piece.numpy()
            b0, sh = off // 8, off % 8
            for i in range((nb + 7) // 8):
                out[b0 + i] |= p[i] >> sh
                if sh:
                    out[b0 + i + 1] |= (int(p[i]) << (8 - sh)) & 0xFF
            off += nb
        idx = np.concatenate([x.numpy() for x in oidx])
        val = np.concatenate([x.numpy() for x in oval])
        sections = (torch.cat(anchors).numpy().astype("<f4").tobytes(),
                    s0.scratch["book"].lengths.tobytes(), out[: (total + 7) // 8].tobytes(),
                    self.O.compact_outliers(idx, val))
        return self.O.serialize(self.cfg, s0.mode, s0.eb, pass2, sections)


def _worker(rank, world, port, full, eb, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        z0, z1 = D.slab_bounds(full.shape[0], world)[rank]
        st = D.SlabState(x=None, extents=full.shape, z0=z0, z1=z1, eb=eb, mode=mode, radius=512)
        comm = D.TorchComm()
        be = OracleSlabBackend(full, eb, mode)
        keys = [be.range_keys(st)]
        comm.allreduce(keys, "min")
        lo_key = int(keys[0][0])
        samp = [be.samples(st)]
        comm.allreduce(samp, "sum")
        full_st = D.SlabState(x=None, extents=full.shape, z0=0, z1=full.shape[0], eb=eb,
                              mode=mode, radius=512)
        assert torch.equal(samp[0], be.samples(full_st))  # exact sample all-reduce
        assert lo_key == float_to_key(np.float32(full.min()))
        blob = D.compress_slabs([st], comm, backend=be, pass2=True)
        q.put((rank, blob))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,shape,eb,mode", [(2, (41, 18, 21), 1e-3, "rel"),
                                                 (3, (57, 16, 19), 1e-5, "rel"),
                                                 (2, (24, 20, 17), 1e-2, "abs")])
def test_gloo_slab_orchestration_matches_oracle(world, shape, eb, mode):
    from oracle import oracle as O

    rng = np.random.default_rng(7)
    full = (np.sin(np.indices(shape).sum(0) * 0.21) + rng.normal(0, 0.05, shape)).astype(np.float32)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, full, eb, mode, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res[0] == O.compress(full, eb, mode=mode)
    assert all(res[r] is None for r in range(1, world))


def test_slab_bounds_partition():
    assert D.slab_bounds(41, 5) == [(0, 16), (16, 24), (24, 32), (32, 40), (40, 41)]
    assert D.slab_bounds(512, 8) == [(64 * r, 64 * (r + 1)) for r in range(8)]
    b = D.slab_bounds(9, 4)
    assert b[0] == (0, 8) and b[1] == (8, 9) and b[2] == (9, 9) and b[3] == (9, 9)
    for nz in (1, 7, 8, 9, 100, 449):
        for w in (1, 2, 3, 8):
            bb = D.slab_bounds(nz, w)
            assert bb[0][0] == 0 and bb[-1][1] == nz
            assert all(a[1] == b[0] for a, b in zip(bb, bb[1:]))
            assert all(z0 % 8 == 0 for z0, _ in bb if z0 < nz)
