"""Multi-GPU compression by z-slabs.

One field, one archive, byte-identical to single-GPU ``compress``.  The
⌈nz/8⌉ anchor tiles along z are split as evenly as possible over the ranks;
rank r owns planes [z0, z1) and holds one closing halo plane (z1) as well,
which is all the tile-confined predictor needs (predictor.py:293-299), so
prediction runs without any exchange.  Collectives:

1. allreduce MIN of (range key min, -range key max, first non-finite index);
2. allreduce SUM of the packed tuner samples (each sample value is owned by
   exactly one rank; float bit patterns, so the sum is exact);
3. allreduce SUM of the uint64[2R] histogram -> identical codebook everywhere;
4. allgather of per-slab (bit count, outlier count);
5. gather of anchors / bitstream / outliers to rank 0, which concatenates the
   bitstreams at their global bit offsets and runs pass-2.

``Comm`` abstracts the collectives: ``TorchComm`` (torch.distributed: NCCL on
GPU tensors, gloo on CPU), ``SimComm`` (N slabs in one process, used to check
GPU-count determinism on a single GPU).  ``GpuSlabBackend`` runs every
per-slab stage in libcszi.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .archive import EB_ABS, EB_REL, HEADER_SIZE, PREDICTOR_INTERP, pack_header, unpack_header
from .errors import EmptyHistogram, Inconsistent, LengthOverflow, NonFiniteValue
from .pipeline import DeviceArchive
from .predictor import count_anchors, ctl_order, ctl_variants, default_layout, make_geom, make_params
from .tuning import compute_alpha

INT64_MAX = (1 << 63) - 1
ANCHOR_TILE = 8  # z-slabs align to the 3-D anchor stride


def slab_bounds(nz: int, world: int, tile: int = ANCHOR_TILE) -> list:
    """Owned z ranges: ⌈nz/tile⌉ tiles, the first (tiles mod world) ranks get one more."""
    tiles = -(-nz // tile)
    base, extra = divmod(tiles, world)
    out, t = [], 0
    for r in range(world):
        cnt = base + (1 if r < extra else 0)
        z0 = min(nz, t * tile)
        z1 = min(nz, (t + cnt) * tile)
        out.append((z0, z1))
        t += cnt
    return out


# ---------------------------------------------------------------------------
# communicators
# ---------------------------------------------------------------------------
class SimComm:
    """All slabs live in this process; collectives reduce across the list."""

    def __init__(self, world: int):
        self.world = world

    def allreduce(self, ts, op: str):
        t = _lib.torch()
        stack = t.stack([x.reshape(-1) for x in ts])
        r = {"sum": stack.sum(0), "min": stack.min(0).values, "max": stack.max(0).values}[op]
        for x in ts:
            x.copy_(r.view_as(x).to(x.dtype))

    def allgather(self, ts):
        return [list(ts) for _ in ts]

    def gather(self, ts, sizes=None):
        return list(ts)  # every slab is local: "root" sees all


class TorchComm:
    """torch.distributed collectives (one slab per process)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def allreduce(self, ts, op: str):
        d = self.dist
        o = {"sum": d.ReduceOp.SUM, "min": d.ReduceOp.MIN, "max": d.ReduceOp.MAX}[op]
        for x in ts:
            d.all_reduce(x, op=o, group=self.group)

    def allgather(self, ts):
        out = []
        for x in ts:
            parts = [x.new_empty(x.shape) for _ in range(self.world)]
            self.dist.all_gather(parts, x, group=self.group)
            out.append(parts)
        return out

    def gather(self, ts, sizes=None):
        """Variable-length 1-D tensors -> list on rank 0 (None elsewhere).
        ``sizes`` (element counts of every rank, when the caller knows them)
        saves the size all-gather and its host round trip."""
        t = _lib.torch()
        (x,) = ts
        if sizes is None:
            n = t.tensor([x.numel()], dtype=t.int64, device=x.device)
            got = [t.empty_like(n) for _ in range(self.world)]
            self.dist.all_gather(got, n, group=self.group)
            sizes = [int(v) for v in t.cat(got).cpu().tolist()]
        m = max(max(sizes), 1)
        pad = x.new_zeros(m)
        pad[: x.numel()] = x.reshape(-1)
        if self.rank == 0:
            parts = [x.new_empty(m) for _ in range(self.world)]
            self.dist.gather(pad, parts, dst=0, group=self.group)
            return [p[:s] for p, s in zip(parts, sizes)]
        self.dist.gather(pad, None, dst=0, group=self.group)
        return None


# ---------------------------------------------------------------------------
# per-slab state + GPU backend
# ---------------------------------------------------------------------------
@dataclass
class SlabState:
    x: object            # local planes [z0, min(z1 + 1, nz)) as float32 (device)
    extents: tuple       # global extents (rank 3)
    z0: int
    z1: int
    eb: float
    mode: str
    radius: int
    scratch: dict = field(default_factory=dict)


class GpuSlabBackend:
    def geom(self, s: SlabState):
        g = s.scratch.get("geom")
        if g is None:
            g = make_geom(s.extents, default_layout(3))
            g.slab[0] = s.z0
            g.slab[1] = s.z1
            s.scratch["geom"] = g
        return g

    def range_keys(self, s: SlabState):
        """Range + finite scan and the tuner's sample gather of the owned
        planes, one libcszi call (the samples wait in scratch for samples())."""
        t = _lib.require_cuda()
        lib = _lib.load()
        ctl = _lib.DeviceCtl()
        s.scratch["ctl"] = ctl
        ny, nx = s.extents[1], s.extents[2]
        n_own = max(s.z1 - s.z0, 0) * ny * nx
        keys = t.empty(3, dtype=t.int64, device="cuda")
        samples = t.empty(_lib.SAMPLE_WORDS, dtype=t.int32, device="cuda")
        _lib.check(lib.cszi_shard_scan(_lib.ptr(s.x) if n_own else None, n_own, s.z0 * ny * nx,
                                       ctypes.byref(self.geom(s)), ctl.ptr, _lib.ptr(keys),
                                       _lib.ptr(samples), _lib.stream_ptr()), "shard_scan")
        s.scratch["samples"] = samples
        return keys

    def set_range(self, s: SlabState, k):
        lib = _lib.load()
        _lib.check(lib.cszi_shard_set_range(s.scratch["ctl"].ptr, _lib.ptr(k), _lib.stream_ptr()),
                   "shard_set_range")
        s.scratch["range"] = k

    def samples(self, s: SlabState):
        return s.scratch["samples"]

    def tune(self, s: SlabState, samples, alpha: float):
        lib = _lib.load()
        g = self.geom(s)
        p = make_params(3, s.mode == "rel", s.eb, s.radius, alpha, 8)
        _lib.check(lib.cszi_tune_from_samples(_lib.ptr(samples), ctypes.byref(g), ctypes.byref(p),
                                              s.scratch["ctl"].ptr, _lib.stream_ptr()), "tune")

    def predict(self, s: SlabState):
        t = _lib.torch()
        lib = _lib.load()
        ny, nx = s.extents[1], s.extents[2]
        n_own = (s.z1 - s.z0) * ny * nx
        sym = t.empty(n_own + 16, dtype=t.int16, device="cuda")
        hist = t.zeros(2 * s.radius, dtype=t.int64, device="cuda")
        # non-R bitmap over the planes held (slab + halo): drives the sparse
        # encoder as in single-GPU compress
        nzmap = t.empty(s.x.numel() // 32 + 4, dtype=t.int32, device="cuda")
        nz_done = ctypes.c_int32(0)
        g = self.geom(s)
        if n_own:
            _lib.check(lib.cszi_predict_nz(_lib.ptr(s.x), ctypes.byref(g), s.radius, 0,
                                           _lib.ptr(sym), _lib.ptr(hist), _lib.ptr(nzmap),
                                           ctypes.byref(nz_done), s.scratch["ctl"].ptr,
                                           _lib.stream_ptr()), "predict")
        s.scratch["sym"] = sym
        s.scratch["n_own"] = n_own
        s.scratch["nzmap"] = nzmap if nz_done.value else None
        s.scratch["hist_local"] = hist.clone() if nz_done.value else None
        return hist

    def codebook(self, s: SlabState, hist):
        t = _lib.torch()
        lib = _lib.load()
        nb = 2 * s.radius
        lengths = t.zeros(nb, dtype=t.uint8, device="cuda")
        words = t.zeros(nb, dtype=t.int32, device="cuda")
        _lib.check(lib.cszi_codebook(_lib.ptr(hist), nb, _lib.ptr(lengths), _lib.ptr(words),
                                     s.scratch["ctl"].ptr, _lib.stream_ptr()), "codebook")
        s.scratch["lengths"] = lengths
        s.scratch["words"] = words

    def piece_bits(self, s: SlabState, hist_local):
        """Bits of this slab's Huffman piece: sum over symbols of count x length
        (outliers and anchors are counted as R, which is how they are coded)."""
        t = _lib.torch()
        out = t.empty(1, dtype=t.int64, device="cuda")
        _lib.check(_lib.load().cszi_shard_piece_bits(_lib.ptr(hist_local),
                                                     _lib.ptr(s.scratch["lengths"]),
                                                     2 * s.radius, _lib.ptr(out),
                                                     _lib.stream_ptr()), "shard_piece_bits")
        return out

    def encode(self, s: SlabState, bit_base: int = 0):
        t = _lib.torch()
        lib = _lib.load()
        s.scratch["bit_base"] = int(bit_base)
        n = s.scratch["n_own"]
        ny, nx = s.extents[1], s.extents[2]
        cap = ((4 * n + 64) + 15) & ~15
        # no zero fill (537 MB per 512-plane slab): the packers write or zero
        # every word of the stream they use (k_enc_zero / k_scan_pair)
        bits = t.empty(cap + 16, dtype=t.uint8, device="cuda")
        ocap = n + 16
        oidx = t.empty(ocap, dtype=t.int64, device="cuda")
        oval = t.empty(ocap, dtype=t.float32, device="cuda")
        ws = _lib.WS.get(int(lib.cszi_encode_sym_workspace_size(max(n, 1))), "enc_slab")
        ctl = s.scratch["ctl"]
        nzmap = s.scratch.get("nzmap")
        if n and nzmap is not None:
            _lib.check(lib.cszi_encode_sym_nz(
                _lib.ptr(s.scratch["sym"]), n, s.radius, _lib.ptr(s.scratch["lengths"]),
                _lib.ptr(s.scratch["words"]), _lib.ptr(s.x), s.z0 * ny * nx, int(bit_base),
                _lib.ptr(bits), cap, _lib.ptr(oidx), _lib.ptr(oval), ocap, _lib.ptr(nzmap),
                _lib.ptr(s.scratch["hist_local"]), _lib.ptr(ws), ctl.ptr, _lib.stream_ptr()),
                "encode")
        elif n:
            _lib.check(lib.cszi_encode_sym_at(
                _lib.ptr(s.scratch["sym"]), n, s.radius, _lib.ptr(s.scratch["lengths"]),
                _lib.ptr(s.scratch["words"]), _lib.ptr(s.x), s.z0 * ny * nx, int(bit_base),
                _lib.ptr(bits), cap, _lib.ptr(oidx), _lib.ptr(oval), ocap, _lib.ptr(ws), ctl.ptr,
                _lib.stream_ptr()), "encode")
        s.scratch.update(bits=bits, oidx=oidx, oval=oval)
        counts = t.empty(2, dtype=t.int64, device="cuda")
        _lib.check(lib.cszi_shard_counts(ctl.ptr, _lib.ptr(counts), _lib.stream_ptr()),
                   "shard_counts")
        return counts

    def anchors(self, s: SlabState):
        t = _lib.torch()
        lib = _lib.load()
        if s.z1 <= s.z0:
            return t.empty(0, dtype=t.float32, device="cuda")
        g = self.geom(s)
        na = int(lib.cszi_slab_anchor_count(ctypes.byref(g)))
        out = t.empty(max(na, 1), dtype=t.float32, device="cuda")
        if na:
            _lib.check(lib.cszi_gather_anchors(_lib.ptr(s.x), ctypes.byref(g), _lib.ptr(out),
                                               _lib.stream_ptr()), "gather_anchors")
        return out[:na]

    def piece_nbytes(self, extents, z0: int, z1: int, counts, bit_base: int):
        """Byte sizes (anchors, bit piece, outlier indices, outlier values) of
        the pieces slab [z0, z1) sends to the root: known on every rank from
        the all-gathered counts, so the gather needs no size exchange."""
        if z1 <= z0:
            na = 0
        else:
            g = make_geom(extents, default_layout(3))
            g.slab[0], g.slab[1] = z0, z1
            na = int(_lib.load().cszi_slab_anchor_count(ctypes.byref(g)))
        nbits, nout = int(counts[0]), int(counts[1])
        return 4 * na, 4 * ((bit_base + nbits + 31) // 32), 8 * nout, 4 * nout

    def pieces(self, s: SlabState, counts):
        """Variable-length payload pieces of this slab (device tensors)."""
        nbits, nout = int(counts[0]), int(counts[1])
        nw = (s.scratch.get("bit_base", 0) + nbits + 31) // 32  # whole words, phase-packed
        bits = s.scratch["bits"][: 4 * nw]
        oidx = s.scratch["oidx"][:nout]
        if s.scratch.get("nzmap") is not None and nout:
            # the bitmap encoder lists outlier indices only: values from the slab
            ny, nx = s.extents[1], s.extents[2]
            oval = s.x.reshape(-1)[oidx - s.z0 * ny * nx]
        else:
            oval = s.scratch["oval"][:nout]
        return bits, oidx, oval

    def assemble(self, s0: SlabState, anchors, bit_pieces, nbits, oidx, oval, pass2: bool,
                 alpha: float):
        """Root: raw payload (anchors ‖ lengths ‖ bitstream ‖ outliers) and
        pass-2 in one libcszi call (cszi_shard_assemble), header ->
        DeviceArchive.  One host read: the slab-0 ctl (flags, tuned
        configuration, payload length)."""
        t = _lib.torch()
        lib = _lib.load()
        st = _lib.stream_ptr()
        ctl = s0.scratch["ctl"]
        lengths = s0.scratch["lengths"]
        npc = len(nbits)
        vp = ctypes.c_void_p * npc
        u64 = ctypes.c_uint64 * npc
        na = [int(x.numel()) for x in anchors]
        no = [int(x.numel()) for x in oidx]
        starts = [0] * npc
        for i in range(1, npc):
            starts[i] = starts[i - 1] + int(nbits[i - 1])
        total_bits = sum(int(b) for b in nbits)
        nbins = int(lengths.numel())
        raw_cap = 4 * sum(na) + nbins + 4 * (total_bits // 32 + 2) + 8 + 12 * sum(no) + 64
        if pass2:
            raw = _lib.WS.get(raw_cap, "shard_raw")
            pay = t.empty(raw_cap + raw_cap // 128 + 16, dtype=t.uint8, device="cuda")
            ws = _lib.WS.get(int(lib.cszi_pass2_encode_workspace_size(raw_cap)), "p2_enc")
        else:
            raw = pay = t.empty(raw_cap, dtype=t.uint8, device="cuda")
            ws = None
        ptrs = lambda xs: vp(*[x.data_ptr() if x.numel() else 0 for x in xs])  # noqa: E731
        _lib.check(lib.cszi_shard_assemble(
            npc, ptrs(anchors), u64(*na), _lib.ptr(lengths), nbins, ptrs(bit_pieces),
            u64(*starts), u64(*[int(b) for b in nbits]), ptrs(oidx), ptrs(oval), u64(*no),
            1 if pass2 else 0, _lib.ptr(raw), raw_cap, _lib.ptr(pay),
            _lib.ptr(ws) if ws is not None else None, ws.numel() if ws is not None else 0,
            ctl.ptr, st), "shard_assemble")
        c = ctl.fetch()
        if c.flags & _lib.F_EB_NONPOSITIVE:
            raise Inconsistent("absolute error bound must be positive")
        if c.flags & _lib.F_LENGTH_OVERFLOW:
            raise LengthOverflow("a symbol would need more than 32 bits")
        if c.flags & _lib.F_EMPTY_HISTOGRAM:
            raise EmptyHistogram("cannot build a codebook from all-zero counts")
        sec = (4 * sum(na), nbins, (total_bits + 7) // 8, 8 + 12 * sum(no))
        payload = pay[: int(c.payload_len)]
        header = pack_header(3, PREDICTOR_INTERP, EB_REL if s0.mode == "rel" else EB_ABS, pass2,
                             0, ctl_variants(c, 3), ctl_order(c, 3), s0.radius, 8, s0.extents,
                             float(s0.eb), float(c.eb_abs), alpha, sec, int(payload.numel()))
        return DeviceArchive(header=header, payload=payload)


# ---------------------------------------------------------------------------
# orchestration
# ---------------------------------------------------------------------------
def compress_slabs(states: list, comm, backend=None, pass2: bool = True):
    """Run the sharded compress over this process's slabs.  Returns the
    archive (backend.assemble) on the root (the first slab's process), else
    None."""
    out = compress_slabs_batch([states], comm, backend, pass2)
    return None if out is None else out[0]


def _batched(comm, per_snap, op, split_sizes=None):
    """One collective for a batch of snapshots: per_snap[k][i] is local slab
    i's tensor for snapshot k.  The snapshot tensors of each slab are
    concatenated, reduced / gathered once, and split back."""
    t = _lib.torch()
    K = len(per_snap)
    sizes = [x.numel() for x in per_snap[0]] if split_sizes is None else split_sizes
    cat = [t.cat([per_snap[k][i].reshape(-1) for k in range(K)]) for i in range(len(per_snap[0]))]
    if op == "gather":
        res = comm.allgather(cat)[0]  # list over ranks
        n = sizes[0]
        return [[r[k * n:(k + 1) * n] for r in res] for k in range(K)]
    comm.allreduce(cat, op)
    return [[c[k * sizes[i]:(k + 1) * sizes[i]] for i, c in enumerate(cat)] for k in range(K)]


def compress_slabs_batch(batch: list, comm, backend=None, pass2: bool = True):
    """Sharded compress of a batch of snapshots with one collective per stage
    for the whole batch (SURVEY §8e "Expected scaling": one K x 2R histogram
    all-reduce instead of K).  batch[k] is the list of this process's slab
    states of snapshot k (same slab layout for every snapshot).  Returns the
    list of K archives on the root, else None.

    Host round trips per batch: the bit lengths of the slab pieces (every
    slab packs at its global bit phase) and the per-slab (bits, outliers)
    counts -- both one small device->host read for the whole batch; a
    relative bound needs the range on the device only, so the non-finite
    check rides on the first of those reads."""
    t = _lib.torch()
    backend = backend or GpuSlabBackend()
    K = len(batch)
    if (isinstance(backend, GpuSlabBackend) and getattr(comm, "world", 0) == 1
            and len(batch[0]) == 1 and batch[0][0].z0 == 0
            and batch[0][0].z1 >= batch[0][0].extents[0]):
        # one rank holding the whole field: nothing to shard -- the
        # single-GPU pipeline (one graph per snapshot), the same bytes
        from .grid import Dims, Grid
        from .pipeline import compress_device

        return [compress_device(Grid(Dims(st.extents), st.x), st.eb, st.mode, pass2=pass2,
                                quant_radius=st.radius) for (st,) in batch]
    # (1) range: K x 3 keys in one all-reduce
    keys = _batched(comm, [[backend.range_keys(s) for s in states] for states in batch], "min")
    for states, ks in zip(batch, keys):
        for s, k in zip(states, ks):
            backend.set_range(s, k)
    key0 = t.stack([ks[0].reshape(-1) for ks in keys])  # K x 3, identical on every slab
    host_keys = None
    if any(states[0].mode != "rel" for states in batch):
        host_keys = key0.cpu().numpy().astype(np.int64)
        _raise_nonfinite(host_keys)
    alphas = []
    for k, states in enumerate(batch):
        s0 = states[0]
        # alpha: rel mode -> compute_alpha(eb); abs mode -> from the global range
        if s0.mode == "rel":
            alphas.append(compute_alpha(float(s0.eb)))
        else:
            from ._keys import key_to_float

            k0 = host_keys[k]
            rng = key_to_float(int(-k0[1])) - key_to_float(int(k0[0]))
            alphas.append(compute_alpha(float(s0.eb) / rng if rng > 0 else float(s0.eb)))
    # (2) tuner samples
    samp = _batched(comm, [[backend.samples(s) for s in states] for states in batch], "sum")
    for states, vs, a in zip(batch, samp, alphas):
        for s, v in zip(states, vs):
            backend.tune(s, v, a)
    # (3) histograms -> shared codebooks: one K x 2R all-reduce
    hists = [[backend.predict(s) for s in states] for states in batch]
    phased = hasattr(backend, "piece_bits")
    local_h = [[h.clone() for h in hs] for hs in hists] if phased else None
    hists = _batched(comm, hists, "sum")
    for states, hs in zip(batch, hists):
        for s, h in zip(states, hs):
            backend.codebook(s, h)
    ranks = _local_ranks(comm, batch[0])
    # (4) bit / outlier counts.  A phase-packing backend first exchanges each
    # slab's stream length (local histogram . code lengths, known before any
    # packing) so every slab packs at its global bit phase and the root
    # merges whole words instead of bit-shifting the pieces.
    bases = None
    if phased:
        pb = _batched(comm, [[backend.piece_bits(s, h) for s, h in zip(states, lh)]
                             for states, lh in zip(batch, local_h)], "gather")
        allpb = t.stack([t.cat([p.reshape(-1) for p in pbk]) for pbk in pb])  # K x world
        if host_keys is None:  # first host read: piece lengths + the range keys
            both = t.cat([allpb.reshape(-1).to(key0.device), key0.reshape(-1)]).cpu().numpy()
            nk = allpb.numel()
            allpb_h = both[:nk].reshape(K, -1).astype(np.int64)
            host_keys = both[nk:].reshape(K, 3).astype(np.int64)
            _raise_nonfinite(host_keys)
        else:
            allpb_h = allpb.cpu().numpy().astype(np.int64)
        starts = np.concatenate([np.zeros((K, 1), np.int64), np.cumsum(allpb_h, 1)[:, :-1]], 1)
        bases = starts % 32
        counts = [[backend.encode(s, bit_base=int(bases[k][r])) for s, r in zip(states, ranks)]
                  for k, states in enumerate(batch)]
    else:
        counts = [[backend.encode(s) for s in states] for states in batch]
    allc = _batched(comm, counts, "gather")
    allc_h = t.stack([t.stack([c.reshape(-1) for c in ck]) for ck in allc]).cpu().numpy()
    if host_keys is None:
        host_keys = key0.cpu().numpy().astype(np.int64)
        _raise_nonfinite(host_keys)
    # (5) pieces to the root
    if (pass2 and isinstance(backend, GpuSlabBackend) and allc_h.shape[1] > 1
            and _pass2_split_pays(allc_h)):
        got = _pass2_split(comm, backend, batch, allc_h, ranks, alphas)
        if got != "fallback":
            return got
    if hasattr(backend, "piece_nbytes") and bases is not None:
        return _gather_packed(comm, backend, batch, allc_h, bases, ranks, alphas, pass2)
    out = []
    for states, ck, a in zip(batch, allc_h, alphas):
        anchors = comm.gather([backend.anchors(s) for s in states])
        pieces = [backend.pieces(s, c) for s, c in zip(states, [ck[i] for i in ranks])]
        bits = comm.gather([p[0] for p in pieces])
        oidx = comm.gather([p[1] for p in pieces])
        oval = comm.gather([p[2] for p in pieces])
        if anchors is None:
            out.append(None)
            continue
        nbits = [int(c[0]) for c in ck]
        out.append(backend.assemble(states[0], anchors, bits, nbits, oidx, oval, pass2, a))
    return None if out[0] is None else out


# Distributed pass-2 pays once the bitstream is long enough that the root's
# pass-2 encode (and the gather of raw pieces) outweighs a few host round
# trips; PASS2_SPLIT_MIN_BYTES = 0 forces it (tests).
PASS2_SPLIT_MIN_BYTES = 48 << 20


def _pass2_split_pays(allc_h) -> bool:
    bits = int(allc_h[:, :, 0].sum(axis=1).max())
    return bits // 8 >= PASS2_SPLIT_MIN_BYTES


def _pass2_split(comm, backend, batch, allc_h, ranks, alphas):
    """Pass-2 encoded where the pieces live (pass2.py:30-67).

    The zero-run codec has a segment boundary right after every run of >= 2
    zero bytes that is followed by a nonzero byte, whatever precedes the run,
    so the raw payload encodes piecewise to the same bytes when cut there.
    Every slab r >= 1 finds the first such cut c_r in the bytes of its bit
    piece that no neighbour shares (the last slab also the last cut e); slab
    r encodes [c_r, c_{r+1}) (slab 0 from the payload start, with the anchor
    and code-length sections in front; slab r borrows slab r+1's piece bytes
    up to c_{r+1}, ORing the shared word), the root encodes the last slab's
    bytes after e plus the outlier section, and concatenates.  Collectives
    per batch: an all-gather of the cuts, an all-gather of the borrowed
    prefixes, a gather of the anchors and a gather of the encoded pieces.
    Returns the archives on the root, None elsewhere, or "fallback" (on every
    rank alike) when a slab has no cut."""
    t = _lib.torch()
    lib = _lib.load()
    st = _lib.stream_ptr()
    from .pass2 import encode_device

    K = len(batch)
    W = allc_h.shape[1]
    geo = []
    for k in range(K):
        nb = [int(allc_h[k][r][0]) for r in range(W)]
        starts = [sum(nb[:r]) for r in range(W)]
        total = sum(nb)
        nbytes = (total + 7) // 8
        gb = [4 * (starts[r] // 32) for r in range(W)]
        ge = [gb[r] + 4 * ((starts[r] % 32 + nb[r] + 31) // 32) for r in range(W)]
        geo.append((nb, total, nbytes, gb, ge))
    # (1) cuts in the bytes no neighbour shares: the first word of a piece
    # holds the previous piece's last bits, the last word the next piece's first
    cuts = []
    for k in range(K):
        nb, total, nbytes, gb, ge = geo[k]
        row = []
        for i, r in enumerate(ranks):
            out = t.full((4,), -1, dtype=t.int64, device="cuda")
            if r > 0:
                hi = (min(ge[r], nbytes) if r == W - 1 else ge[r] - 4) - gb[r]
                bits = batch[k][i].scratch["bits"]
                _lib.check(lib.cszi_find_cuts(_lib.ptr(bits), 4, max(hi, 4), _lib.ptr(out), st),
                           "find_cuts")
            row.append(out[:2])
        cuts.append(row)
    allcut = _batched(comm, cuts, "gather")
    cut_h = t.stack([t.stack([c.reshape(-1) for c in ck]) for ck in allcut]).cpu().numpy()
    c = [[0] * (W + 1) for _ in range(K)]
    for k in range(K):
        nb, total, nbytes, gb, ge = geo[k]
        for r in range(1, W):
            if cut_h[k][r][0] < 0:
                return "fallback"
            c[k][r] = gb[r] + int(cut_h[k][r][0])
        last = int(cut_h[k][W - 1][1])
        if last < 0 or gb[W - 1] + last < c[k][W - 1]:
            return "fallback"
        c[k][W] = gb[W - 1] + last  # the root encodes from here to the end
    # (2) borrowed prefixes: slab r >= 1 lends bytes [gb_r, c_r) of its piece
    plen = [[c[k][r] - geo[k][3][r] if r > 0 else 0 for r in range(W)] for k in range(K)]
    pmax = max(max(p) for p in plen) or 1
    lend = []
    for i, r in enumerate(ranks):
        buf = t.zeros(K * pmax, dtype=t.uint8, device="cuda")
        for k in range(K):
            if plen[k][r]:
                buf[k * pmax:k * pmax + plen[k][r]] = batch[k][i].scratch["bits"][:plen[k][r]]
        lend.append(buf)
    lent = comm.allgather(lend)[0]  # list over ranks
    # (3) anchors to the root (the root's piece carries the anchor section)
    anc_local = [t.cat([backend.anchors(batch[k][i]).reshape(-1).view(t.uint8)
                        for k in range(K)]) for i in range(len(ranks))]
    na_b = [[backend.piece_nbytes(batch[0][0].extents, *_slab_of(batch, comm, r, W),
                                  allc_h[k][r], 0)[0] for r in range(W)] for k in range(K)]
    anc_got = comm.gather(anc_local, sizes=[sum(na_b[k][r] for k in range(K)) for r in range(W)])
    # (4) each slab encodes its cut range
    enc = []
    for i, r in enumerate(ranks):
        parts = []
        for k in range(K):
            nb, total, nbytes, gb, ge = geo[k]
            s_ = batch[k][i]
            a, e = c[k][r], c[k][r + 1]
            seg = t.zeros(max(e - a, 0) + 8, dtype=t.uint8, device="cuda")
            bits = s_.scratch["bits"]
            lo, hi = max(a, gb[r]), min(e, ge[r])
            if hi > lo:
                seg[lo - a:hi - a] = bits[lo - gb[r]:hi - gb[r]]
            if r + 1 < W and plen[k][r + 1]:
                q0 = gb[r + 1]
                pre = lent[r + 1][k * pmax:k * pmax + plen[k][r + 1]]
                seg[q0 - a:q0 - a + pre.numel()].bitwise_or_(pre)
            seg = seg[:max(e - a, 0)]
            if r == 0:  # anchor section (every slab, lattice order) + code lengths in front
                pieces = []
                for rr in range(W):
                    o = sum(na_b[kk][rr] for kk in range(k))
                    pieces.append(anc_got[rr][o:o + na_b[k][rr]])
                seg = t.cat(pieces + [s_.scratch["lengths"], seg])
            out, m = encode_device(seg, int(seg.numel()))
            parts.append(out[:m])
        enc.append(parts)
    # (5) encoded pieces, the last slab's tail bytes and the outliers to the root
    packed = []
    meta = []
    for i, r in enumerate(ranks):
        chunks = []
        row = []
        for k in range(K):
            nb, total, nbytes, gb, ge = geo[k]
            s_ = batch[k][i]
            tail = s_.scratch["bits"][c[k][W] - gb[r]:nbytes - gb[r]] if r == W - 1 else \
                s_.scratch["bits"][:0]
            _, oi, ov = backend.pieces(s_, allc_h[k][r])
            for x in (enc[i][k], tail, oi.reshape(-1).view(t.uint8), ov.reshape(-1).view(t.uint8)):
                chunks.append(x)
            row += [enc[i][k].numel(), tail.numel(), oi.numel()]
        meta.append(t.tensor(row, dtype=t.int64, device="cuda").view(t.uint8))
        packed.append(t.cat([meta[-1]] + chunks))
    got = comm.gather(packed)
    if got is None:
        return None
    out = []
    for k in range(K):
        s0 = batch[k][0]
        nb, total, nbytes, gb, ge = geo[k]
        encs, oidx, oval, tail = [], [], [], None
        for r in range(W):
            buf = got[r]
            m = buf[:24 * K].clone().view(t.int64).cpu().numpy().reshape(K, 3)
            o = 24 * K
            for kk in range(K):
                le, lt, no = (int(v) for v in m[kk])
                if kk == k:
                    encs.append(buf[o:o + le])
                    if r == W - 1:
                        tail = buf[o + le:o + le + lt]
                    oidx.append(buf[o + le + lt:o + le + lt + 8 * no].clone().view(t.int64))
                    oval.append(buf[o + le + lt + 8 * no:o + le + lt + 12 * no].clone()
                                .view(t.float32))
                o += le + lt + 12 * no
        kt = sum(int(x.numel()) for x in oidx)
        osec = t.empty(8 + 12 * kt, dtype=t.uint8, device="cuda")
        idx = t.cat(oidx) if kt else t.zeros(1, dtype=t.int64, device="cuda")
        val = t.cat(oval) if kt else t.zeros(1, dtype=t.float32, device="cuda")
        _lib.check(lib.cszi_pack_outliers(_lib.ptr(idx), _lib.ptr(val), kt, _lib.ptr(osec), st),
                   "pack_outliers")
        last = t.cat([tail, osec])
        tout, tm = encode_device(last, int(last.numel()))
        payload = t.cat(encs + [tout[:tm]])
        ctl = s0.scratch["ctl"]
        cc = ctl.fetch()
        if cc.flags & _lib.F_EB_NONPOSITIVE:
            raise Inconsistent("absolute error bound must be positive")
        if cc.flags & _lib.F_LENGTH_OVERFLOW:
            raise LengthOverflow("a symbol would need more than 32 bits")
        if cc.flags & _lib.F_EMPTY_HISTOGRAM:
            raise EmptyHistogram("cannot build a codebook from all-zero counts")
        na_total = sum(na_b[k][r] for r in range(W))
        nbins = int(s0.scratch["lengths"].numel())
        sec = (na_total, nbins, nbytes, 8 + 12 * kt)
        header = pack_header(3, PREDICTOR_INTERP, EB_REL if s0.mode == "rel" else EB_ABS, True,
                             0, ctl_variants(cc, 3), ctl_order(cc, 3), s0.radius, 8, s0.extents,
                             float(s0.eb), float(cc.eb_abs), alphas[k], sec,
                             int(payload.numel()))
        out.append(DeviceArchive(header=header, payload=payload))
    return out


def _slab_of(batch, comm, r, W):
    if isinstance(comm, SimComm):
        s = batch[0][r]
        return s.z0, s.z1
    return slab_bounds(batch[0][0].extents[0], W)[r]


def _raise_nonfinite(host_keys):
    for k0 in host_keys:
        if int(k0[2]) != INT64_MAX:
            raise NonFiniteValue(int(k0[2]))


def _gather_packed(comm, backend, batch, allc_h, bases, ranks, alphas, pass2):
    """One gather for the whole batch: every slab packs (anchors, bit piece,
    outlier indices, outlier values) of all K snapshots into one byte
    buffer; the sizes of every slab's parts follow from the all-gathered
    counts, so no rank exchanges sizes and the root splits the buffers."""
    t = _lib.torch()
    K = len(batch)
    s0 = batch[0][0]
    world = allc_h.shape[1]
    if isinstance(comm, SimComm):
        bounds = [(s.z0, s.z1) for s in batch[0]]
    else:
        bounds = slab_bounds(s0.extents[0], world)
    sizes = [[backend.piece_nbytes(s0.extents, bounds[r][0], bounds[r][1], allc_h[k][r],
                                   int(bases[k][r])) for r in range(world)] for k in range(K)]
    packed = []
    for i, r in enumerate(ranks):
        parts = []
        for k in range(K):
            st = batch[k][i]
            a = backend.anchors(st)
            b, oi, ov = backend.pieces(st, allc_h[k][r])
            for x, nb in zip((a, b, oi, ov), sizes[k][r]):
                v = x.reshape(-1).view(t.uint8)
                assert v.numel() == nb, (v.numel(), nb)
                parts.append(v)
        packed.append(t.cat(parts) if parts else t.empty(0, dtype=t.uint8, device="cuda"))
    per_rank = [sum(sum(sizes[k][r]) for k in range(K)) for r in range(world)]
    got = comm.gather(packed, sizes=per_rank)
    if got is None:
        return None
    out = []
    offs = [0] * world
    for k in range(K):
        anchors, bits, oidx, oval = [], [], [], []
        for r in range(world):
            buf = got[r]
            o = offs[r]
            na, nb, ni, nv = sizes[k][r]
            anchors.append(buf[o:o + na].view(t.float32))
            bits.append(buf[o + na:o + na + nb])
            # (an int64 view needs an 8-byte aligned offset: copy)
            oidx.append(buf[o + na + nb:o + na + nb + ni].clone().view(t.int64))
            oval.append(buf[o + na + nb + ni:o + na + nb + ni + nv].view(t.float32))
            offs[r] = o + na + nb + ni + nv
        nbits = [int(allc_h[k][r][0]) for r in range(world)]
        out.append(backend.assemble(batch[k][0], anchors, bits, nbits, oidx, oval, pass2,
                                    alphas[k]))
    return out


def _local_ranks(comm, states):
    if isinstance(comm, SimComm):
        return list(range(len(states)))
    return [comm.rank]


def compress_sharded(local_x, extents, z0: int, z1: int, eb: float, mode: str = "rel",
                     pass2: bool = True, quant_radius: int = 512, group=None):
    """torch.distributed entry point: this rank owns planes [z0, z1) of the
    global 3-D field ``extents``; ``local_x`` holds planes [z0, min(z1+1, nz))."""
    st = SlabState(x=local_x.contiguous(), extents=tuple(int(e) for e in extents), z0=z0, z1=z1,
                   eb=float(eb), mode=mode, radius=int(quant_radius))
    return compress_slabs([st], TorchComm(group), pass2=pass2)


def compress_sharded_batch(local_xs, extents, z0: int, z1: int, eb: float, mode: str = "rel",
                           pass2: bool = True, quant_radius: int = 512, group=None, comm=None):
    """torch.distributed entry point for a batch of snapshots of one shape
    (e.g. the 8 RTM snapshots): this rank owns planes [z0, z1) of every
    snapshot; local_xs[k] holds planes [z0, min(z1+1, nz)) of snapshot k.
    One collective per stage for the whole batch.  -> list of archives on
    rank 0, None elsewhere."""
    batch = [[SlabState(x=x.contiguous(), extents=tuple(int(e) for e in extents), z0=z0, z1=z1,
                        eb=float(eb), mode=mode, radius=int(quant_radius))] for x in local_xs]
    return compress_slabs_batch(batch, comm if comm is not None else TorchComm(group),
                                pass2=pass2)


def compress_simulated_batch(xs, world: int, eb: float, mode: str = "rel", pass2: bool = True,
                             quant_radius: int = 512):
    """compress_sharded_batch with all ``world`` slabs in this process."""
    batch = []
    for x in xs:
        nz = int(x.shape[0])
        batch.append([SlabState(x=x[z0:min(z1 + 1, nz)].contiguous(), extents=tuple(x.shape),
                                z0=z0, z1=z1, eb=float(eb), mode=mode, radius=int(quant_radius))
                      for z0, z1 in slab_bounds(nz, world)])
    return compress_slabs_batch(batch, SimComm(world), pass2=pass2)


def compress_simulated(x, world: int, eb: float, mode: str = "rel", pass2: bool = True,
                       quant_radius: int = 512):
    """All ``world`` slabs of a 3-D CUDA field in this process (GPU-count
    determinism check on one device)."""
    nz = int(x.shape[0])
    states = []
    for z0, z1 in slab_bounds(nz, world):
        states.append(SlabState(x=x[z0:min(z1 + 1, nz)].contiguous(), extents=tuple(x.shape),
                                z0=z0, z1=z1, eb=float(eb), mode=mode, radius=int(quant_radius)))
    return compress_slabs(states, SimComm(world), pass2=pass2)


# ---------------------------------------------------------------------------
# sharded decompress: every rank holds the archive, synchronises
# the Huffman stream, decodes only its slab's symbol window and reconstructs
# its planes.  No exchange: the archive is the shared input.
# ---------------------------------------------------------------------------
def decompress_slab(data, z0: int, z1: int):
    """Planes [z0, z1) of a 3-D archive as a (z1 - z0, ny, nx) CUDA tensor."""
    from .pipeline import decompress_device

    return decompress_device(data, slab=(z0, z1))


class _SplitSlab:
    """One slab's split-decompress state (workspace, ctl, chunk range)."""

    def __init__(self, plan, z0: int, z1: int, h0: int, h1: int):
        t = _lib.torch()
        lib = _lib.load()
        self.z0, self.z1, self.h0, self.h1 = z0, z1, h0, h1
        self.geom = make_geom(plan["extents"], default_layout(3))
        self.geom.slab[0], self.geom.slab[1] = z0, z1
        self.ctl = _lib.DeviceCtl()
        self.ws = t.empty(int(lib.cszi_decompress_workspace_size(
            ctypes.byref(self.geom), plan["R"], plan["sec"], plan["plen"])),
            dtype=t.uint8, device="cuda")
        self.entry_used = t.zeros(1, dtype=t.int64, device="cuda")


def _split_plan(data):
    """Header checks and launch arguments shared by every slab, or None when
    the archive must take the single-rank path (host-side errors raise
    there, in the reference's order; other codecs / layouts / predictors)."""
    from .archive import HEADER_SIZE, PREDICTOR_INTERP, unpack_header
    from .pass2 import DEFAULT_CODEC
    from .pipeline import _host_checks, _split_input
    from .grid import Dims
    from .predictor import plan_levels

    head, d_payload, h_payload, total = _split_input(data)
    if total < HEADER_SIZE:
        return None
    h = unpack_header(head, total)
    if h.predictor != PREDICTOR_INTERP or h.rank != 3 or h.anchor_stride != 8:
        return None
    if h.pass2 and h.pass2_codec != DEFAULT_CODEC:
        return None
    err, layout = _host_checks(h, Dims(h.extents))
    if err is not None or h.sec_lens[1] != 2 * h.quant_radius:
        return None
    if d_payload is None:
        d_payload = _lib.to_device_u8(h_payload)
    if h.pass2 and sum(h.sec_lens) > 128 * d_payload.numel():
        return None
    if not h.pass2 and d_payload.numel() != sum(h.sec_lens):
        return None
    lp = plan_levels(layout.anchor_stride, h.eb_abs, h.alpha)
    return dict(h=h, payload=d_payload, plen=int(d_payload.numel()), pass2=1 if h.pass2 else 0,
                extents=tuple(h.extents), R=h.quant_radius,
                sec=(ctypes.c_uint64 * 4)(*h.sec_lens),
                leb=(ctypes.c_double * _lib.MAX_LEVELS)(*[v.eb for v in lp.levels]),
                nlev=len(lp.levels), var=(ctypes.c_int32 * 3)(*h.variants),
                order=(ctypes.c_int32 * 3)(*h.dim_order))


# The split saves each rank (1 - 1/world) of the whole-stream synchronisation
# (~80 us per 535K chunks on a B200) and costs a few host round trips and
# one all-gather (~150 us): worth it for long streams only.
SPLIT_MIN_SAVED_CHUNKS = 1 << 20


def split_pays(data, world: int) -> bool:
    """Whether decompress_sharded splits the Huffman synchronisation for
    this archive over `world` ranks."""
    from .archive import HEADER_SIZE, unpack_header

    if world < 2:
        return False
    head = data.header if isinstance(data, DeviceArchive) else bytes(data[:HEADER_SIZE])
    try:
        h = unpack_header(head, len(data))
    except Exception:
        return False
    M = (h.sec_lens[2] * 8 + 255) // 256
    return M * (world - 1) // world >= SPLIT_MIN_SAVED_CHUNKS


# The pass-2 decode of the payload splits as well once the payload is long
# (each rank: 1/world of the chunk tables, one all-gather, the chain resolve,
# and only the raw ranges it reads); PASS2 decode of a 2.7 MB payload takes
# ~100 us on one B200.
P2D_SPLIT_MIN_BYTES = 8 << 20


class _SplitPass2:
    """Pass-2 decode split by the encoded payload's 1 KiB chunks: tables of
    this rank's chunks, all-gathered; the chain resolve and the count scan on
    every rank; then each slab expands only the raw byte ranges it reads
    (its anchor planes, the code lengths, the bitstream of its Huffman chunk
    range and later of its symbol window, the outlier section)."""

    def __init__(self, plan, S, slabs, comm, world, hper):
        t = _lib.torch()
        lib = self.lib = _lib.load()
        st = _lib.stream_ptr()
        self.plan = plan
        n = plan["plen"]
        self.n = n
        Mp = self.Mp = int(lib.cszi_p2d_chunks(n))
        perp = -(-Mp // world)
        D = 129
        tab = t.empty(Mp * D, dtype=t.uint8, device="cuda")
        ctab = t.empty(Mp * D, dtype=t.int32, device="cuda")
        pay = _lib.ptr(plan["payload"])
        shares = []
        for (r, _, _) in slabs:
            p0, p1 = min(Mp, r * perp), min(Mp, (r + 1) * perp)
            _lib.check(lib.cszi_p2d_tables(pay, n, p0, p1, _lib.ptr(tab), _lib.ptr(ctab), st),
                       "p2d_tables")
            # share: the uint32 table first (4-byte aligned views), then the bytes
            sh = t.zeros(perp * 5 * D, dtype=t.uint8, device="cuda")
            if p1 > p0:
                sh[:(p1 - p0) * 4 * D] = ctab[p0 * D:p1 * D].view(t.uint8)
                sh[perp * 4 * D:perp * 4 * D + (p1 - p0) * D] = tab[p0 * D:p1 * D]
            shares.append(sh)
        got = comm.allgather(shares)[0]
        for r, g in enumerate(got):
            p0, p1 = min(Mp, r * perp), min(Mp, (r + 1) * perp)
            if p1 > p0:
                ctab[p0 * D:p1 * D] = g[:(p1 - p0) * 4 * D].view(t.int32)
                tab[p0 * D:p1 * D] = g[perp * 4 * D:perp * 4 * D + (p1 - p0) * D]
        self.E = t.empty(Mp, dtype=t.uint8, device="cuda")
        self.cnt = t.empty(Mp, dtype=t.int32, device="cuda")
        self.off = t.empty(Mp, dtype=t.int64, device="cuda")
        ws = t.empty(int(lib.cszi_p2d_resolve_scratch_size(n)), dtype=t.uint8, device="cuda")
        ctl = S[0].ctl
        _lib.check(lib.cszi_ctl_init(ctl.ptr, st), "ctl_init")
        _lib.check(lib.cszi_p2d_resolve(_lib.ptr(tab), _lib.ptr(ctab), n, _lib.ptr(self.E),
                                        _lib.ptr(self.cnt), _lib.ptr(self.off), _lib.ptr(ws),
                                        ctl.ptr, st), "p2d_resolve")
        c = ctl.fetch()
        h = plan["h"]
        self.raw_len = sum(h.sec_lens)
        self.ok = (int(c.raw_len) == self.raw_len and not (c.flags & _lib.F_P2_CORRUPT))
        self.off_h = self.off.cpu().numpy().tolist()
        sec = h.sec_lens
        self.head = sec[0] + sec[1]
        if not self.ok:
            return
        ny, nx = plan["extents"][1], plan["extents"][2]
        nz = plan["extents"][0]
        na1 = (ny - 1) // 8 + 1 + (1 if (ny - 1) % 8 else 0)
        na2 = (nx - 1) // 8 + 1 + (1 if (nx - 1) % 8 else 0)
        zl = list(range(0, nz, 8)) + ([nz - 1] if (nz - 1) % 8 else [])
        for s in S:
            rngs = [(sec[0], self.head),                                     # code lengths
                    (self.head + sec[2], self.raw_len)]                      # outlier section
            if s.z1 > s.z0:  # the anchor planes of the slab and its closing plane
                top = min(s.z1, nz - 1)
                k0 = s.z0 // 8
                k1 = max(i for i, zc in enumerate(zl) if zc <= top)
                rngs.append((4 * k0 * na1 * na2, 4 * (k1 + 1) * na1 * na2))
            if s.h1 > s.h0:  # the bitstream of the Huffman range (+ one chunk each side)
                rngs.append((self.head + max(0, (s.h0 - 1) * 32 - 8),
                             self.head + min(sec[2], (s.h1 + 1) * 32 + 16)))
            self._expand(s, rngs)

    def _expand(self, s, rngs):
        import bisect

        lib = self.lib
        raw = s.ws[int(lib.cszi_decompress_raw_offset(ctypes.byref(s.geom), self.plan["R"],
                                                      self.plan["sec"], self.n)):]
        cap = self.raw_len + 64
        for lo, hi in rngs:
            if hi <= lo:
                continue
            ja = max(0, bisect.bisect_right(self.off_h, lo) - 1)
            jb = bisect.bisect_left(self.off_h, hi)
            _lib.check(lib.cszi_p2d_expand(_lib.ptr(self.plan["payload"]), self.n,
                                           _lib.ptr(self.E), _lib.ptr(self.off),
                                           _lib.ptr(self.cnt), ja, jb, _lib.ptr(raw), cap,
                                           s.ctl.ptr, _lib.stream_ptr()), "p2d_expand")

    def expand_windows(self, S, X, K, plan):
        """The bitstream bytes of the chunks holding each slab's symbol window
        (plus its halo plane), known once the chunk records are gathered."""
        t = _lib.torch()
        ny, nx = plan["extents"][1], plan["extents"][2]
        nz = plan["extents"][0]
        nb = plan["h"].sec_lens[2]
        for s, x, k in zip(S, X, K):
            if s.z1 <= s.z0:
                continue
            w0, w1 = s.z0 * ny * nx, min(s.z1 + 1, nz) * ny * nx
            cum = t.cumsum(k.to(t.int64), 0)
            ja = int(t.searchsorted(cum, t.tensor([w0], device=cum.device), right=True).item())
            jb = int(t.searchsorted(cum - k.to(t.int64), t.tensor([w1], device=cum.device)).item())
            jb = max(jb - 1, ja)
            b_lo = int(x[ja - 1].item()) if ja > 0 else 0
            b_hi = int(x[min(jb, x.numel() - 1)].item())
            self._expand(s, [(self.head + max(0, b_lo // 8 - 8),
                              self.head + min(nb, b_hi // 8 + 16))])


def _split_pass2_decode(plan, S, slabs, comm, world, hper):
    p2 = _SplitPass2(plan, S, slabs, comm, world, hper)
    return p2 if p2.ok else None


def decompress_slabs_split(data, slabs, comm, world: int):
    """Sharded decompress with the Huffman synchronisation split by chunk
    ranges: this process's slabs [(rank, z0, z1), ...] each synchronise
    1/world of the stream's 256-bit chunks, the (exit, count, dead) records
    are all-gathered (one collective), a range whose assumed entry differs
    from its predecessor's true exit re-synchronises (rare: chains meet
    within a few codewords), then every slab writes its own symbol window
    and reconstructs its planes.  Returns [(z0, z1, tensor), ...] or None
    when the archive needs the single-rank path.  Bit-identical to
    decompress_device(slab=...) (tests/test_gpu_distributed.py)."""
    t = _lib.require_cuda()
    lib = _lib.load()
    st = _lib.stream_ptr()
    plan = _split_plan(data)
    if plan is None:
        return None
    M = int(lib.cszi_huff_chunks(plan["h"].sec_lens[2]))
    per = -(-M // world)
    S = [_SplitSlab(plan, z0, z1, min(M, r * per), min(M, (r + 1) * per)) for r, z0, z1 in slabs]
    pay = _lib.ptr(plan["payload"])
    args = lambda s: (pay, plan["plen"], plan["pass2"], plan["sec"], ctypes.byref(s.geom),  # noqa
                      plan["R"])
    X = [t.zeros(M, dtype=t.int64, device="cuda") for _ in S]
    K = [t.zeros(M, dtype=t.int32, device="cuda") for _ in S]
    D = [t.zeros(M, dtype=t.uint8, device="cuda") for _ in S]
    p2 = None
    if plan["pass2"] and plan["plen"] >= P2D_SPLIT_MIN_BYTES:
        p2 = _split_pass2_decode(plan, S, slabs, comm, world, per)
        if p2 is None:
            return None  # raw length mismatch: the single-rank path raises it
    for s, x, k, d in zip(S, X, K, D):
        if p2 is None:
            _lib.check(lib.cszi_decompress_prologue(*args(s), _lib.ptr(s.ws), s.ws.numel(),
                                                    s.ctl.ptr, st), "decompress_prologue")
        else:
            _lib.check(lib.cszi_decompress_prologue_raw(plan["plen"], plan["sec"],
                                                        ctypes.byref(s.geom), plan["R"],
                                                        _lib.ptr(s.ws), s.ws.numel(), s.ctl.ptr,
                                                        st), "decompress_prologue_raw")
    entries = [None] * len(S)  # None: speculative entry
    for _round in range(world + 1):
        for i, (s, x, k, d) in enumerate(zip(S, X, K, D)):
            if _round == 0 or entries[i] is not None:
                e = (1 << 64) - 1 if entries[i] is None else int(entries[i])
                _lib.check(lib.cszi_decompress_sync_range(
                    *args(s), s.h0, s.h1, e, _lib.ptr(x), _lib.ptr(k), _lib.ptr(d),
                    _lib.ptr(s.entry_used), _lib.ptr(s.ws), s.ws.numel(), s.ctl.ptr, st),
                    "decompress_sync_range")
        # one all-gather of every range's records: (exit, count | dead << 32) per chunk
        shares = []
        for s, x, k, d in zip(S, X, K, D):
            rec = t.zeros(2 * per, dtype=t.int64, device="cuda")
            nrec = s.h1 - s.h0
            if nrec:
                rec[0:2 * nrec:2] = x[s.h0:s.h1]
                rec[1:2 * nrec:2] = (k[s.h0:s.h1].to(t.int64) & 0xFFFFFFFF) | \
                    (d[s.h0:s.h1].to(t.int64) << 32)
            shares.append(rec)
        got = comm.allgather(shares)[0]  # list over ranks
        xa = t.cat([g[0::2] for g in got])[:M]
        kd = t.cat([g[1::2] for g in got])[:M]
        ka = (kd & 0xFFFFFFFF).to(t.int32)
        da = (kd >> 32).to(t.uint8)
        for x, k, d in zip(X, K, D):
            x.copy_(xa)
            k.copy_(ka)
            d.copy_(da)
        # ranges whose assumed entry is not their predecessor's true exit
        flags = []
        for s in S:
            if s.h0 == 0 or s.h1 <= s.h0:
                flags.append(t.zeros(1, dtype=t.int64, device="cuda"))
            else:
                flags.append((xa[s.h0 - 1:s.h0] != s.entry_used).to(t.int64))
        moved = [f.clone() for f in flags]
        comm.allreduce(moved, "max")
        if int(t.stack(moved).max().item()) == 0:
            break
        entries = [int(xa[s.h0 - 1].item()) if int(f.item()) else None for s, f in zip(S, flags)]
    if p2 is not None:  # the bit ranges of each slab's symbol window
        p2.expand_windows(S, X, K, plan)
    out = []
    for s, x, k, d in zip(S, X, K, D):
        c = s.ctl.fetch()
        if c.scratch[1] != 0:
            return None  # a range did not synchronise: the single-rank path (table mode)
        _lib.check(lib.cszi_decompress_write_window(*args(s), _lib.ptr(x), _lib.ptr(k),
                                                    _lib.ptr(d), _lib.ptr(s.ws), s.ws.numel(),
                                                    s.ctl.ptr, st), "decompress_write_window")
        ny, nx = plan["extents"][1], plan["extents"][2]
        y = t.empty((max(s.z1 - s.z0, 0), ny, nx), dtype=t.float32, device="cuda")
        if s.z1 > s.z0:
            _lib.check(lib.cszi_decompress_epilogue(*args(s), plan["leb"], plan["nlev"],
                                                    plan["var"], plan["order"], _lib.ptr(y),
                                                    _lib.ptr(s.ws), s.ws.numel(), s.ctl.ptr,
                                                    st), "decompress_epilogue")
        c = s.ctl.fetch()
        from .pipeline import _raise_device_flags

        _raise_device_flags(c, int(np.prod(plan["extents"])))
        if c.flags & _lib.F_OUTLIER_INDEX:
            raise IndexError("outlier index out of bounds for the grid")
        out.append((s.z0, s.z1, y))
    return out


def decompress_sharded(data, nz: int = None, group=None):
    """torch.distributed entry point: this rank's slab of the decompressed
    field -> (z0, z1, tensor).  ``nz`` defaults to the archive's extent.
    The Huffman synchronisation is split across the ranks
    (decompress_slabs_split); archives that need the single-rank path
    (other codecs, non-converging streams, host-side errors) decode the slab
    on each rank."""
    import torch.distributed as dist

    from .archive import HEADER_SIZE, unpack_header

    if nz is None:
        head = data[:HEADER_SIZE] if not isinstance(data, DeviceArchive) else data.header
        nz = unpack_header(bytes(head), len(data)).extents[0]
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    z0, z1 = slab_bounds(nz, world)[rank]
    if split_pays(data, world):
        got = decompress_slabs_split(data, [(rank, z0, z1)], TorchComm(group), world)
        if got is not None:
            return got[0]
    if z1 <= z0:  # more ranks than z tiles: this rank owns no planes
        t = _lib.require_cuda()
        head = data.header if isinstance(data, DeviceArchive) else bytes(data[:HEADER_SIZE])
        ext = unpack_header(head, len(data)).extents
        return z0, z1, t.empty((0, ext[1], ext[2]), dtype=t.float32, device="cuda")
    return z0, z1, decompress_slab(data, z0, z1)


def decompress_simulated(data, world: int, split: bool = False):
    """All ``world`` slabs in this process, concatenated (GPU-count
    determinism check on one device); ``split`` runs the chunk-range split
    of decompress_sharded over SimComm."""
    from .archive import HEADER_SIZE, unpack_header

    t = _lib.torch()
    head = data.header if isinstance(data, DeviceArchive) else bytes(data[:HEADER_SIZE])
    nz = unpack_header(head, len(data)).extents[0]
    bounds = slab_bounds(nz, world)
    if split:
        got = decompress_slabs_split(data, [(r, z0, z1) for r, (z0, z1) in enumerate(bounds)],
                                     SimComm(world), world)
        if got is not None:
            return t.cat([y for z0, z1, y in got if z1 > z0], 0)
    parts = [decompress_slab(data, z0, z1) for z0, z1 in bounds if z1 > z0]
    return t.cat(parts, 0)
