"""Quick GPU-vs-oracle parity probe (debug tool; the real gate is tests/)."""
import sys, time, traceback, hashlib
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
import paper_2312_05492_b200 as P
from oracle import oracle as O

def field(rng, shape, kind):
    axes = np.indices(shape).astype(np.float64)
    out = np.zeros(shape)
    for ax, coord in enumerate(axes):
        for _ in range(int(rng.integers(1, 4))):
            freq = rng.uniform(0.5, 3.0) / max(shape[ax], 2)
            out += rng.uniform(0.3, 1.0) * np.sin(2 * np.pi * freq * coord + rng.uniform(0, 6.28))
    if kind == "noisy":
        out = out + rng.normal(0, 0.2, shape)
    if kind == "const":
        out = np.full(shape, rng.uniform(-5, 5))
    return out.astype(np.float32)

fails = 0
def cmp(name, a, b):
    global fails
    if a != b:
        fails += 1
        print("MISMATCH", name, len(a) if hasattr(a,'__len__') else a, len(b) if hasattr(b,'__len__') else b)
        return False
    return True

g64 = O.sinusoid_64()
t0 = time.time()
try:
    blob = P.compress(P.Grid(P.Dims(g64.shape), g64), 1e-3)
    ref = O.compress(g64, 1e-3)
    print("sin64", len(blob), len(ref), blob == ref, hashlib.sha256(blob).hexdigest()[:16], time.time()-t0)
    if blob != ref:
        # stage diagnosis
        cfg = O.select_config(g64, "rel", 1e-3)
        codes, isout, _ = O.predict(g64, cfg)
        pc = P.PredictorConfig(P.ChunkLayout(8, 3, (8,8,32)), cfg.alpha, cfg.variants, cfg.dim_order, cfg.eb_abs)
        qf = P.compress_predict(P.Grid(P.Dims(g64.shape), g64), pc)
        d = np.nonzero(qf.codes != codes)[0]
        print(" codes diff count", d.size, d[:10], qf.codes[d[:10]], codes[d[:10]])
        print(" outliers", len(qf.outliers), int(isout.sum()))
        h = unpack = P.archive.unpack_header(blob, len(blob)); hr = P.archive.unpack_header(ref, len(ref))
        print(" hdr", h)
        print(" ref", hr)
    back = P.decompress(ref)
    rb = O.decompress(ref)
    cmp("sin64 decompress", back.data.tobytes(), rb.tobytes())
except Exception:
    traceback.print_exc(); fails += 1

rng = np.random.default_rng(5)
for i in range(60):
    rank = i % 3 + 1
    shape = tuple(int(rng.integers(1, 45)) for _ in range(rank))
    kind = ["smooth", "noisy", "const"][i % 3]
    data = field(rng, shape, kind)
    for mode, eb in (("rel", 1e-3), ("abs", 1e-2), ("rel", 1e-5)):
        try:
            blob = P.compress(P.Grid(P.Dims(shape), data), eb, mode=mode)
            ref = O.compress(data, eb, mode=mode)
            if not cmp(f"compress {shape} {kind} {mode} {eb}", blob, ref):
                continue
            back = P.decompress(blob)
            cmp(f"decompress {shape} {kind}", back.data.tobytes(), O.decompress(ref).tobytes())
        except Exception:
            print("EXC", shape, kind, mode, eb); traceback.print_exc(); fails += 1
print("fails", fails)
