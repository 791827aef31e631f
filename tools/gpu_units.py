"""Stage-level GPU-vs-oracle probes (debug tool)."""
import sys, traceback
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2312_05492_b200 as P
from oracle import oracle as O

rng = np.random.default_rng(1)
# pass2
for data in [b"", b"\x00"*5, b"AB", b"\x00", b"A\x00B", b"\x00"*300, bytes(range(1,256))*2,
             bytes(rng.integers(0, 3, 5000).astype(np.uint8)), bytes((rng.random(100000) < 0.7).astype(np.uint8))]:
    try:
        e = P.pass2_encode(data); r = O.pass2_encode(data)
        d = P.pass2_decode(r)
        print("p2", len(data), e == r, d == data, len(e), len(r))
    except Exception:
        traceback.print_exc()
# huffman
for vals in [[0]*10, [0,1,-1,0,1,1,0,-1]*8, list(rng.integers(-20,21,4000)), list(rng.integers(-3,4,100000)), list(rng.integers(0, 8, 50000))]:
    try:
        codes = np.asarray(vals, dtype=np.int32)
        R = 32
        h = P.build_histogram(codes, R); hr = O.histogram(codes, R)
        cb = P.build_codebook(h); lr = O.code_lengths(hr); cr = O.canonical(lr)
        print("hist", np.array_equal(h.counts, hr), "len", np.array_equal(cb.code_lengths, lr), "words", np.array_equal(cb.words, cr.words),
              "fc", np.array_equal(cb.first_code, cr.first_code), "fi", np.array_equal(cb.first_index, cr.first_index), np.array_equal(cb.sorted_symbols, cr.sorted_symbols))
        s, b = P.huffman_encode(codes, cb); sr, br = O.huffman_encode(codes, cr, R)
        print(" enc", s == sr, b, br, len(s), len(sr))
        dec = P.huffman_decode(sr, cb, codes.size)
        print(" dec", np.array_equal(dec, codes), dec[:8], codes[:8])
    except Exception:
        traceback.print_exc()
# predictor
g = O.sinusoid_64()
cfg = O.select_config(g, "rel", 1e-3)
codes, isout, rec = O.predict(g, cfg)
pc = P.PredictorConfig(P.ChunkLayout(8, 3, (8,8,32)), cfg.alpha, cfg.variants, cfg.dim_order, cfg.eb_abs)
qf = P.compress_predict(P.Grid(P.Dims(g.shape), g), pc)
d = np.nonzero(qf.codes != codes)[0]
print("predict codes diff", d.size, d[:10], qf.codes[d[:10]], codes[d[:10]], "outl", len(qf.outliers), int(isout.sum()))
st = P.profile_samples(P.Grid(P.Dims(g.shape), g))
print("profile", st.value_min, st.value_max, st.err_sum.tolist(), st.sample_count.tolist())
print("oracle ", O.profile(g)[:3], O.profile(g)[3].tolist())
back = P.decompress_predict(qf, pc, P.Dims(g.shape))
print("decompress_predict eq", back.data.tobytes() == rec.tobytes())
