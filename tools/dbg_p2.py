"""Pass-2 decode on the GPU vs the oracle on payloads of the bench field."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
import paper_2312_05492_b200 as P
from paper_2312_05492_b200 import pass2 as P2
rng = np.random.default_rng(1)
cases = []
for n in (5000, 70000, 300000):
    raw = (rng.random(n) < 0.15).astype(np.uint8) * rng.integers(1, 256, n, dtype=np.uint8)
    cases.append(("rand%d" % n, raw.tobytes()))
shape = (256, 256, 256)
d = O.smooth_field(shape)
blob = O.compress(d, 1e-3, pass2=False)
cases.append(("field", blob[112:]))
for name, raw in cases:
    enc = O.pass2_encode(raw)
    got = P2._zero_run_decode(enc) if hasattr(P2, "_zero_run_decode") else P2.pass2_decode(enc, 0)
    ok = got == raw
    print(name, len(raw), len(enc), "ok" if ok else "MISMATCH")
    if not ok:
        a = np.frombuffer(got, np.uint8); b = np.frombuffer(raw, np.uint8)
        m = min(len(a), len(b)); bad = np.nonzero(a[:m] != b[:m])[0]
        print("  len", len(a), len(b), "first bad", bad[:10], "count", len(bad))
        if len(bad):
            i = bad[0]; print("  got", a[i-4:i+12], "want", b[i-4:i+12])
