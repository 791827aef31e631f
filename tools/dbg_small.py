"""Small compress/decompress round trip vs the oracle (for compute-sanitizer runs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2312_05492_b200 as P
from oracle import oracle as O
shape = tuple(int(s) for s in (sys.argv[1] if len(sys.argv) > 1 else "64,64,64").split(","))
eb = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-3
z, y, x = np.meshgrid(*[np.arange(s, dtype=np.float64) for s in shape], indexing="ij")
d = (np.sin(2 * np.pi * 2 * z / shape[0]) + 0.7 * np.cos(2 * np.pi * 3 * y / shape[1])
     + 0.5 * np.sin(2 * np.pi * 1.5 * x / shape[2])).astype(np.float32)
g = P.Grid(P.Dims(shape), torch.from_numpy(d).cuda())
a = P.compress_device(g, eb)
blob = a.to_bytes()
ref = O.compress(d, eb)
print("compress match", blob == ref, len(blob), len(ref))
yv = P.decompress_device(a)
print("decompress match", yv.data.tobytes() == O.decompress(ref).tobytes())
