import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2312_05492_b200 as P
from oracle import oracle as O
for shape in [(20, 24, 500), (17, 9, 33), (27, 18, 235)]:
    rng = np.random.default_rng(1)
    z,y,x = np.meshgrid(*[np.arange(s) for s in shape], indexing='ij')
    data = (np.sin(z/7.)+np.cos(y/5.)+np.sin(x/11.)).astype(np.float32)
    blob = P.compress(P.Grid(P.Dims(shape), data), 1e-3)
    print(shape, "compress ok", blob == O.compress(data, 1e-3), flush=True)
    out = P.decompress(blob)
    print(shape, "decompress ok", out.data.tobytes() == O.decompress(blob).tobytes(), flush=True)
