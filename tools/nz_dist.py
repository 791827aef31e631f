"""Distribution of non-R symbols per 4096-symbol super-chunk and per 128-
symbol lane range in the bench workload (sizing the bitmap encoder)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2312_05492_b200 as P
from paper_2312_05492_b200 import _lib
from bench import smooth_field_gpu
x = smooth_field_gpu((512, 512, 512))
n = x.numel()
a = P.compress_device(P.Grid(P.Dims(x.shape), x), 1e-3)
print("outliers", len(P.parse_archive(a.to_bytes()).outliers))
ws = _lib.WS._bufs[(0, "compress")]
sym = ws[3840: 3840 + 2 * n].view(torch.int16)
nz = (sym != 512)
for name, g in (("super-chunk", 4096), ("lane", 128), ("row", 32)):
    k = nz.view(-1, g).sum(1).float()
    q = torch.quantile(k[:1 << 24], torch.tensor([0.5, 0.9, 0.99, 0.999], device=k.device))
    print(name, "mean", k.mean().item(), "max", k.max().item(), "q50/90/99/99.9", q.tolist(),
          "n>g/4", (k > g / 4).sum().item(), "of", k.numel())
