"""Density of non-R quant-codes in the bench workload: fraction of symbols
and of 32-symbol rows holding one (sizing the non-R bitmap encoder)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2312_05492_b200 as P
from paper_2312_05492_b200 import _lib
from bench import smooth_field_gpu
for eb in (1e-3, 1e-4, 1e-5):
    x = smooth_field_gpu((512, 512, 512))
    n = x.numel()
    P.compress_device(P.Grid(P.Dims(x.shape), x), eb)
    ws = _lib.WS._bufs[(0, "compress")]
    sym = ws[3840: 3840 + 2 * n].view(torch.int16).view(-1, 32)
    nz = sym != 512
    print(f"eb {eb}: nonR symbols {nz.float().mean().item():.4f}, rows with nonR "
          f"{nz.any(1).float().mean().item():.4f}, 8-groups {nz.view(-1,8).any(1).float().mean().item():.4f}")
