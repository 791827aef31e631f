"""Non-zero histogram bins (Huffman leaves) of the bench workload."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2312_05492_b200 as P
from paper_2312_05492_b200 import _lib
from bench import smooth_field_gpu
al = lambda b: (b + 255) & ~255
for eb in (1e-2, 1e-3, 1e-4):
    x = smooth_field_gpu((512, 512, 512)); n = x.numel()
    P.compress_device(P.Grid(P.Dims(x.shape), x), eb)
    ws = _lib.WS._bufs[(0, "compress")]
    off = al(4 * 960) + al(2 * n + 32) + al(n // 8 + 16)
    h = ws[off: off + 8 * 1024].view(torch.int64)
    print(f"eb {eb}: nonzero bins {(h != 0).sum().item()}, total {h.sum().item()} (n {n})")
