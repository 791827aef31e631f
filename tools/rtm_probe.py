"""bench.py's RTM x 8 leg run on its own, three times, with the caching
allocator's counters (a slow outlier of that leg inside a full bench run was
not reproducible here).  Usage: rtm_probe.py"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2312_05492_b200 as P
args = argparse.Namespace(steps=20, warmup=3, eb=1e-3)
for i in range(3):
    r = bench.rtm8_leg(args, P, 0, 1)
    s = torch.cuda.memory_stats()
    print(i, r['compress_ms_per_step'], r['decompress_ms_per_step'], 'retries', s.get('num_alloc_retries'), 'cudaMalloc', s.get('num_device_alloc'), 'frees', s.get('num_device_free'), flush=True)
