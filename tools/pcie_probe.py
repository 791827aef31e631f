"""Host<->device copy rates for the e2e legs: one 537 MB pinned copy per
direction against the same bytes split over k streams (copy-engine
parallelism).  Usage: pcie_probe.py [MB]"""
import sys
import time

import torch


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def main():
    mb = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    n = mb * (1 << 20)
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for k in (1, 2, 4, 8):
        streams = [torch.cuda.Stream() for _ in range(k)]
        step = (n + k - 1) // k

        def h2d():
            for i, s in enumerate(streams):
                with torch.cuda.stream(s):
                    d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)

        def d2h():
            for i, s in enumerate(streams):
                with torch.cuda.stream(s):
                    h[i * step:(i + 1) * step].copy_(d[i * step:(i + 1) * step], non_blocking=True)

        th, td = timed(h2d), timed(d2h)
        print(f"{mb} MB over {k} stream(s): H2D {n / th / 1e9:6.2f} GB/s  D2H {n / td / 1e9:6.2f} GB/s",
              flush=True)


if __name__ == "__main__":
    main()
