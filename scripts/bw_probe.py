#!/usr/bin/env python
"""Achievable HBM bandwidth vs transfer size (torch copy, L2 flushed by a
256 MB read before each timed copy) -- calibrates kernel-level roofline
fractions for working sets the size of one solver kernel."""
import torch


def main():
    flush = torch.ones(32 << 20, dtype=torch.float64, device="cuda")
    sink = torch.empty((), dtype=torch.float64, device="cuda")
    for mb in (8, 16, 37, 73, 146, 292, 1024, 4096):
        n = (mb << 20) // 16          # read mb/2 MB, write mb/2 MB
        a = torch.rand(n, dtype=torch.float64, device="cuda")
        b = torch.empty_like(a)
        ts = []
        for r in range(12):
            torch.sum(flush, dim=0, out=sink)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); b.copy_(a); e1.record(); e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        t = sorted(ts)[len(ts) // 2]
        print(f"copy {mb:5d} MB (read+write): {t:9.2f} us  {2 * n * 8 / t / 1e3:7.0f} GB/s")
        del a, b


if __name__ == "__main__":
    main()
