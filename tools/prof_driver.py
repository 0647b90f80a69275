#!/usr/bin/env python3
"""Small driver for ncu / timing experiments: runs `--iters` forward+backward
steps of a BASELINE config through the C ABI (no graphs, so every launch is a
separate ncu result), optionally timing an empty-kernel graph to measure the
per-node launch overhead.

    python tools/prof_driver.py --config metric --iters 6
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="metric")
    p.add_argument("--iters", type=int, default=6)
    p.add_argument("--sets", type=int, default=4)
    p.add_argument("--overhead", action="store_true")
    a = p.parse_args()
    torch.cuda.set_device(0)
    work = bench.make_work(bench.cfg_key(a.config), 0)
    sets = [work.alloc_set(0) for _ in range(a.sets)]
    for i in range(a.iters):
        s = sets[i % a.sets]
        work.fwd(s)
        work.bwd(s)
    torch.cuda.synchronize()
    if a.overhead:
        x = torch.zeros(1, device="cuda")
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        with torch.cuda.stream(st), torch.cuda.graph(g, stream=st):
            for _ in range(200):
                x.add_(1.0)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        print(f"empty-kernel graph node: {e0.elapsed_time(e1) * 1e3 / 2000:.3f} us per node")


if __name__ == "__main__":
    main()
