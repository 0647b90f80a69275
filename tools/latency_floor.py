#!/usr/bin/env python3
"""Latency floor of the headline step (backbone L=700): per-launch time of the
packed forward and coordinate backward against the batch size, next to an
empty kernel, all in CUDA graphs of back-to-back launches (inputs L2-warm:
this measures the per-chain critical path, not HBM).

    python tools/latency_floor.py [--L 700] [--reps 50]

One line per (kernel, B): us per launch.  B = 1 is one chain's critical path
alone; B = 148 is one chain per SM; B = 256 is the metric (108 SMs run two
chains); B = 296 is two chains on every SM.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1812_01108_b200 import _abi  # noqa: E402


def per_launch_us(fn, reps):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(reps):
            fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    out = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        with torch.cuda.stream(st):
            g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) * 1e3 / reps)
    out.sort()
    return out[len(out) // 2]


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--L", type=int, default=700)
    p.add_argument("--reps", type=int, default=50)
    p.add_argument("--B", type=int, nargs="*", default=[1, 74, 148, 256, 296])
    a = p.parse_args()
    torch.cuda.set_device(0)
    one = torch.zeros(1, device="cuda")
    print(f"empty kernel (1-element fill): {per_launch_us(lambda: one.fill_(0.0), a.reps):6.2f} us/launch")
    for B in a.B:
        ang = synth.angles_uniform(B, a.L, 3, 1).cuda()
        ln = torch.full((B,), a.L, dtype=torch.int32, device="cuda")
        c = torch.zeros(B, 3 * a.L, 3, device="cuda")
        ws = torch.zeros(_abi.tpl_workspace_bytes(0, B, a.L), dtype=torch.uint8, device="cuda")
        g = torch.randn(B, 3 * a.L, 3, device="cuda")
        ga = torch.zeros(B, a.L, 3, device="cuda")
        f = per_launch_us(lambda: _abi.tpl_backbone_forward(ang, ln, c, ws, torch.cuda.current_stream()), a.reps)
        b = per_launch_us(lambda: _abi.tpl_backbone_backward_from_coords(c, ln, g, ga, ws,
                                                                         torch.cuda.current_stream()), a.reps)

        def step():
            _abi.tpl_backbone_forward(ang, ln, c, ws, torch.cuda.current_stream())
            _abi.tpl_backbone_backward_from_coords(c, ln, g, ga, ws, torch.cuda.current_stream())

        s = per_launch_us(step, a.reps)
        print(f"B={B:4d} L={a.L}: forward {f:6.2f} us  backward {b:6.2f} us  step {s:6.2f} us (L2-warm)")


if __name__ == "__main__":
    main()
