#!/usr/bin/env python3
"""Per-launch time of the backbone kernels over a (B, L) grid, in CUDA graphs,
hot (one buffer set) and cold (rotating sets > 4x L2).  Separates the fixed
per-launch latency from the per-residue cost.

    python tools/latency_sweep.py
"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1812_01108_b200 import _abi  # noqa: E402


def sets_for(B, L, n):
    out = []
    ang = synth.angles_uniform(B, L, 3, 1).cuda()
    grad = synth.grad_normal((B, 3 * L, 3), 2).cuda()
    for _ in range(n):
        out.append(dict(a=ang.clone(), l=torch.full((B,), L, dtype=torch.int32, device="cuda"), g=grad.clone(),
                        c=torch.empty(B, 3 * L, 3, device="cuda"), ga=torch.empty(B, L, 3, device="cuda"),
                        ws=torch.zeros(_abi.tpl_workspace_bytes(0, B, L), dtype=torch.uint8, device="cuda")))
    return out


def time_graph(fn, sets, reps=50):
    for s in sets[:2]:
        fn(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st), torch.cuda.graph(g, stream=st):
        for i in range(reps):
            fn(sets[i % len(sets)])
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
    return best


def main():
    torch.cuda.set_device(0)
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    fwd = lambda s: _abi.tpl_backbone_forward(s["a"], s["l"], s["c"], s["ws"])  # noqa: E731
    bwd = lambda s: _abi.tpl_backbone_backward(s["a"], s["l"], s["g"], s["ga"], s["ws"])  # noqa: E731
    print(f"{'B':>6} {'L':>5} {'fwd hot':>8} {'fwd cold':>8} {'bwd hot':>8} {'bwd cold':>8}  (us per launch)")
    for B, L in [(1, 16), (1, 700), (16, 700), (64, 700), (148, 700), (256, 700), (512, 700), (1024, 700),
                 (256, 128), (256, 256), (2048, 700), (4096, 700)]:
        foot = B * L * 96
        n = max(2, math.ceil(4 * l2 / foot))
        n = min(n, 64)
        hot = sets_for(B, L, 1)
        cold = sets_for(B, L, n) if n > 1 else hot
        r = [time_graph(fwd, hot), time_graph(fwd, cold), time_graph(bwd, hot), time_graph(bwd, cold)]
        print(f"{B:>6} {L:>5} " + " ".join(f"{x:8.2f}" for x in r))
        del hot, cold
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
