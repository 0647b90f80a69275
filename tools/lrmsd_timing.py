#!/usr/bin/env python3
"""Per-launch times of the LRMSD forward / backward kernels (CUDA graph, rotating sets)."""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1812_01108_b200 import _abi  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--B", type=int, default=256)
    p.add_argument("--N", type=int, default=2100)
    p.add_argument("--K", type=int, default=100)
    a = p.parse_args()
    torch.cuda.set_device(0)
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    n = min(64, max(2, math.ceil(4 * l2 / (a.B * a.N * 36))))
    sets = [dict(x=synth.grad_normal((a.B, a.N, 3), 1 + i).cuda(), y=synth.grad_normal((a.B, a.N, 3), 100 + i).cuda(),
                 na=torch.full((a.B,), a.N, dtype=torch.int32, device="cuda"), out=torch.empty(a.B, device="cuda"),
                 st=torch.empty(a.B, 16, device="cuda"), gl=torch.ones(a.B, device="cuda"),
                 gx=torch.empty(a.B, a.N, 3, device="cuda"),
                 ws=torch.zeros(_abi.tpl_workspace_bytes(0, a.B, 16), dtype=torch.uint8, device="cuda"))
            for i in range(n)]
    fwd = lambda s: _abi.tpl_lrmsd_forward(s["x"], s["y"], s["na"], s["out"], s["st"], s["ws"])  # noqa: E731
    bwd = lambda s: _abi.tpl_lrmsd_backward(s["x"], s["y"], s["na"], s["st"], s["gl"], s["gx"], s["ws"])  # noqa: E731

    def timeit(f):
        for i in range(3):
            f(sets[i % n])
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        with torch.cuda.stream(st), torch.cuda.graph(g, stream=st):
            for i in range(a.K):
                f(sets[i % n])
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(5):
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / a.K)
        return best

    for s in sets[:3]:
        fwd(s)
    print(f"lrmsd B={a.B} N={a.N}: fwd {timeit(fwd):.2f} us, bwd {timeit(bwd):.2f} us")


if __name__ == "__main__":
    main()
