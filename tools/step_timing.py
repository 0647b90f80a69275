#!/usr/bin/env python3
"""Per-launch times (CUDA graphs, rotating cold buffer sets) of fwd-only,
bwd-only and alternating fwd/bwd sequences for a backbone B x L batch.

    python tools/step_timing.py --B 256 --L 700
"""
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
    p.add_argument("--L", type=int, default=700)
    p.add_argument("--K", type=int, default=120)
    p.add_argument("--xyz", action="store_true", help="backward from the forward's coordinates")
    p.add_argument("--precise", action="store_true", help="the fp64-internal forward (f2)")
    a = p.parse_args()
    torch.cuda.set_device(0)
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    n = min(64, max(2, math.ceil(4 * l2 / (a.B * a.L * 96))))
    ang = synth.angles_uniform(a.B, a.L, 3, 1).cuda()
    g = synth.grad_normal((a.B, 3 * a.L, 3), 2).cuda()
    sets = [dict(a=ang.clone(), l=torch.full((a.B,), a.L, dtype=torch.int32, device="cuda"), g=g.clone(),
                 c=torch.empty(a.B, 3 * a.L, 3, device="cuda"), ga=torch.empty(a.B, a.L, 3, device="cuda"),
                 ws=torch.zeros(_abi.tpl_workspace_bytes(0, a.B, a.L), dtype=torch.uint8, device="cuda"))
            for _ in range(n)]
    if a.precise:
        fwd = lambda s: _abi.tpl_backbone_forward_precise(s["a"], s["l"], s["c"], s["ws"])  # noqa: E731
        bwd = lambda s: _abi.tpl_backbone_backward_from_coords(s["c"], s["l"], s["g"], s["ga"], s["ws"])  # noqa: E731
    elif a.xyz:
        fwd = lambda s: _abi.tpl_backbone_forward(s["a"], s["l"], s["c"], s["ws"])  # noqa: E731
        bwd = lambda s: _abi.tpl_backbone_backward_from_coords(s["c"], s["l"], s["g"], s["ga"], s["ws"])  # noqa: E731
    else:
        fwd = lambda s: _abi.tpl_backbone_forward(s["a"], s["l"], s["c"], s["ws"])  # noqa: E731
        bwd = lambda s: _abi.tpl_backbone_backward(s["a"], s["l"], s["g"], s["ga"], s["ws"])  # noqa: E731

    def timeit(seq):
        for i in range(3):
            for f in seq:
                f(sets[i % n])
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        with torch.cuda.stream(st), torch.cuda.graph(gr, stream=st):
            for i in range(a.K):
                for f in seq:
                    f(sets[i % n])
        gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(7):
            e0.record()
            gr.replay()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / a.K)
        return best

    f, b, fb = timeit([fwd]), timeit([bwd]), timeit([fwd, bwd])
    print(f"{'precise ' if a.precise else 'xyz ' if a.xyz else ''}{os.environ.get('TPL_BBX', '')} B={a.B} L={a.L} sets={n}: fwd {f:.2f} us, bwd {b:.2f} us, fwd+bwd step {fb:.2f} us "
          f"(sum {f + b:.2f}, step overhead {fb - f - b:+.2f})")


if __name__ == "__main__":
    main()
