#!/usr/bin/env python3
"""Kernel boundaries inside the bench's step graph (needs the phase-stamp build):

    python -m paper_1812_01108_b200.build --phases
    TPL_LIB=paper_1812_01108_b200/build/libtpl_phases.so python tools/step_gaps.py [--B 256 --L 700]

Captures K (forward, coordinate backward) steps of the packed kernels in one CUDA
graph over rotating buffer sets (as bench.py), replays it, and reads the last
step's %globaltimer stamps: forward CTAs write slots 0-7, backward CTAs 8-15.
Prints the first CTA start / last CTA end of both kernels and the gaps, beside
the CUDA-event time per step.
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1812_01108_b200 import _abi  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--B", type=int, default=256)
    p.add_argument("--L", type=int, default=700)
    p.add_argument("--K", type=int, default=20)
    p.add_argument("--sets", type=int, default=20)
    a = p.parse_args()
    torch.cuda.set_device(0)
    lib = _abi.lib
    lib.tpl_debug_stamps_packed.argtypes = [ctypes.c_void_p, ctypes.c_int]
    sets = []
    for i in range(a.sets):
        sets.append(dict(ang=synth.angles_uniform(a.B, a.L, 3, 1 + i).cuda(),
                         ln=torch.full((a.B,), a.L, dtype=torch.int32, device="cuda"),
                         c=torch.empty(a.B, 3 * a.L, 3, device="cuda"),
                         g=torch.randn(a.B, 3 * a.L, 3, device="cuda"),
                         ga=torch.empty(a.B, a.L, 3, device="cuda"),
                         ws=torch.zeros(_abi.tpl_workspace_bytes(0, a.B, a.L), dtype=torch.uint8, device="cuda")))

    def step(s):
        _abi.tpl_backbone_forward(s["ang"], s["ln"], s["c"], s["ws"])
        _abi.tpl_backbone_backward_from_coords(s["c"], s["ln"], s["g"], s["ga"], s["ws"])

    for s in sets[:3]:
        step(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            for k in range(a.K):
                step(sets[k % len(sets)])
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    n = min(a.B, 4096)
    buf = (ctypes.c_ulonglong * (n * 16))()
    lib.tpl_debug_stamps_packed(buf, n * 16)
    st_ = np.array(buf, dtype=np.int64).reshape(n, 16)
    f, b = st_[:, :8], st_[:, 8:]
    t0 = f[:, 0].min()
    print(f"B={a.B} L={a.L}: CUDA-event {e0.elapsed_time(e1) * 1e3 / a.K:.2f} us/step (graph of {a.K})")
    print(f"  fwd CTA start first {0:.2f} last {(f[:, 0].max() - t0) / 1e3:.2f}; end first {(f[:, 7].min() - t0) / 1e3:.2f} last {(f[:, 7].max() - t0) / 1e3:.2f} us")
    print(f"  bwd CTA start first {(b[:, 0].min() - t0) / 1e3:.2f} last {(b[:, 0].max() - t0) / 1e3:.2f}; end first {(b[:, 7].min() - t0) / 1e3:.2f} last {(b[:, 7].max() - t0) / 1e3:.2f} us")
    print(f"  gap fwd last end -> bwd first start {(b[:, 0].min() - f[:, 7].max()) / 1e3:.2f} us")


if __name__ == "__main__":
    main()
