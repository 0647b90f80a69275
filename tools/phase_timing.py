#!/usr/bin/env python3
"""Phase timeline of bb_forward_kernel CTAs (needs the phase-stamp build):

    python -m paper_1812_01108_b200.build --phases
    TPL_LIB=paper_1812_01108_b200/build/libtpl_phases.so python tools/phase_timing.py --B 256 --L 700

Prints, over CTAs, the median / max time (ns, %globaltimer) of each phase
relative to the earliest CTA start.
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

NAMES = ["start", "lengths", "tma issued", "tma landed", "pass1 done", "scan done", "pass2 done", "synced",
         "store issued", "store done"]


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--B", type=int, default=256)
    p.add_argument("--L", type=int, default=700)
    p.add_argument("--bwd", action="store_true", help="the coordinate backward (two tiles per CTA stamped)")
    p.add_argument("--fused", action="store_true", help="fused_lrmsd.cu one-pass kernel: stamps 0..6")
    p.add_argument("--packed", action="store_true", help="packed.cu kernels: stamps 0..7 (start, issued, landed, pass1, scan, pass2, store issued, end)")
    a = p.parse_args()
    torch.cuda.set_device(0)
    L = _abi.lib
    L.tpl_debug_stamps.argtypes = [ctypes.c_void_p, ctypes.c_int]
    ang = synth.angles_uniform(a.B, a.L, 3, 1).cuda()
    ln = torch.full((a.B,), a.L, dtype=torch.int32, device="cuda")
    c = torch.empty(a.B, 3 * a.L, 3, device="cuda")
    ws = torch.zeros(_abi.tpl_workspace_bytes(0, a.B, a.L), dtype=torch.uint8, device="cuda")
    g = torch.randn(a.B, 3 * a.L, 3, device="cuda")
    ga = torch.empty(a.B, a.L, 3, device="cuda")

    tgt = torch.randn(a.B, 3 * a.L, 3, device="cuda") * 20
    st16 = torch.empty(a.B, 16, device="cuda")
    lo = torch.empty(a.B, device="cuda")

    def run():
        if a.fused:
            _abi.tpl_backbone_lrmsd_fused(ang, ln, tgt, None, lo, st16, ga, ws)
        elif a.bwd:
            _abi.tpl_backbone_backward_from_coords(c, ln, g, ga, ws)
        else:
            _abi.tpl_backbone_forward(ang, ln, c, ws)

    _abi.tpl_backbone_forward(ang, ln, c, ws)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    L.tpl_debug_stamps_clear()
    run()
    torch.cuda.synchronize()
    n = min(a.B, 4096)
    buf = (ctypes.c_ulonglong * (n * 16))()
    if a.fused:
        L.tpl_debug_stamps_fused.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.tpl_debug_stamps_fused(buf, n * 16)
        names = ["start", "angles landed", "fwd done", "target landed", "M1 computed", "M1 synced", "M2 computed",
                 "M2 synced", "solve", "bwd pass1+scan", "end"]
        st = np.array(buf, dtype=np.int64).reshape(n, 16)[:, [0, 1, 2, 7, 8, 9, 10, 3, 4, 5, 6]]
        st = st[(st > 0).all(axis=1)]
        rel = st - st[:, 0].min()
        print(f"fused B={a.B} L={a.L}: {len(st)} CTAs, span {rel.max() / 1e3:.2f} us")
        for i, nm in enumerate(names):
            step = (st[:, i] - st[:, i - 1]) if i else rel[:, 0]
            print(f"  {nm:15s} at median {np.median(rel[:, i]) / 1e3:6.2f} us, max {rel[:, i].max() / 1e3:6.2f};"
                  f"  phase median {np.median(step) / 1e3:6.2f} us max {step.max() / 1e3:6.2f}")
        return
    if a.packed:
        L.tpl_debug_stamps_packed(buf, n * 16)
    else:
        L.tpl_debug_stamps(buf, n * 16)
    if a.packed:
        names = ["start", "issued", "landed", "pass1", "scan", "pass2", "store issued", "end"]
        st = np.array(buf, dtype=np.int64).reshape(n, 16)[:, 8:16] if a.bwd else np.array(buf, dtype=np.int64).reshape(n, 16)[:, :8]
        for c in range(1, st.shape[1]):  # a phase without a stamp (e.g. no separate store issue) takes the one before
            st[:, c] = np.where(st[:, c] > 0, st[:, c], st[:, c - 1])
        st = st[(st > 0).all(axis=1)]
        rel = st - st[:, 0].min()
        print(f"{'bwd' if a.bwd else 'fwd'} B={a.B} L={a.L}: {len(st)} CTAs, span {rel.max() / 1e3:.2f} us")
        for i, nm in enumerate(names):
            step = (st[:, i] - st[:, i - 1]) if i else rel[:, 0]
            print(f"  {nm:13s} at median {np.median(rel[:, i]) / 1e3:6.2f} us, max {rel[:, i].max() / 1e3:6.2f};"
                  f"  phase median {np.median(step) / 1e3:6.2f} us max {step.max() / 1e3:6.2f}")
        return
    if a.bwd:
        names = ["start", "tile A landed", "tile A pass1", "tile A scan", "tile A walk", "tile A stored",
                 "tile B landed", "tile B pass1", "tile B scan", "tile B walk", "tile B stored", "end"]
        st = np.array(buf, dtype=np.int64).reshape(n, 16)[:, [0, 2, 3, 4, 11, 5, 6, 7, 8, 12, 9, 10]]
        st = st[(st > 0).all(axis=1)] if ((st > 0).all(axis=1)).any() else st[:, [0, 1, 2, 3, 4, 5, 11]]
        t0 = st[:, 0].min()
        rel = st - t0
        print(f"bwd B={a.B} L={a.L}: CTAs with two tiles {len(st)}; span {rel[:, -1].max() / 1e3:.2f} us")
        for i in range(st.shape[1]):
            step = (st[:, i] - st[:, i - 1]) if i else rel[:, 0]
            print(f"  {names[i] if st.shape[1] == 12 else str(i):15s} at median {np.median(rel[:, i]) / 1e3:6.2f} us"
                  f"  phase median {np.median(step) / 1e3:6.2f} us")
        return
    st = np.array(buf, dtype=np.int64).reshape(n, 16)[:, :10]
    t0 = st[:, 0].min()
    rel = st - t0
    print(f"B={a.B} L={a.L}: kernel span {rel[:, 9].max() / 1e3:.2f} us (first CTA start -> last store done)")
    for i, nm in enumerate(NAMES):
        d = rel[:, i]
        step = (st[:, i] - st[:, i - 1]) if i else rel[:, 0]
        print(f"  {nm:13s} at median {np.median(d) / 1e3:6.2f} us, max {d.max() / 1e3:6.2f} us;"
              f"  phase median {np.median(step) / 1e3:6.2f} us max {step.max() / 1e3:6.2f}")


if __name__ == "__main__":
    main()
