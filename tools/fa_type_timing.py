#!/usr/bin/env python3
"""Full-atom forward/backward per-launch time for a given residue-type mix:
random 20 types vs a single type (GLY: no side chain, TRP: the largest)."""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_1812_01108_b200 as tpl  # noqa: E402
from paper_1812_01108_b200 import _abi  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--B", type=int, default=2048)
    p.add_argument("--L", type=int, default=500)
    a = p.parse_args()
    torch.cuda.set_device(0)
    table = synth.load_residue_table()
    tables = tpl.Tables(table)
    names = [t["name"] for t in table["types"]]
    for mix in ("random", "GLY", "ALA", "TRP"):
        rt = synth.restype_uniform(a.B, a.L, 20, 5) if mix == "random" else \
            torch.full((a.B, a.L), names.index(mix), dtype=torch.uint8)
        ln = torch.full((a.B,), a.L, dtype=torch.int32)
        apc, stride = tables.atoms(rt, ln)
        ang = synth.angles_uniform(a.B, a.L, 8, 6).cuda()
        r, l = rt.cuda(), ln.cuda()
        c = torch.empty(a.B, stride, 3, device="cuda")
        g = torch.randn(a.B, stride, 3, device="cuda")
        ga = torch.empty(a.B, a.L, 8, device="cuda")
        ws = torch.zeros(_abi.tpl_workspace_bytes(1, a.B, a.L), dtype=torch.uint8, device="cuda")
        fwd = lambda: _abi.tpl_fullatom_forward(tables.handle, ang, r, l, c, ws)  # noqa: E731
        bwd = lambda: _abi.tpl_fullatom_backward_from_coords(tables.handle, c, r, l, g, ga, ws)  # noqa: E731
        res = []
        for f in (fwd, bwd):
            for _ in range(3):
                f()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                f()
            e1.record()
            torch.cuda.synchronize()
            res.append(e0.elapsed_time(e1) * 100)
        atoms = int(apc.sum())
        print(f"{mix:7s} B={a.B} L={a.L}: {atoms / (a.B * a.L):5.2f} atoms/res  fwd {res[0]:8.1f} us  bwd {res[1]:8.1f} us")


if __name__ == "__main__":
    main()
