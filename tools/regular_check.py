#!/usr/bin/env python3
"""Backbone forward error on regular structures (helix / strand / extended) at
L = 700 and 1000 against the fp64 oracle: the worst case for fp32 drift, since
every residue repeats the same rounding (DESIGN reading Q21).

    TPL_ORTHO=2 python tools/regular_check.py [--precise] [--json out.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (test infrastructure)
import synth  # noqa: E402
from paper_1812_01108_b200 import _abi  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--precise", action="store_true", help="tpl_backbone_forward_precise (f2) instead")
    p.add_argument("--json", default=None)
    args = p.parse_args()
    fwd = _abi.tpl_backbone_forward_precise if args.precise else _abi.tpl_backbone_forward
    mode = "precise" if args.precise else f"fp32 TPL_ORTHO={os.environ.get('TPL_ORTHO', '1')}"
    torch.cuda.set_device(0)
    oracle.build()
    rows = []
    for L in (700, 1000):
        for kind in ("helix", "strand", "extended"):
            ang = synth.regular_angles(2, L, kind)
            ln = torch.full((2,), L, dtype=torch.int32)
            c = torch.empty(2, 3 * L, 3, device="cuda")
            ws = torch.zeros(_abi.tpl_workspace_bytes(0, 2, L), dtype=torch.uint8, device="cuda")
            fwd(ang.cuda(), ln.cuda(), c, ws)
            _abi.tpl_sync_status(ws)
            X = oracle.backbone_forward(synth.numpy64(ang), ln.numpy())
            err = float(np.abs(c.cpu().numpy() - X).max())
            ext = float(np.linalg.norm(X, axis=2).max())
            print(f"{mode} L={L} {kind:9s} max err {err:.3e} A  extent {ext:.0f} A")
            rows.append({"mode": mode, "L": L, "kind": kind, "max_err_A": err, "extent_A": ext})
    if args.json:
        with open(args.json, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
