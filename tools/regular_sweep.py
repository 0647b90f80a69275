#!/usr/bin/env python3
"""Forward error of regular chains vs the fp64 oracle over a range of L (which
kernel/shape serves each L is the launcher's choice):  python tools/regular_sweep.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (test infrastructure)
import synth  # noqa: E402
from paper_1812_01108_b200 import _abi  # noqa: E402

oracle.build()
for kind in sys.argv[1:] or ["extended", "helix", "strand"]:
    for L in (256, 512, 600, 700, 768, 769, 800, 900, 1000, 1024):
        ang = synth.regular_angles(2, L, kind)
        ln = torch.full((2,), L, dtype=torch.int32)
        c = torch.empty(2, 3 * L, 3, device="cuda")
        ws = torch.zeros(_abi.tpl_workspace_bytes(0, 2, L), dtype=torch.uint8, device="cuda")
        _abi.tpl_backbone_forward(ang.cuda(), ln.cuda(), c, ws)
        X = oracle.backbone_forward(synth.numpy64(ang), ln.numpy())
        e = np.abs(c.cpu().numpy() - X).max(axis=2)[0]
        i = int(np.argmax(e))
        print(f"{kind:9s} L={L:5d} max err {e.max():.2e} A at atom {i} (|r| {np.linalg.norm(X[0, i]):.0f} A)")
