#!/usr/bin/env python3
"""Run backbone fwd+bwd on a uniform B x L batch (no graphs) for ncu captures."""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import synth  # noqa: E402
from paper_1812_01108_b200 import _abi  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--B", type=int, default=4096)
p.add_argument("--L", type=int, default=700)
p.add_argument("--iters", type=int, default=3)
a = p.parse_args()
torch.cuda.set_device(0)
ang = synth.angles_uniform(a.B, a.L, 3, 1).cuda()
ln = torch.full((a.B,), a.L, dtype=torch.int32, device="cuda")
g = synth.grad_normal((a.B, 3 * a.L, 3), 2).cuda()
c = torch.empty(a.B, 3 * a.L, 3, device="cuda")
ga = torch.empty(a.B, a.L, 3, device="cuda")
ws = torch.zeros(_abi.tpl_workspace_bytes(0, a.B, a.L), dtype=torch.uint8, device="cuda")
for _ in range(a.iters):
    _abi.tpl_backbone_forward(ang, ln, c, ws)
    _abi.tpl_backbone_backward(ang, ln, g, ga, ws)
torch.cuda.synchronize()
print("ok")
