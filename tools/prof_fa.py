#!/usr/bin/env python3
"""Run full-atom fwd+bwd on a B x L batch of random types (no graphs) for ncu captures."""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import synth  # noqa: E402
import paper_1812_01108_b200 as tpl  # noqa: E402
from paper_1812_01108_b200 import _abi  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--B", type=int, default=1024)
p.add_argument("--L", type=int, default=500)
p.add_argument("--iters", type=int, default=3)
p.add_argument("--angles-bwd", action="store_true", help="backward from the angles (default: from coords)")
a = p.parse_args()
torch.cuda.set_device(0)
tables = tpl.Tables(synth.load_residue_table())
ang = synth.angles_uniform(a.B, a.L, 8, 1)
rt = synth.restype_uniform(a.B, a.L, 20, 2)
ln = torch.full((a.B,), a.L, dtype=torch.int32)
apc, stride = tables.atoms(rt, ln)
g = synth.grad_normal((a.B, stride, 3), 3).cuda()
ang, rt, ln = ang.cuda(), rt.cuda(), ln.cuda()
c = torch.empty(a.B, stride, 3, device="cuda")
ga = torch.empty(a.B, a.L, 8, device="cuda")
ws = torch.zeros(_abi.tpl_workspace_bytes(1, a.B, a.L), dtype=torch.uint8, device="cuda")
for _ in range(a.iters):
    _abi.tpl_fullatom_forward(tables.handle, ang, rt, ln, c, ws)
    if a.angles_bwd:
        _abi.tpl_fullatom_backward(tables.handle, ang, rt, ln, g, ga, ws)
    else:
        _abi.tpl_fullatom_backward_from_coords(tables.handle, c, rt, ln, g, ga, ws)
torch.cuda.synchronize()
print("ok")
