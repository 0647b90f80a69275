#!/usr/bin/env python3
"""One small invocation of every kernel family, for compute-sanitizer (tools/sanitize.sh):

    python tools/sanitize_cases.py CASE     CASE in: bb1 ragged packed lrmsd fa3 long dl cluster segment paper precise

Each case runs the C-ABI calls once (forward and both backward entry points where
they exist) and synchronises; results are not checked here (the parity suite does
that) -- the point is the sanitizer's view of the memory accesses, shared-memory
races, barrier use and uninitialised reads of the same launches.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1812_01108_b200 import _abi  # noqa: E402


def bb(B, Lmax, lengths=None, seed=1):
    ang = synth.angles_uniform(B, Lmax, 3, seed).cuda()
    ln = (torch.full((B,), Lmax, dtype=torch.int32) if lengths is None else lengths).cuda()
    g = synth.grad_normal((B, 3 * Lmax, 3), seed + 1).cuda()
    c = torch.zeros(B, 3 * Lmax, 3, device="cuda")
    ga = torch.zeros(B, Lmax, 3, device="cuda")
    gx = torch.zeros(B, Lmax, 3, device="cuda")
    ws = torch.zeros(_abi.tpl_workspace_bytes(0, B, Lmax), dtype=torch.uint8, device="cuda")
    _abi.tpl_backbone_forward(ang, ln, c, ws)
    _abi.tpl_backbone_backward_from_coords(c, ln, g, gx, ws)
    _abi.tpl_backbone_backward(ang, ln, g, ga, ws)
    _abi.tpl_sync_status(ws)
    return ang, ln, c, ws


def lrmsd(B, Lmax, lengths=None):
    ang, ln, c, ws = bb(B, Lmax, lengths)
    tgt = synth.grad_normal((B, 3 * Lmax, 3), 9).cuda() * 20
    out, st = torch.zeros(B, device="cuda"), torch.zeros(B, 16, device="cuda")
    g = torch.zeros(B, Lmax, 3, device="cuda")
    _abi.tpl_backbone_lrmsd_fused(ang, ln, tgt, c, out, st, g, ws)
    _abi.tpl_chain_scale(g, out, g)
    # the two-call fused pair and the stand-alone loss
    _abi.tpl_backbone_lrmsd_forward(ang, ln, tgt, c, out, st, ws)
    _abi.tpl_backbone_lrmsd_backward(c, ln, tgt, st, torch.ones(B, device="cuda"), g, ws)
    na = (3 * ln).to(torch.int32)
    _abi.tpl_lrmsd_forward(c, tgt, na, out, st, ws)
    gx = torch.zeros_like(c)
    _abi.tpl_lrmsd_backward(c, tgt, na, st, torch.ones(B, device="cuda"), gx, ws)
    _abi.tpl_sync_status(ws)


def fa(B, L):
    import paper_1812_01108_b200 as tpl

    table = synth.load_residue_table()
    tables = tpl.Tables(table)
    ang, rt, ln = synth.fullatom_inputs(3, B=B, L=L)
    apc, stride = tables.atoms(rt, ln)
    a, r, l = ang.cuda(), rt.cuda(), ln.cuda()
    c = torch.zeros(B, stride, 3, device="cuda")
    g = synth.grad_normal((B, stride, 3), 3).cuda()
    ga = torch.zeros(B, L, 8, device="cuda")
    ws = torch.zeros(_abi.tpl_workspace_bytes(1, B, L), dtype=torch.uint8, device="cuda")
    _abi.tpl_fullatom_forward(tables.handle, a, r, l, c, ws)
    _abi.tpl_fullatom_backward_from_coords(tables.handle, c, r, l, g, ga, ws)
    _abi.tpl_fullatom_backward(tables.handle, a, r, l, g, ga, ws)
    _abi.tpl_sync_status(ws)


def main(case):
    torch.cuda.set_device(0)
    if case == "bb1":
        bb(1, 16)
    elif case == "ragged":
        bb(40, 700, synth.lengths_uniform(40, 1, 700, 5))
        bb(9, 701, synth.lengths_uniform(9, 1, 701, 6))  # chain bases not 16-byte aligned
    elif case == "packed":
        bb(256, 700)
        bb(300, 1000)
    elif case == "lrmsd":
        lrmsd(12, 700, synth.lengths_uniform(12, 1, 700, 7))
        lrmsd(3, 1100)
    elif case == "fa3":
        fa(64, 300)
    elif case == "long":
        bb(1, 20000)  # decoupled tiles over CTAs (epoch flags)
    elif case == "dl":
        bb(64, 3000, synth.lengths_uniform(64, 1025, 3000, 8))
    elif case == "cluster":
        bb(128, 1400)  # 2-CTA cluster backward (1153-1536 residues, <= SMs chains)
    elif case == "serial":  # the chain-serial / cluster-split kernels the packed ones replaced (TPL_PACKED=0)
        bb(64, 700)
        bb(256, 700)
        bb(300, 2000, synth.lengths_uniform(300, 50, 2000, 14))
    elif case == "segment":  # f4 segment kernels, the exchange stacked in-process (2 segments)
        B, L, bounds = 3, 1500, [(0, 750), (750, 1500)]
        ang = synth.angles_uniform(B, L, 3, 11)
        grad = synth.grad_normal((B, 3 * L, 3), 12)
        parts = []
        for (j0, j1) in bounds:
            n = j1 - j0
            a = ang[:, j0:j1].contiguous().cuda()
            ln = torch.full((B,), n, dtype=torch.int32, device="cuda")
            om = ang[:, j0 - 1, 2].contiguous().cuda() if j0 > 0 else None
            ws = torch.zeros(_abi.tpl_workspace_bytes(0, B, n), dtype=torch.uint8, device="cuda")
            c = torch.zeros(B, 3 * n, 3, device="cuda")
            agg = torch.zeros(B, 12, device="cuda")
            _abi.tpl_backbone_segment_forward(a, ln, om, c, agg, ws)
            parts.append(dict(ln=ln, ws=ws, c=c, agg=agg, g=grad[:, 3 * j0:3 * j1].contiguous().cuda()))
        aggs = torch.stack([p["agg"] for p in parts])
        for s_, p in enumerate(parts):
            _abi.tpl_backbone_segment_place(p["c"], p["ln"], aggs, s_, p["ws"])
            p["tot"] = torch.zeros(B, 12, device="cuda")
            _abi.tpl_backbone_segment_totals(p["c"], p["ln"], p["g"], p["tot"], p["ws"])
        tots = torch.stack([p["tot"] for p in parts])
        for s_, p in enumerate(parts):
            ga = torch.zeros(B, p["c"].shape[1] // 3, 3, device="cuda")
            _abi.tpl_backbone_segment_backward(p["c"], p["ln"], p["g"], tots, s_, ga, p["ws"])
            _abi.tpl_sync_status(p["ws"])
    elif case == "paper":
        B, L = 8, 300
        ang = synth.angles_uniform(B, L, 3, 12).cuda()
        ln = torch.full((B,), L, dtype=torch.int32, device="cuda")
        c = torch.zeros(B, 3 * L, 3, device="cuda")
        M = torch.zeros(_abi.tpl_paper_backbone_saved_floats(B, L), device="cuda")
        g = torch.randn(B, 3 * L, 3, device="cuda")
        ga = torch.zeros(B, L, 3, device="cuda")
        ws = torch.zeros(_abi.tpl_workspace_bytes(0, B, L), dtype=torch.uint8, device="cuda")
        _abi.tpl_paper_backbone_forward(ang, ln, c, M, ws)
        _abi.tpl_paper_backbone_backward(ang, ln, M, g, ga, ws)
        _abi.tpl_sync_status(ws)
    elif case == "precise":
        B, L = 8, 500
        ang = synth.angles_uniform(B, L, 3, 13).cuda()
        ln = torch.full((B,), L, dtype=torch.int32, device="cuda")
        c = torch.zeros(B, 3 * L, 3, device="cuda")
        ws = torch.zeros(_abi.tpl_workspace_bytes(0, B, L), dtype=torch.uint8, device="cuda")
        _abi.tpl_backbone_forward_precise(ang, ln, c, ws)
        _abi.tpl_sync_status(ws)
    else:
        raise SystemExit(f"unknown case {case}")
    torch.cuda.synchronize()
    print(f"case {case} ok")


if __name__ == "__main__":
    main(sys.argv[1])
