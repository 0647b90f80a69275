#!/usr/bin/env python3
"""precision profile of the fp32 GPU path against the fp64 oracle.

Reproduces the methodology of Fig:ErrorEstimate: the error of each
atom's position as a function of its index along the chain, mean and 95% CI
over 10 random chains of L = 700 (random angles), for the product
forward (backbone kernel and the full-atom kernel's backbone atoms), and
extends it to regular structures (alpha helix, beta strand, fully extended),
where fp32 error grows fastest.  Also reports the gradient error of both
backward entry points.

    python tools/precision_profile.py            # writes profiles/r01_precision_profile.{md,json}
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: the fp64 reference)
import synth  # noqa: E402
import paper_1812_01108_b200 as tpl  # noqa: E402
from paper_1812_01108_b200 import _abi  # noqa: E402

L = 700
N_CHAINS = 10
CHECKPOINTS = [0, 99, 299, 599, 999, 1499, 2099]  # atom indices reported in the table


def run_backbone(ang, lengths, grad):
    B, Lmax, _ = ang.shape
    a, ln, g = ang.cuda(), lengths.cuda(), grad.cuda()
    coords = torch.empty(B, 3 * Lmax, 3, device="cuda")
    ga = torch.zeros(B, Lmax, 3, device="cuda")
    gx = torch.zeros(B, Lmax, 3, device="cuda")
    ws = torch.zeros(_abi.tpl_workspace_bytes(0, B, Lmax), dtype=torch.uint8, device="cuda")
    _abi.tpl_backbone_forward(a, ln, coords, ws)
    _abi.tpl_backbone_backward(a, ln, g, ga, ws)
    _abi.tpl_backbone_backward_from_coords(coords, ln, g, gx, ws)
    _abi.tpl_sync_status(ws)
    return coords.cpu().numpy(), ga.cpu().numpy(), gx.cpu().numpy()


def per_atom_stats(err):
    """err [chains, atoms] -> mean, 95% CI half-width (t-distribution, n-1 dof ~ 2.262 for n=10)."""
    n = err.shape[0]
    mean = err.mean(axis=0)
    sd = err.std(axis=0, ddof=1) if n > 1 else np.zeros_like(mean)
    t = {10: 2.262, 2: 12.706}.get(n, 1.96)
    return mean, t * sd / math.sqrt(n)


def grad_err(g, G):
    return float(max(np.abs(g[b] - G[b]).max() / max(np.abs(G[b]).max(), 1e-30) for b in range(g.shape[0])))


def main():
    torch.cuda.set_device(0)
    oracle.build()
    out = {"L": L, "chains": N_CHAINS, "cases": {}}
    # random chains (the paper's figure)
    ang = synth.angles_uniform(N_CHAINS, L, 3, 7001)
    ln = torch.full((N_CHAINS,), L, dtype=torch.int32)
    grad = synth.grad_normal((N_CHAINS, 3 * L, 3), 7002)
    cases = [("random", ang, grad)]
    for kind in ("helix", "strand", "extended"):
        cases.append((kind, synth.regular_angles(2, L, kind), synth.grad_normal((2, 3 * L, 3), 7003)))
    for name, a, g in cases:
        B = a.shape[0]
        lens = torch.full((B,), L, dtype=torch.int32)
        X = oracle.backbone_forward(synth.numpy64(a), lens.numpy())
        G = oracle.backbone_backward(synth.numpy64(a), lens.numpy(), synth.numpy64(g))
        c, ga, gx = run_backbone(a, lens, g)
        err = np.linalg.norm(c - X, axis=2)  # [B, 3L] Angstrom
        mean, ci = per_atom_stats(err)
        extent = float(np.linalg.norm(X, axis=2).max())
        out["cases"][name] = {
            "chains": B, "max_err_A": float(err.max()), "max_extent_A": extent,
            "mean_at": {str(i): float(mean[i]) for i in CHECKPOINTS},
            "ci95_at": {str(i): float(ci[i]) for i in CHECKPOINTS},
            "grad_rel_err_from_angles": grad_err(ga, G), "grad_rel_err_from_coords": grad_err(gx, G),
            "first_atom_over_1e-3": int(np.argmax(err.max(axis=0) > 1e-3)) if (err > 1e-3).any() else None,
        }
    # full-atom model: its N, CA, C against the backbone oracle (P:276 compares the two models)
    table = synth.load_residue_table()
    tables = tpl.Tables(table)
    rt = synth.restype_uniform(N_CHAINS, L, 20, 7004)
    fa_ang = synth.angles_uniform(N_CHAINS, L, 8, 7005)
    fa = tpl.fullatom(fa_ang.cuda(), rt.cuda(), ln.cuda(), tables).cpu().numpy()
    Xbb = oracle.backbone_forward(synth.numpy64(fa_ang[..., :3].contiguous()), ln.numpy())
    n_at = np.array([len(t["atoms"]) for t in table["types"]])
    errs = np.zeros((N_CHAINS, 3 * L))
    for b in range(N_CHAINS):
        off = 0
        for j in range(L):
            t = int(rt[b, j])
            for k, slot in ((0, 0), (1, 1), (int(n_at[t]) - 2, 2)):  # N, CA, C (C, O are the last two)
                errs[b, 3 * j + slot] = np.linalg.norm(fa[b, off + k] - Xbb[b, 3 * j + slot])
            off += int(n_at[t])
    mean, ci = per_atom_stats(errs)
    out["cases"]["fullatom_backbone_atoms"] = {
        "chains": N_CHAINS, "max_err_A": float(errs.max()),
        "mean_at": {str(i): float(mean[i]) for i in CHECKPOINTS}, "ci95_at": {str(i): float(ci[i]) for i in CHECKPOINTS}}

    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "r01_precision_profile.json"), "w") as f:
        json.dump(out, f, indent=1)
    lines = ["# Precision profile (SURVEY f2; Fig:ErrorEstimate methodology, P:276-283)", "",
             f"fp32 GPU forward vs the fp64 oracle on identical fp32 inputs, L = {L}; |Δr| in Å per atom index "
             "(mean ± 95% CI over the chains of each case). Gradient: per-chain max|Δg| / max|g_ref| (Q18).", "",
             "| case | chains | " + " | ".join(f"atom {i}" for i in CHECKPOINTS) + " | max | grad (angles) | grad (coords) |",
             "|---|---|" + "---|" * len(CHECKPOINTS) + "---|---|---|"]
    for name, d in out["cases"].items():
        cells = " | ".join(f"{d['mean_at'][str(i)]:.1e} ± {d['ci95_at'][str(i)]:.0e}" for i in CHECKPOINTS)
        ga = f"{d['grad_rel_err_from_angles']:.1e}" if "grad_rel_err_from_angles" in d else "—"
        gx = f"{d['grad_rel_err_from_coords']:.1e}" if "grad_rel_err_from_coords" in d else "—"
        lines.append(f"| {name} | {d['chains']} | {cells} | {d['max_err_A']:.1e} | {ga} | {gx} |")
    with open(os.path.join(ROOT, "profiles", "r01_precision_profile.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
