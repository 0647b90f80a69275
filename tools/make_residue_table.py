#!/usr/bin/env python3
"""Build-time generator of the default per-residue-type rigid-group table.

DATA, not method.  The paper gives the full-atom *model* (§2, P:19-59:
rigid groups with standard coordinates r°, per-node fixed (θ_i, d_i), the
out-of-plane R′ at the CB branch) but prints no side-chain geometry (only the
threonine topology).  This script converts the ideal rigid-group
geometry shipped in the image (OpenFold/AlphaFold ``residue_constants``,
Apache-2.0, (c) DeepMind / AlQuraishi Lab) into that model and writes
``synth/residue_table.json``.  Both the oracle and the CUDA path consume the
JSON as an *input*, exactly like the angles.

Model conventions (readings Q5, Q8-Q11):
  * per residue the atom order is  N, CA, side chain (group by group, DFS), C, O;
  * side-chain group k (k = 1..n) has its origin at the χ_k axis-end atom X_k
    (CB for k = 1) and its frame's xz-plane (z < 0) contains the χ_k-defining
    atom D_k, so that the measured dihedral of chi_angles_atoms[k-1] equals the
    input χ_k;
  * group 1 hangs off the CA frame through R′ = R_x(pre_rx) then
    R(χ1, θ_CB, d_CB); group k > 1 hangs off group k-1 through R(χ_k, θ_k, d_k);
  * θ = π - (bond angle at the parent origin), d = bond length;
  * O lives in the C frame at τ = π (dihedral N-CA-C-O = ψ + π);
  * PRO χ1/χ2, ALA's CB group and ARG χ5 are fixed (slot -1) at the ideal
    geometry's torsion (Q11; Q10: χ5 exists as a slot, a test table frees it).

Run:  python tools/make_residue_table.py   (needs transformers importable)
"""
import json
import math
import os
import sys

import numpy as np

from transformers.models.esm.openfold_utils import residue_constants as rc

# "R' corresponds to a counterclockwise rotation of 122.686°
# about the x axis".  Reading Q5: with right-handed R_x the +sign
# produces D-chirality in this frame convention, so the table stores -122.686°.
# tests/test_oracle_fullatom.py::test_chirality_matches_alphafold pins the sign
# against the ideal L-residue geometry of residue_constants.
R_PRIME_DEG = -122.686

SLOT_CHI1 = 3
OWNER = {"N": -3, "CA": -2, "C": -1}


def _frame(ex, ey, t):
    m = rc._make_rigid_transformation_4x4(np.asarray(ex, float), np.asarray(ey, float), np.asarray(t, float))
    return np.asarray(m, dtype=np.float64)


def ideal_residue(resname):
    """Global coordinates (AlphaFold backbone frame) of the ideal residue with
    all AlphaFold torsion rotations at zero."""
    pos = {n: np.array(p, dtype=np.float64) for n, _, p in rc.rigid_group_atom_positions[resname]}
    grp = {n: g for n, g, _ in rc.rigid_group_atom_positions[resname]}
    frames = {0: np.eye(4)}
    frames[3] = _frame(pos["C"] - pos["CA"], pos["CA"] - pos["N"], pos["C"])
    chis = rc.chi_angles_atoms[resname]
    if chis:
        a = [pos[n] for n in chis[0][:3]]
        frames[4] = _frame(a[2] - a[1], a[0] - a[1], a[2])
    for k in range(1, len(chis)):
        p = pos[chis[k][2]]
        frames[4 + k] = frames[3 + k] @ _frame(p, np.array([-1.0, 0.0, 0.0]), p)
    out = {}
    for n, p in pos.items():
        out[n] = (frames[grp[n]] @ np.append(p, 1.0))[:3]
    return out


def _angle(a, b, c):
    u, v = a - b, c - b
    return math.acos(float(np.dot(u, v) / (np.linalg.norm(u) * np.linalg.norm(v))))


def _dihedral(p0, p1, p2, p3):
    b0, b1, b2 = p0 - p1, p2 - p1, p3 - p2
    b1n = b1 / np.linalg.norm(b1)
    v = b0 - np.dot(b0, b1n) * b1n
    w = b2 - np.dot(b2, b1n) * b1n
    return math.atan2(float(np.dot(np.cross(b1n, v), w)), float(np.dot(v, w)))


def _model_frame(origin, prev, defining):
    """Frame with origin X_k, x along prev->X_k, defining atom in xz-plane, z<0."""
    ex = origin - prev
    ex /= np.linalg.norm(ex)
    v = defining - origin
    zp = v - np.dot(v, ex) * ex
    zp /= np.linalg.norm(zp)
    ez = -zp
    ey = np.cross(ez, ex)
    return np.stack([ex, ey, ez], axis=1)  # columns


def residue_entry(resname, chi5=True):
    xyz = ideal_residue(resname)
    chis = [list(c) for c in rc.chi_angles_atoms[resname]]
    if resname == "ARG" and chi5:
        chis.append(["CD", "NE", "CZ", "NH1"])  # χ5 (fixed in the default table)
    af_group = {n: g for n, g, _ in rc.rigid_group_atom_positions[resname]}
    side = [n for n, _, _ in rc.rigid_group_atom_positions[resname] if n not in ("N", "CA", "C", "O")]

    groups, atoms = [], []
    atoms.append({"name": "N", "owner": OWNER["N"], "r": [0.0, 0.0, 0.0]})
    atoms.append({"name": "CA", "owner": OWNER["CA"], "r": [0.0, 0.0, 0.0]})

    if side:
        n_groups = max(1, len(chis))
        origins = ["CB"] + [c[2] for c in chis[1:]]
        chain = ["N", "CA"] + origins  # X_{-1}=N, X_0=CA, X_1=CB, ...
        # assign side-chain atoms to groups
        member = {g: [] for g in range(n_groups)}
        for n in side:
            if n in origins:
                member[origins.index(n)].append(n)
                continue
            g = af_group[n] - 4  # AlphaFold chi-group index (0-based)
            if resname == "ARG" and chi5 and n in ("NH1", "NH2"):
                g = 4
            member[g].append(n)
        for g in range(n_groups):
            X = xyz[origins[g]]
            Xp = xyz[chain[g + 1]]
            Xpp = xyz[chain[g]]
            theta = math.pi - _angle(Xpp, Xp, X)
            d = float(np.linalg.norm(X - Xp))
            if g < len(chis):
                alpha = _dihedral(*[xyz[n] for n in chis[g]])
            else:  # ALA: no χ, CB group only; its orientation about CA-CB is irrelevant
                alpha = 0.0
            if resname == "PRO" or resname == "ALA" or (resname == "ARG" and chi5 and g == 4):
                slot = -1
            else:
                slot = SLOT_CHI1 + g
            Rk = _model_frame(X, Xp, xyz[chis[g][3]]) if g < len(chis) else np.eye(3)
            groups.append({
                "parent": -1 if g == 0 else g - 1,
                "slot": slot,
                "alpha": alpha if slot == -1 else 0.0,
                "theta": theta,
                "d": d,
                "pre_rx": math.radians(R_PRIME_DEG) if g == 0 else 0.0,
                "chi_atoms": chis[g] if g < len(chis) else [],
            })
            ordered = [origins[g]] + [n for n in member[g] if n != origins[g]]
            for n in ordered:
                r = Rk.T @ (xyz[n] - X)
                if n == origins[g]:
                    r = np.zeros(3)
                if g < len(chis) and n == chis[g][3]:
                    r[1] = 0.0  # exactly in the xz-plane by construction
                atoms.append({"name": n, "owner": g, "r": [float(v) for v in r]})
    atoms.append({"name": "C", "owner": OWNER["C"], "r": [0.0, 0.0, 0.0]})
    # O: bond length and angle CA-C-O from the ideal geometry, torsion τ = π.
    dO = float(np.linalg.norm(xyz["O"] - xyz["C"]))
    bO = _angle(xyz["CA"], xyz["C"], xyz["O"])
    atoms.append({"name": "O", "owner": OWNER["C"],
                  "r": [-dO * math.cos(bO), 0.0, dO * math.sin(bO)]})
    return {"name": resname, "code": rc.restype_3to1[resname], "groups": groups, "atoms": atoms}


def main():
    order = [rc.restype_1to3[c] for c in rc.restypes]  # ARNDCQEGHILKMFPSTWYV
    table = {
        "source": "transformers/models/esm/openfold_utils/residue_constants.py (Apache-2.0, (c) DeepMind, AlQuraishi Lab)",
        "generator": "tools/make_residue_table.py",
        "r_prime_deg": R_PRIME_DEG,
        "owner_codes": OWNER,
        "slots": ["phi", "psi", "omega", "chi1", "chi2", "chi3", "chi4", "chi5"],
        "types": [residue_entry(n) for n in order],
    }
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "synth", "residue_table.json")
    with open(out, "w") as f:
        json.dump(table, f, indent=1)
    n_atoms = [len(t["atoms"]) for t in table["types"]]
    print("wrote", os.path.normpath(out), "types", len(n_atoms), "mean atoms/res", sum(n_atoms) / len(n_atoms),
          "max", max(n_atoms), file=sys.stderr)


if __name__ == "__main__":
    main()
