"""Pins of the fp64 full-atom oracle (PAPER §2) against things other than itself.

V12 backbone atoms of the full-atom model == backbone model (Fig:ErrorEstimate
    methodology, in fp64)
V13 rigidity of groups, bond geometry, χ_k measured back ==
    input, O dihedral == ψ + π, chirality of R′ (reading Q5) == the
    ideal L-residue geometry shipped in the image
V15 Eq. 1 (depth-first, O(L^2)) == central finite differences (all 20 types
    and the χ5 table); subtree locality; structural zeros
"""
import math

import numpy as np
import pytest

from conftest import BB_D, angdiff, dihedral


def _rand(rng, B, L, n_types=20):
    ang = rng.uniform(-math.pi, math.pi, size=(B, L, 8))
    rt = rng.integers(0, n_types, size=(B, L)).astype(np.uint8)
    return ang, rt


def _offsets(table, rt_row, L):
    n = [len(table["types"][t]["atoms"]) for t in rt_row[:L]]
    return np.concatenate([[0], np.cumsum(n)])


def test_threonine_topology(table):
    """threonine = 7 heavy atoms, transforms R_1(φ), R_2(χ), R_3(ψ), R_4(ω)."""
    thr = [t for t in table["types"] if t["name"] == "THR"][0]
    assert [a["name"] for a in thr["atoms"]] == ["N", "CA", "CB", "CG2", "OG1", "C", "O"]
    assert len(thr["groups"]) == 1 and thr["groups"][0]["slot"] == 3
    counts = [len(t["atoms"]) for t in table["types"]]
    assert abs(np.mean(counts) - 8.35) < 1e-9 and max(counts) == 14 and min(counts) == 4


def test_backbone_coincides_with_backbone_model(oracle_lib, table):
    rng = np.random.default_rng(1)
    B, L = 3, 40
    ang, rt = _rand(rng, B, L)
    X, nat = oracle_lib.fullatom_forward(table, ang, rt, np.full(B, L))
    Y = oracle_lib.backbone_forward(ang[..., :3], np.full(B, L))
    for b in range(B):
        off = _offsets(table, rt[b], L)
        assert nat[b] == off[-1]
        for j in range(L):
            n_j = len(table["types"][rt[b, j]]["atoms"])
            np.testing.assert_allclose(X[b, off[j]], Y[b, 3 * j], atol=1e-9)          # N
            np.testing.assert_allclose(X[b, off[j] + 1], Y[b, 3 * j + 1], atol=1e-9)  # CA
            np.testing.assert_allclose(X[b, off[j] + n_j - 2], Y[b, 3 * j + 2], atol=1e-9)  # C


@pytest.mark.parametrize("variant", ["default", "chi5"])
def test_rigidity_geometry_and_chi(oracle_lib, variant, table, table_chi5):
    tab = table if variant == "default" else table_chi5
    rng = np.random.default_rng(2)
    B, L = 4, 20
    ang, rt = _rand(rng, B, L)
    rt[0, :] = np.arange(20)  # every type at least once
    X, _ = oracle_lib.fullatom_forward(tab, ang, rt, np.full(B, L))
    for b in range(B):
        off = _offsets(tab, rt[b], L)
        for j in range(L):
            ty = tab["types"][rt[b, j]]
            at = ty["atoms"]
            R = X[b, off[j]: off[j + 1]]
            name = {a["name"]: R[k] for k, a in enumerate(at)}
            assert abs(np.linalg.norm(name["CA"] - name["N"]) - BB_D[1]) < 1e-9
            # rigidity: atoms sharing an owner keep their standard-frame distances
            for k1 in range(len(at)):
                for k2 in range(k1 + 1, len(at)):
                    if at[k1]["owner"] == at[k2]["owner"]:
                        d0 = np.linalg.norm(np.array(at[k1]["r"]) - np.array(at[k2]["r"]))
                        assert abs(np.linalg.norm(R[k1] - R[k2]) - d0) < 1e-9
            # group origins sit at distance d from the parent origin
            for g, gr in enumerate(ty["groups"]):
                origin = [k for k, a in enumerate(at) if a["owner"] == g][0]
                par = name["CA"] if gr["parent"] < 0 else R[[k for k, a in enumerate(at) if a["owner"] == gr["parent"]][0]]
                assert abs(np.linalg.norm(R[origin] - par) - gr["d"]) < 1e-9
                # chi_k measured back from the output equals the input (or the fixed value)
                if gr["chi_atoms"]:
                    chi = dihedral(*[name[n] for n in gr["chi_atoms"]])
                    want = ang[b, j, gr["slot"]] if gr["slot"] >= 0 else gr["alpha"]
                    assert abs(angdiff(chi, want)) < 1e-9
            # O is trans to N_{j+1}: dihedral N-CA-C-O = psi + pi (reading Q12)
            assert abs(angdiff(dihedral(name["N"], name["CA"], name["C"], name["O"]), ang[b, j, 1] + math.pi)) < 1e-9


def test_chirality_matches_ideal_L_residue(oracle_lib, table):
    """Reading Q5: the improper dihedral C-N-CA-CB of the model equals R′'s angle;
    its sign must match the ideal L-amino-acid geometry shipped in the image."""
    from transformers.models.esm.openfold_utils import residue_constants as rc

    ala = {n: np.array(p) for n, _, p in rc.rigid_group_atom_positions["ALA"]}
    ideal = dihedral(ala["C"], ala["N"], ala["CA"], ala["CB"])
    rng = np.random.default_rng(3)
    ang, rt = _rand(rng, 1, 6)
    rt[:] = 0  # ALA
    X, _ = oracle_lib.fullatom_forward(table, ang, rt, [6])
    for j in range(6):
        N, CA, CB, C = X[0, 5 * j: 5 * j + 4]
        model = dihedral(C, N, CA, CB)
        assert abs(angdiff(model, math.radians(-122.686))) < 1e-9
        assert abs(angdiff(model, ideal)) < math.radians(1.0)


@pytest.mark.parametrize("variant,L", [("default", 1), ("default", 3), ("default", 8), ("chi5", 6)])
def test_eq1_matches_finite_differences(oracle_lib, table, table_chi5, variant, L):
    tab = table if variant == "default" else table_chi5
    rng = np.random.default_rng(10 + L)
    B = 3
    ang, rt = _rand(rng, B, L)
    if variant == "chi5":
        rt[:] = 1  # ARG everywhere: chi1..chi5 all variable
    else:
        rt[0, :L] = np.arange(L) % 20
    lengths = np.full(B, L)
    X, nat = oracle_lib.fullatom_forward(tab, ang, rt, lengths)
    g = rng.standard_normal(X.shape)
    grad = oracle_lib.fullatom_backward(tab, ang, rt, lengths, g)
    h = 1e-6
    fd = np.zeros_like(grad)
    for j in range(L):
        for s in range(8):
            ap, am = ang.copy(), ang.copy()
            ap[:, j, s] += h
            am[:, j, s] -= h
            fp = (oracle_lib.fullatom_forward(tab, ap, rt, lengths, X.shape[1])[0] * g).sum(axis=(1, 2))
            fm = (oracle_lib.fullatom_forward(tab, am, rt, lengths, X.shape[1])[0] * g).sum(axis=(1, 2))
            fd[:, j, s] = (fp - fm) / (2 * h)
    for b in range(B):
        assert np.abs(grad[b] - fd[b]).max() / np.abs(fd[b]).max() < 1e-7
    # unused slots are exactly zero; omega_{L-1} drives nothing
    for b in range(B):
        for j in range(L):
            ty = tab["types"][rt[b, j]]
            used = {0, 1, 2} | {gr["slot"] for gr in ty["groups"] if gr["slot"] >= 0}
            for s in range(8):
                if s not in used:
                    assert grad[b, j, s] == 0.0
        assert grad[b, L - 1, 2] == 0.0


def test_subtree_locality(oracle_lib, table):
    """A loss on residue j's atoms only: every angle of residues > j, and the χ of
    residues < j... no: χ of residues < j do not move residue j -> exactly 0."""
    rng = np.random.default_rng(4)
    L = 12
    ang, rt = _rand(rng, 1, L)
    rt[0] = np.arange(L) + 1
    X, nat = oracle_lib.fullatom_forward(table, ang, rt, [L])
    off = _offsets(table, rt[0], L)
    j = 6
    g = np.zeros_like(X)
    g[0, off[j]: off[j + 1]] = rng.standard_normal((off[j + 1] - off[j], 3))
    gr = oracle_lib.fullatom_backward(table, ang, rt, [L], g)[0]
    assert np.abs(gr[j + 1:]).max() == 0.0
    assert np.abs(gr[:j, 3:]).max() == 0.0  # side chains of earlier residues
    assert gr[j, 2] == 0.0  # omega_j moves residue j+1 only
    assert np.abs(gr[:j, :3]).max() > 0.0


def test_psi_last_moves_O(oracle_lib, table):
    rng = np.random.default_rng(5)
    L = 4
    ang, rt = _rand(rng, 1, L)
    X, _ = oracle_lib.fullatom_forward(table, ang, rt, [L])
    g = rng.standard_normal(X.shape)
    gr = oracle_lib.fullatom_backward(table, ang, rt, [L], g)[0]
    assert abs(gr[L - 1, 1]) > 1e-6 and gr[L - 1, 2] == 0.0


def test_input_validation(oracle_lib, table):
    ang = np.zeros((1, 3, 8))
    with pytest.raises(ValueError):
        oracle_lib.fullatom_forward(table, ang, np.array([[0, 1, 25]], dtype=np.uint8), [3])
    with pytest.raises(ValueError):
        oracle_lib.fullatom_forward(table, ang, np.zeros((1, 3), dtype=np.uint8), [0])
    with pytest.raises(ValueError):
        oracle_lib.fullatom_forward(table, ang, np.zeros((1, 3), dtype=np.uint8), [3], atom_stride=10)


# Textbook covalent radii (Å) of the heavy elements in the 20 residues; a bond is a
# pair closer than r1 + r2 + 0.25 Å.  Independent of the table generator (reading Q8).
_COV = {"C": 0.76, "N": 0.71, "O": 0.66, "S": 1.05}


def _element(atom_name):
    return atom_name[0]


def _bond_angles(R, bond):
    out = {}
    for k in range(len(R)):
        nbr = np.nonzero(bond[k])[0]
        for i1 in range(len(nbr)):
            for i2 in range(i1 + 1, len(nbr)):
                u, v = R[nbr[i1]] - R[k], R[nbr[i2]] - R[k]
                out[(nbr[i1], k, nbr[i2])] = math.degrees(
                    math.acos(np.dot(u, v) / np.linalg.norm(u) / np.linalg.norm(v)))
    return out


def test_side_chain_covalent_geometry(oracle_lib, table):
    """Reading Q8 pin against chemistry rather than the table itself: the placed side
    chains have the standard covalent geometry (Engh & Huber 1991).

    At the all-trans rotamer (every χ = π, random φ/ψ/ω) the bond graph (pairs closer
    than the sum of covalent radii + 0.25 Å) over N, CA, side chain, C, O is
    connected; bonds are 1.2-1.9 Å; bond angles are 100-135° (5-ring exocyclic angles
    reach 131°); 1-3 pairs are 2.1-2.9 Å apart (carboxylate O-O 2.19 Å, CA-SG 2.8 Å),
    farther pairs > 1.9 Å except with O (ψ is random: O may clash with the side chain); CA-CB = 1.53 Å; N-CA-CB = 110.5° (PRO 103.0°); PHE/TYR
    rings are planar.  C-CA-CB follows from the paper's N-CA-C (reading Q7) and is
    skipped.  Under random χ every bond length and bond angle is unchanged (torsions
    move no covalent geometry)."""
    rng = np.random.default_rng(11)
    B, L = 3, 20
    ang, rt = _rand(rng, B, L)
    rt[0, :] = np.arange(20)
    trans = ang.copy()
    trans[..., 3:] = math.pi
    X0, _ = oracle_lib.fullatom_forward(table, trans, rt, np.full(B, L))
    X1, _ = oracle_lib.fullatom_forward(table, ang, rt, np.full(B, L))
    checked = set()
    for b in range(B):
        off = _offsets(table, rt[b], L)
        for j in range(L):
            ty = table["types"][rt[b, j]]
            names = [a["name"] for a in ty["atoms"]]
            n = len(names)
            R = X0[b, off[j]: off[j + 1]]
            pos = dict(zip(names, R))
            D = np.linalg.norm(R[:, None] - R[None], axis=-1)
            cut = np.array([[_COV[_element(a)] + _COV[_element(c)] + 0.25 for c in names] for a in names])
            bond = (D < cut) & ~np.eye(n, dtype=bool)
            assert np.all((D[bond] > 1.2) & (D[bond] < 1.9)), (ty["name"], D[bond])
            # bond-graph distances (BFS from every atom); the graph is connected
            hops = np.full((n, n), -1)
            for s0 in range(n):
                hops[s0, s0], todo = 0, [s0]
                while todo:
                    k = todo.pop(0)
                    for m in np.nonzero(bond[k])[0]:
                        if hops[s0, m] < 0:
                            hops[s0, m] = hops[s0, k] + 1
                            todo.append(m)
            assert np.all(hops >= 0), (ty["name"], [names[k] for k in range(n) if hops[0, k] < 0])
            assert np.all((D[hops == 2] > 2.1) & (D[hops == 2] < 2.9)), (ty["name"], sorted(D[hops == 2]))
            far = (hops >= 3) & ~np.isin(np.array(names), ["O"])[:, None] & ~np.isin(np.array(names), ["O"])[None]
            assert np.all(D[far] > 1.9), (ty["name"], [(names[p], names[q], D[p, q]) for p, q in zip(*np.nonzero(far & (D <= 1.9)))])
            ba = _bond_angles(R, bond)
            for (i, k, m), a in ba.items():
                if names[k] == "CA" and "C" in (names[i], names[m]):
                    continue  # fixed by the paper's backbone constants (reading Q7)
                assert 100.0 < a < 135.0, (ty["name"], names[i], names[k], names[m], a)
            if "CB" in pos:
                assert abs(np.linalg.norm(pos["CB"] - pos["CA"]) - 1.53) < 0.03, ty["name"]
                u, v = pos["N"] - pos["CA"], pos["CB"] - pos["CA"]
                a = math.degrees(math.acos(np.dot(u, v) / np.linalg.norm(u) / np.linalg.norm(v)))
                assert abs(a - (103.0 if ty["name"] == "PRO" else 110.5)) < 2.0, (ty["name"], a)
            if ty["name"] in ("PHE", "TYR"):
                P = np.array([pos[a] for a in ("CG", "CD1", "CD2", "CE1", "CE2", "CZ")])
                assert np.linalg.svd(P - P.mean(0), compute_uv=False)[-1] < 0.02, ty["name"]
            # random chi: the same covalent geometry
            R1 = X1[b, off[j]: off[j + 1]]
            D1 = np.linalg.norm(R1[:, None] - R1[None], axis=-1)
            np.testing.assert_allclose(D1[bond], D[bond], atol=1e-9)
            ba1 = _bond_angles(R1, bond)
            for key, a in ba.items():
                assert abs(ba1[key] - a) < 1e-6, (ty["name"], key)
            checked.add(ty["name"])
    assert len(checked) == 20
