"""Pins of the fp64 backbone oracle (PAPER §3) against things other than itself.

V1  printed matrix P:149-155 == factored R_y(θ)T_x(d)R_x(α) of P:32
V2  bond lengths == d          V3  bond angles == π - θ
V4  dihedrals measured back == input angles (φ, ψ, ω)
V5  L=1 closed form                          V6/V7  all-π / all-0 closed forms
V8  NeRF (Parsons et al. 2005) rebuild == chain
V9  central finite differences == Eq. 2      V10 Eq. 2 == rotation-axis suffix identity
V11 structural zeros and linearity           V14 L=2 golden fixture (tests/golden)
"""
import json
import math
import os

import numpy as np
import pytest

from conftest import BB_D, BB_THETA, angdiff, bond_angle, dihedral

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rx(a):
    c, s = math.cos(a), math.sin(a)
    return np.array([[1, 0, 0, 0], [0, c, -s, 0], [0, s, c, 0], [0, 0, 0, 1.0]])


def _ry(t):
    c, s = math.cos(t), math.sin(t)
    return np.array([[c, 0, s, 0], [0, 1, 0, 0], [-s, 0, c, 0], [0, 0, 0, 1.0]])


def _tx(d):
    m = np.eye(4)
    m[0, 3] = d
    return m


def _rand_angles(rng, B, L):
    return rng.uniform(-math.pi, math.pi, size=(B, L, 3))


# ---------------------------------------------------------------- V1
def test_printed_matrix_equals_factored_form(oracle_lib):
    rng = np.random.default_rng(1)
    for _ in range(1000):
        a, t, d = rng.uniform(-4, 4), rng.uniform(0, math.pi), rng.uniform(0.5, 2.0)
        ref = _ry(t) @ _tx(d) @ _rx(a)  # P:32, right-handed rotations (reading Q4)
        np.testing.assert_allclose(oracle_lib.bond_transform(a, t, d), ref, atol=1e-12, rtol=0)


def test_dalpha_matches_finite_difference(oracle_lib):
    rng = np.random.default_rng(2)
    h = 1e-6
    for _ in range(200):
        a, t, d = rng.uniform(-4, 4), rng.uniform(0, math.pi), rng.uniform(0.5, 2.0)
        fd = (oracle_lib.bond_transform(a + h, t, d) - oracle_lib.bond_transform(a - h, t, d)) / (2 * h)
        np.testing.assert_allclose(oracle_lib.bond_transform_dalpha(a, t, d), fd, atol=1e-8)


def test_identity_and_generator(oracle_lib):
    np.testing.assert_allclose(oracle_lib.bond_transform(0, 0, 0), np.eye(4), atol=0)
    g = oracle_lib.bond_transform_dalpha(0, 0, 0)
    ref = np.zeros((4, 4))
    ref[1, 2], ref[2, 1] = -1, 1
    np.testing.assert_allclose(g, ref, atol=0)


# ---------------------------------------------------------------- V2, V3, V4
@pytest.mark.parametrize("L", [1, 2, 5, 64, 300])
def test_bond_lengths_angles_dihedrals(oracle_lib, L):
    rng = np.random.default_rng(10 + L)
    ang = _rand_angles(rng, 3, L)
    lengths = np.full(3, L)
    X = oracle_lib.backbone_forward(ang, lengths)
    for b in range(3):
        r = X[b]
        for i in range(1, 3 * L):
            assert abs(np.linalg.norm(r[i] - r[i - 1]) - BB_D[i % 3]) < 1e-9
        for i in range(2, 3 * L):
            assert abs(bond_angle(r[i - 2], r[i - 1], r[i]) - (math.pi - BB_THETA[i % 3])) < 1e-9
        # dihedral(r_{i-2}, r_{i-1}, r_i, r_{i+1}) = alpha_i (transform i's angle)
        for j in range(L):
            if j >= 1:
                assert abs(angdiff(dihedral(r[3 * j - 1], r[3 * j], r[3 * j + 1], r[3 * j + 2]), ang[b, j, 0])) < 1e-9
            if j <= L - 2:
                assert abs(angdiff(dihedral(r[3 * j], r[3 * j + 1], r[3 * j + 2], r[3 * j + 3]), ang[b, j, 1])) < 1e-9
                assert abs(angdiff(dihedral(r[3 * j + 1], r[3 * j + 2], r[3 * j + 3], r[3 * j + 4]), ang[b, j, 2])) < 1e-9


# ---------------------------------------------------------------- V5
def test_single_residue_closed_form(oracle_lib):
    for phi in (-3.0, 0.0, 1.234):
        X = oracle_lib.backbone_forward(np.array([[[phi, 0.7, -0.3]]]), [1])[0]
        np.testing.assert_allclose(X[0], [0, 0, 0], atol=0)
        t, d = math.pi - 1.9391, 1.460
        np.testing.assert_allclose(X[1], [d * math.cos(t), 0, -d * math.sin(t)], atol=1e-15)
        np.testing.assert_allclose(X[1], [0.525648736, 0, -1.362091556], atol=1e-9)


# ---------------------------------------------------------------- V6, V7
def _planar_closed_form(L, sign):
    """r_n = sum_{k=1..n} d_k (cos A_k, 0, sin A_k); A_k = sum_{m<=k} s_m θ_m with
    s_m = (-1)^m for the all-π chain (each R_x(π) flips the y and z axes) and
    s_m = -1 for the all-0 chain (no flips)."""
    pts = [np.zeros(3)]
    A = 0.0
    for k in range(1, 3 * L):
        s = (-1) ** k if sign == "alt" else -1
        A += s * BB_THETA[k % 3]
        pts.append(pts[-1] + BB_D[k % 3] * np.array([math.cos(A), 0.0, math.sin(A)]))
    return np.array(pts)


def test_all_pi_closed_form(oracle_lib):
    L = 40
    X = oracle_lib.backbone_forward(np.full((1, L, 3), math.pi), [L])[0]
    np.testing.assert_allclose(X, _planar_closed_form(L, "alt"), atol=1e-11)
    # period-6 translation (two residues) of the extended chain
    D = X[6:] - X[:-6]
    np.testing.assert_allclose(D, np.tile(D[0], (len(D), 1)), atol=1e-11)
    with open(os.path.join(GOLDEN, "backbone_L2.json")) as f:
        g = json.load(f)
    np.testing.assert_allclose(X[:7], np.array(g["all_pi_L3_first7"]), atol=1e-8)


def test_all_zero_closed_form(oracle_lib):
    L = 25
    X = oracle_lib.backbone_forward(np.zeros((1, L, 3)), [L])[0]
    np.testing.assert_allclose(X, _planar_closed_form(L, "same"), atol=1e-11)


# ---------------------------------------------------------------- V8
def _nerf(a, b, c, d, beta, tau):
    """Natural extension reference frame placement (Parsons et al. 2005)."""
    bc = c - b
    bc /= np.linalg.norm(bc)
    n = np.cross(b - a, bc)
    n /= np.linalg.norm(n)
    m = np.stack([bc, np.cross(n, bc), n], axis=1)
    d2 = np.array([-d * math.cos(beta), d * math.sin(beta) * math.cos(tau), d * math.sin(beta) * math.sin(tau)])
    return c + m @ d2


def test_nerf_rebuild(oracle_lib):
    rng = np.random.default_rng(5)
    L = 200
    ang = _rand_angles(rng, 1, L)
    X = oracle_lib.backbone_forward(ang, [L])[0]
    alpha = {}
    for j in range(L):
        alpha[3 * j + 1], alpha[3 * j + 2] = ang[0, j, 0], ang[0, j, 1]
        alpha[3 * j + 3] = ang[0, j, 2]
    t1, d1 = BB_THETA[1], BB_D[1]
    pts = [np.array([-1.0, 0, 0]), np.zeros(3), np.array([d1 * math.cos(t1), 0, -d1 * math.sin(t1)])]
    for i in range(2, 3 * L):
        pts.append(_nerf(pts[-3], pts[-2], pts[-1], BB_D[i % 3], math.pi - BB_THETA[i % 3], alpha[i - 1]))
    np.testing.assert_allclose(X, np.array(pts[1:]), atol=1e-10)


# ---------------------------------------------------------------- V9
@pytest.mark.parametrize("L", [1, 2, 3, 7, 16])
def test_eq2_matches_finite_differences(oracle_lib, L):
    rng = np.random.default_rng(100 + L)
    ang = _rand_angles(rng, 2, L)
    g = rng.standard_normal((2, 3 * L, 3))
    lengths = np.full(2, L)
    grad = oracle_lib.backbone_backward(ang, lengths, g)
    h = 1e-6
    fd = np.zeros_like(grad)
    for j in range(L):
        for k in range(3):
            ap, am = ang.copy(), ang.copy()
            ap[:, j, k] += h
            am[:, j, k] -= h
            fp = (oracle_lib.backbone_forward(ap, lengths) * g).sum(axis=(1, 2))
            fm = (oracle_lib.backbone_forward(am, lengths) * g).sum(axis=(1, 2))
            fd[:, j, k] = (fp - fm) / (2 * h)
    for b in range(2):
        scale = max(np.abs(fd[b]).max(), 1e-300)
        assert np.abs(grad[b] - fd[b]).max() / scale < 1e-7


# ---------------------------------------------------------------- V10
def _suffix_identity(r, g):
    """grad α_i = e_i · (T_i - o_i × S_i), S_i = Σ_{j>i} g_j, T_i = Σ_{j>i} r_j × g_j,
    e_i the unit bond vector into atom i, o_i = r_i (north star identity)."""
    n = len(r)
    S = np.zeros(3)
    T = np.zeros(3)
    out = np.zeros(n)
    for i in range(n - 1, 0, -1):
        e = (r[i] - r[i - 1]) / np.linalg.norm(r[i] - r[i - 1])
        out[i] = np.dot(e, T - np.cross(r[i], S))
        S = S + g[i]
        T = T + np.cross(r[i], g[i])
    return out


def test_eq2_equals_rotation_axis_identity(oracle_lib):
    rng = np.random.default_rng(7)
    L = 120
    ang = _rand_angles(rng, 1, L)
    g = rng.standard_normal((1, 3 * L, 3))
    grad = oracle_lib.backbone_backward(ang, [L], g)[0]
    r = oracle_lib.backbone_forward(ang, [L])[0]
    ident = _suffix_identity(r, g[0])
    ref = np.zeros((L, 3))
    for i in range(1, 3 * L):
        j, k = divmod(i, 3)
        if k == 0:
            ref[j - 1, 2] = ident[i]
        else:
            ref[j, k - 1] = ident[i]
    ref[L - 1, 1] = 0.0
    np.testing.assert_allclose(grad, ref, atol=1e-9 * np.abs(ref).max())


# ---------------------------------------------------------------- V11
def test_structural_zeros_and_linearity(oracle_lib):
    rng = np.random.default_rng(8)
    L = 30
    ang = _rand_angles(rng, 1, L)
    g = np.zeros((1, 3 * L, 3))
    g[0, 0] = rng.standard_normal(3)  # loss supported on N_0 only
    assert np.abs(oracle_lib.backbone_backward(ang, [L], g)).max() == 0.0
    g1 = rng.standard_normal((1, 3 * L, 3))
    g2 = rng.standard_normal((1, 3 * L, 3))
    a, b = 0.7, -1.3
    lhs = oracle_lib.backbone_backward(ang, [L], a * g1 + b * g2)
    rhs = a * oracle_lib.backbone_backward(ang, [L], g1) + b * oracle_lib.backbone_backward(ang, [L], g2)
    np.testing.assert_allclose(lhs, rhs, atol=1e-10)
    assert lhs[0, L - 1, 1] == 0.0 and lhs[0, L - 1, 2] == 0.0  # psi_{L-1}, omega_{L-1}
    # causality: a loss on residue j's atoms gives zero gradient for every later angle
    j = 12
    g3 = np.zeros((1, 3 * L, 3))
    g3[0, 3 * j: 3 * j + 3] = rng.standard_normal((3, 3))
    gr = oracle_lib.backbone_backward(ang, [L], g3)[0]
    assert np.abs(gr[j + 1:]).max() == 0.0 and gr[j, 2] == 0.0
    assert abs(gr[j, 1]) < 1e-12  # psi_j moves only its own C_j origin: 0 up to rounding


def test_padding_untouched_and_ragged(oracle_lib):
    rng = np.random.default_rng(9)
    ang = _rand_angles(rng, 3, 10)
    lengths = np.array([10, 1, 4])
    X = oracle_lib.backbone_forward(ang, lengths)
    assert np.abs(X[1, 3:]).max() == 0 and np.abs(X[2, 12:]).max() == 0
    X2 = oracle_lib.backbone_forward(ang[2:3, :4], [4])
    np.testing.assert_array_equal(X[2, :12], X2[0])
    with pytest.raises(ValueError):
        oracle_lib.backbone_forward(ang, [10, 0, 4])
    with pytest.raises(ValueError):
        oracle_lib.backbone_forward(ang, [11, 1, 4])


# ---------------------------------------------------------------- V14
def test_golden_L2_fixture(oracle_lib):
    with open(os.path.join(GOLDEN, "backbone_L2.json")) as f:
        g = json.load(f)
    ang = np.array([g["angles"]])
    X = oracle_lib.backbone_forward(ang, [2])[0]
    np.testing.assert_allclose(X, np.array(g["coords"]), atol=g["tolerance"])
    ones = np.zeros((1, 6, 3))
    ones[..., 0] = 1.0
    ramp = (np.arange(18, dtype=float) / 10.0).reshape(1, 6, 3)
    for key, gc in (("grad_ones_x", ones), ("grad_ramp", ramp)):
        gr = oracle_lib.backbone_backward(ang, [2], gc)[0]
        np.testing.assert_allclose(gr[:, 0], g[key]["phi"], atol=g["tolerance"])
        np.testing.assert_allclose(gr[:, 1], g[key]["psi"], atol=g["tolerance"])
        np.testing.assert_allclose(gr[:, 2], g[key]["omega"], atol=g["tolerance"])
