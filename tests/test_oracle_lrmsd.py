"""Pins of the fp64 LRMSD oracle (PAPER §4) against independent facts:
Kabsch/SVD superposition (a different algorithm), rigid invariance, a brute-force
rotation search, finite differences, translation/rotation invariance of the gradient."""
import math

import numpy as np
import pytest

from oracle import lrmsd as L


def _rot(rng):
    q = rng.standard_normal(4)
    q /= np.linalg.norm(q)
    return L.rotation(q)


def _kabsch_rmsd(x, y):
    """Minimum RMSD over proper rotations by SVD (Kabsch 1976)."""
    xc = x - x.mean(0)
    yc = y - y.mean(0)
    H = yc.T @ xc
    U, S, Vt = np.linalg.svd(H)
    d = np.sign(np.linalg.det(Vt.T @ U.T))
    D = np.diag([1.0, 1.0, d])
    Rm = Vt.T @ D @ U.T
    return math.sqrt(np.mean(np.sum((xc - yc @ Rm.T) ** 2, axis=1)))


def test_t_matrix_printed_entries():
    T = L.t_matrix(np.eye(3))
    np.testing.assert_array_equal(T, np.diag([3.0, -1.0, -1.0, -1.0]))
    R = np.random.default_rng(0).standard_normal((3, 3))
    T = L.t_matrix(R)
    np.testing.assert_allclose(T, T.T, atol=0)
    assert abs(np.trace(T)) < 1e-14


def test_rotation_of_unit_quaternion_is_proper():
    rng = np.random.default_rng(1)
    for _ in range(100):
        U = _rot(rng)
        np.testing.assert_allclose(U.T @ U, np.eye(3), atol=1e-12)
        assert abs(np.linalg.det(U) - 1.0) < 1e-12
    th = 0.7
    Ux = L.rotation([math.cos(th / 2), math.sin(th / 2), 0, 0])
    np.testing.assert_allclose(Ux, [[1, 0, 0], [0, math.cos(th), -math.sin(th)], [0, math.sin(th), math.cos(th)]],
                               atol=1e-15)


@pytest.mark.parametrize("n", [3, 5, 40, 700])
def test_value_equals_kabsch_and_superposition(n):
    rng = np.random.default_rng(n)
    for _ in range(10):
        x = rng.standard_normal((n, 3)) * 10
        y = rng.standard_normal((n, 3)) * 10
        v, U, cx, cy = L.lrmsd(x, y)
        assert abs(v - _kabsch_rmsd(x, y)) < 1e-9 * max(1.0, v)
        # the printed U superposes: sqrt(mean |x~ - U^T y~|^2) == value
        xc, yc = x - cx, y - cy
        assert abs(math.sqrt(np.mean(np.sum((xc - yc @ U) ** 2, axis=1))) - v) < 1e-9 * max(1.0, v)
        assert abs(L.lrmsd(y, x)[0] - v) < 1e-9 * max(1.0, v)


def test_rigid_invariance():
    rng = np.random.default_rng(2)
    x = rng.standard_normal((50, 3)) * 5
    for _ in range(20):
        Q = _rot(rng)
        t = rng.standard_normal(3) * 30
        assert L.lrmsd(x, x @ Q.T + t)[0] < 1e-6
        y = rng.standard_normal((50, 3))
        assert abs(L.lrmsd(x, y @ Q.T + t)[0] - L.lrmsd(x, y)[0]) < 1e-8


def test_brute_force_rotation_search():
    """SPEC oracle: grid over axis-angle rotations + local refinement (5 atoms)."""
    rng = np.random.default_rng(3)
    x = rng.standard_normal((5, 3))
    y = rng.standard_normal((5, 3))
    xc, yc = x - x.mean(0), y - y.mean(0)

    def rmsd(p):
        a = np.asarray(p)
        th = np.linalg.norm(a)
        if th < 1e-15:
            Rm = np.eye(3)
        else:
            k = a / th
            K = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
            Rm = np.eye(3) + math.sin(th) * K + (1 - math.cos(th)) * K @ K
        return math.sqrt(np.mean(np.sum((xc - yc @ Rm.T) ** 2, axis=1)))

    g = np.linspace(-math.pi, math.pi, 16)
    best = min((rmsd((a, b, c)), (a, b, c)) for a in g for b in g for c in g)
    p, step = np.array(best[1]), 0.2
    f = best[0]
    for _ in range(300):
        moved = False
        for d in range(3):
            for s in (+1, -1):
                q = p.copy()
                q[d] += s * step
                fq = rmsd(q)
                if fq < f:
                    p, f, moved = q, fq, True
        if not moved:
            step *= 0.5
    v = L.lrmsd(x, y)[0]
    assert v <= f + 1e-9 and f - v < 1e-3


def test_gradient_fd_and_invariances():
    rng = np.random.default_rng(4)
    x = rng.standard_normal((12, 3)) * 4
    y = rng.standard_normal((12, 3)) * 4
    g, v = L.lrmsd_grad(x, y)
    h = 1e-6
    fd = np.zeros_like(x)
    for i in range(12):
        for a in range(3):
            xp, xm = x.copy(), x.copy()
            xp[i, a] += h
            xm[i, a] -= h
            fd[i, a] = (L.lrmsd(xp, y)[0] - L.lrmsd(xm, y)[0]) / (2 * h)
    assert np.abs(g - fd).max() / np.abs(fd).max() < 1e-6
    np.testing.assert_allclose(g.sum(axis=0), 0.0, atol=1e-12)  # translation invariance
    W = np.array([[0, -0.3, 0.2], [0.3, 0, -0.1], [-0.2, 0.1, 0]])  # infinitesimal rotation
    assert abs(np.sum(g * ((x - x.mean(0)) @ W.T))) < 1e-10


def test_batch_padding():
    rng = np.random.default_rng(5)
    x = rng.standard_normal((3, 10, 3))
    y = rng.standard_normal((3, 10, 3))
    vals, grads = L.batch(x, y, [10, 4, 7])
    assert grads[1, 4:].max() == 0 and grads[2, 7:].max() == 0
    assert abs(vals[1] - L.lrmsd(x[1, :4], y[1, :4])[0]) < 1e-15
