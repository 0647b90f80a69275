"""fp64 LRMSD oracle (§4) -- TEST INFRASTRUCTURE ONLY.

The Coutsias-Seok-Dill quaternion method exactly as the paper outlines it:
  1. move both structures to their barycentres
  2. correlation matrix R = sum_i x_i y_i^T
  3. the symmetric 4x4 T built from R, entries as printed
  4. lambda = largest eigenvalue of T, q its eigenvector
  5. the rotation U(q), entries as printed
  6. LRMSD = sqrt((sum_i |x_i|^2 + |y_i|^2 - 2 lambda) / N)
  7. gradient: the paper prints x_i - U^T y_i; reading Q19:
     dLRMSD/dx_i = (x~_i - U^T y~_i) / (N * LRMSD), x~/y~ centred, x = the
     structure that is differentiated, y = the reference.
numpy.linalg.eigh serves as the library routine of step 4.
"""
import numpy as np


def center(x):
    x = np.asarray(x, dtype=np.float64)
    c = x.mean(axis=0)
    return x - c, c


def correlation(xc, yc):
    return np.einsum("ia,ib->ab", xc, yc)  # R_ab = sum_i x_ia y_ib


def t_matrix(R):
    (r11, r12, r13), (r21, r22, r23), (r31, r32, r33) = R
    return np.array([
        [r11 + r22 + r33, r23 - r32, r31 - r13, r12 - r21],
        [r23 - r32, r11 - r22 - r33, r12 + r21, r13 + r31],
        [r31 - r13, r12 + r21, -r11 + r22 - r33, r23 + r32],
        [r12 - r21, r13 + r31, r23 + r32, -r11 - r22 + r33],
    ])


def max_eigenpair(T):
    w, V = np.linalg.eigh(T)
    q = V[:, -1]
    if q[np.flatnonzero(np.abs(q) > 1e-12)[0]] < 0:  # sign convention: first nonzero component > 0
        q = -q
    return w[-1], q


def rotation(q):
    q0, q1, q2, q3 = q
    return np.array([
        [q0 * q0 + q1 * q1 - q2 * q2 - q3 * q3, 2 * (q1 * q2 - q0 * q3), 2 * (q1 * q3 + q0 * q2)],
        [2 * (q1 * q2 + q0 * q3), q0 * q0 - q1 * q1 + q2 * q2 - q3 * q3, 2 * (q2 * q3 - q0 * q1)],
        [2 * (q1 * q3 - q0 * q2), 2 * (q2 * q3 + q0 * q1), q0 * q0 - q1 * q1 - q2 * q2 + q3 * q3],
    ])


def lrmsd(x, y):
    """Returns (value, U, x centroid, y centroid)."""
    xc, cx = center(x)
    yc, cy = center(y)
    N = xc.shape[0]
    lam, q = max_eigenpair(t_matrix(correlation(xc, yc)))
    U = rotation(q)
    e = (np.sum(xc * xc) + np.sum(yc * yc) - 2.0 * lam) / N
    return float(np.sqrt(max(e, 0.0))), U, cx, cy


def lrmsd_grad(x, y):
    """dLRMSD/dx_i = (x~_i - U^T y~_i) / (N LRMSD)   (P:239-241 + normalisation, reading Q19)."""
    val, U, cx, cy = lrmsd(x, y)
    xc = np.asarray(x, np.float64) - cx
    yc = np.asarray(y, np.float64) - cy
    N = xc.shape[0]
    if val <= 1e-12:  # LRMSD == 0: the gradient is undefined; the ABI returns 0 there
        return np.zeros_like(xc), val
    return (xc - yc @ U) / (N * val), val  # row i: x~_i - U^T y~_i


def batch(x, y, n_atoms):
    """Per chain of padded [B, S, 3] arrays: (values [B], grads [B, S, 3]) (pads 0)."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    B = x.shape[0]
    vals = np.zeros(B)
    grads = np.zeros_like(x)
    for b in range(B):
        n = int(n_atoms[b])
        g, v = lrmsd_grad(x[b, :n], y[b, :n])
        vals[b] = v
        grads[b, :n] = g
    return vals, grads
