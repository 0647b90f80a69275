// lrmsd_math.cuh -- steps 2-3 of the LRMSD (§4) for one
// chain from its raw fp64 moments: the 4x4 T, its largest eigenpair, U, the
// value and the backward's scale.  Shared by lrmsd.cu (the stand-alone loss)
// and backbone.cu (the fused forward).
#pragma once
#include "common.cuh"

namespace tpl {

// Largest eigenpair of a symmetric 4x4 (fp64, cyclic Jacobi).  Out of line: it is
// only the fallback for a degenerate pair, and its dynamically indexed arrays
// must not put the fast path on the stack.
static __device__ __noinline__ void sym4_max_eigen(double A[4][4], double* lam, double q[4]) {
    double V[4][4];
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) V[i][j] = i == j ? 1.0 : 0.0;
    double scale = 0.0;
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) scale += A[i][j] * A[i][j];
    for (int sweep = 0; sweep < 32; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < 4; ++p)
            for (int r = p + 1; r < 4; ++r) off += A[p][r] * A[p][r];
        if (off <= 1e-30 * scale || off == 0.0) break;
        for (int p = 0; p < 4; ++p) {
            for (int r = p + 1; r < 4; ++r) {
                const double apr = A[p][r];
                if (apr == 0.0) continue;
                const double th = (A[r][r] - A[p][p]) / (2.0 * apr);
                const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
                const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < 4; ++k) {  // A <- J^T A J
                    const double akp = A[k][p], akr = A[k][r];
                    A[k][p] = c * akp - s * akr;
                    A[k][r] = s * akp + c * akr;
                }
                for (int k = 0; k < 4; ++k) {
                    const double apk = A[p][k], ark = A[r][k];
                    A[p][k] = c * apk - s * ark;
                    A[r][k] = s * apk + c * ark;
                }
                for (int k = 0; k < 4; ++k) {  // V <- V J
                    const double vkp = V[k][p], vkr = V[k][r];
                    V[k][p] = c * vkp - s * vkr;
                    V[k][r] = s * vkp + c * vkr;
                }
            }
        }
    }
    int m = 0;
    for (int i = 1; i < 4; ++i)
        if (A[i][i] > A[m][m]) m = i;
    *lam = A[m][m];
    double nrm = 0.0;
    for (int i = 0; i < 4; ++i) nrm += V[i][m] * V[i][m];
    nrm = 1.0 / sqrt(nrm);
    int first = 0;
    while (first < 3 && fabs(V[first][m]) < 1e-12) ++first;
    const double sg = V[first][m] < 0.0 ? -nrm : nrm;  // first nonzero component > 0
    for (int i = 0; i < 4; ++i) q[i] = V[i][m] * sg;
}

static __device__ __forceinline__ double det3(double a, double b, double c, double d, double e, double f, double g,
                                       double h, double i) {
    return a * (e * i - f * h) - b * (d * i - f * g) + c * (d * h - e * g);
}

// Largest eigenpair of the traceless symmetric 4x4 T of P:220-227, the fast way:
// Newton on its characteristic polynomial lambda^4 + c2 lambda^2 + c1 lambda + c0
// (c2 = -2 |R|_F^2, c1 = -8 det R, c0 = det T) from the upper bound e0 =
// (|x~|^2 + |y~|^2) / 2, which converges monotonically to the largest root; the
// eigenvector is the largest column of adj(T - lambda I).  A degenerate pair
// (adjugate ~ 0) falls back to Jacobi.  Returns false on fallback needed.
static __device__ bool sym4_max_eigen_newton(const double T[4][4], const double R[3][3], double e0, double* lam,
                                      double q[4]) {
    double c2 = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) c2 += R[a][c] * R[a][c];
    c2 *= -2.0;
    const double c1 = -8.0 * det3(R[0][0], R[0][1], R[0][2], R[1][0], R[1][1], R[1][2], R[2][0], R[2][1], R[2][2]);
    // det T by cofactors along row 0
    double c0 = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        double m[9];
        int k = 0;
#pragma unroll
        for (int r = 1; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (c != j) m[k++] = T[r][c];
        const double mn = det3(m[0], m[1], m[2], m[3], m[4], m[5], m[6], m[7], m[8]);
        c0 += ((j & 1) ? -1.0 : 1.0) * T[0][j] * mn;
    }
    // the approach from e0 in fp32 on the scaled polynomial (u = lambda / e0 in (0, 1]),
    // where Newton from far above creeps (x3/4 per step); fp64 polishes (quadratic)
    double l = e0;
    if (e0 > 0.0) {
        const double ie = 1.0 / e0;
        const float a2 = float(c2 * ie * ie), a1 = float(c1 * ie * ie * ie), a0 = float(c0 * ie * ie * ie * ie);
        float u = 1.f;
        for (int it = 0; it < 80; ++it) {
            const float u2 = u * u;
            const float p = fmaf(fmaf(u2 + a2, u, a1), u, a0);
            const float dp = fmaf(fmaf(4.f * u, u, 2.f * a2), u, a1);
            if (!(dp > 0.f)) break;
            const float nu = u - p / dp;
            if (fabsf(nu - u) <= 2e-6f * fabsf(nu)) {
                u = nu;
                break;
            }
            u = nu;
        }
        l = double(u) * e0;
    }
    for (int it = 0; it < 8; ++it) {
        const double l2 = l * l;
        const double p = (l2 + c2) * l2 + c1 * l + c0;
        const double dp = 4.0 * l2 * l + 2.0 * c2 * l + c1;
        if (dp == 0.0) break;
        const double nl = l - p / dp;
        if (fabs(nl - l) <= 1e-13 * fabs(nl)) {
            l = nl;
            break;
        }
        l = nl;
    }
    *lam = l;
    double M[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) M[i][j] = T[i][j] - (i == j ? l : 0.0);
    // adj(M)[i][j] = (-1)^(i+j) det(M without row j, column i); keep the largest column
    double best[4] = {0, 0, 0, 0}, bn = -1.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        double col[4], n2 = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            double m[9];
            int k = 0;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                if (r == j) continue;
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (c != i) m[k++] = M[r][c];
            }
            col[i] = (((i + j) & 1) ? -1.0 : 1.0) * det3(m[0], m[1], m[2], m[3], m[4], m[5], m[6], m[7], m[8]);
            n2 += col[i] * col[i];
        }
        const bool better = n2 > bn;
        bn = better ? n2 : bn;
#pragma unroll
        for (int i = 0; i < 4; ++i) best[i] = better ? col[i] : best[i];
    }
    const double scale = fmax(fabs(l), 1e-300);
    if (!(bn > 1e-24 * scale * scale * scale * scale * scale * scale)) return false;  // degenerate: Jacobi
    const double inv = 1.0 / sqrt(bn);
    // first nonzero component > 0 (as the oracle)
    const double lead = fabs(best[0]) * inv >= 1e-12 ? best[0]
                      : fabs(best[1]) * inv >= 1e-12 ? best[1]
                      : fabs(best[2]) * inv >= 1e-12 ? best[2] : best[3];
    const double sg = lead < 0.0 ? -inv : inv;
#pragma unroll
    for (int i = 0; i < 4; ++i) q[i] = best[i] * sg;
    return true;
}

// Steps 2-3 for one chain from its raw fp64 moments s[17] (sum x, sum y, sum x y^T,
// sum |x|^2, sum |y|^2) over n atoms: writes out_b = LRMSD and st_b[16] = U (9),
// x barycentre (3), y barycentre (3), 1/(n LRMSD).
static __device__ void lrmsd_solve(const double* s, double n, float* out_b, float* st) {
    const double cx[3] = {s[0] / n, s[1] / n, s[2] / n}, cy[3] = {s[3] / n, s[4] / n, s[5] / n};
    double R[3][3];  // R_ac = sum (x_a - cx_a)(y_c - cy_c) = sum x_a y_c - N cx_a cy_c
    for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 3; ++c) R[a][c] = s[6 + 3 * a + c] - n * cx[a] * cy[c];
    const double sxx = s[15] - n * (cx[0] * cx[0] + cx[1] * cx[1] + cx[2] * cx[2]);
    const double syy = s[16] - n * (cy[0] * cy[0] + cy[1] * cy[1] + cy[2] * cy[2]);
    // T, entries as printed (R_ab is 1-based there)
    double T[4][4] = {
        {R[0][0] + R[1][1] + R[2][2], R[1][2] - R[2][1], R[2][0] - R[0][2], R[0][1] - R[1][0]},
        {R[1][2] - R[2][1], R[0][0] - R[1][1] - R[2][2], R[0][1] + R[1][0], R[0][2] + R[2][0]},
        {R[2][0] - R[0][2], R[0][1] + R[1][0], -R[0][0] + R[1][1] - R[2][2], R[1][2] + R[2][1]},
        {R[0][1] - R[1][0], R[0][2] + R[2][0], R[1][2] + R[2][1], -R[0][0] - R[1][1] + R[2][2]},
    };
    double lam, q[4];
    if (!sym4_max_eigen_newton(T, R, 0.5 * (sxx + syy), &lam, q)) {
        double A[4][4];  // the fallback works on a copy (the fast path keeps T in registers)
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) A[i][j] = T[i][j];
        sym4_max_eigen(A, &lam, q);
    }
    const double q0 = q[0], q1 = q[1], q2 = q[2], q3 = q[3];
    const double U[9] = {q0 * q0 + q1 * q1 - q2 * q2 - q3 * q3, 2 * (q1 * q2 - q0 * q3), 2 * (q1 * q3 + q0 * q2),
                         2 * (q1 * q2 + q0 * q3), q0 * q0 - q1 * q1 + q2 * q2 - q3 * q3, 2 * (q2 * q3 - q0 * q1),
                         2 * (q1 * q3 - q0 * q2), 2 * (q2 * q3 + q0 * q1), q0 * q0 - q1 * q1 - q2 * q2 + q3 * q3};
    const double e = (sxx + syy - 2.0 * lam) / n;
    const double v = e > 0.0 ? sqrt(e) : 0.0;
    *out_b = float(v);
    for (int k = 0; k < 9; ++k) st[k] = float(U[k]);
    for (int k = 0; k < 3; ++k) {
        st[9 + k] = float(cx[k]);
        st[12 + k] = float(cy[k]);
    }
    // 1/(N LRMSD); 0 where LRMSD vanishes (the gradient is undefined there)
    st[15] = v > 1e-12 ? float(1.0 / (n * v)) : 0.f;
}

}  // namespace tpl
