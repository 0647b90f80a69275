// lrmsd_math.cuh -- steps 2-3 of the LRMSD (§4) for one
// chain from its raw fp64 moments: the 4x4 T, its largest eigenpair, U, the
// value and the backward's scale.  Shared by lrmsd.cu (the stand-alone loss)
// and backbone.cu (the fused forward).
#pragma once
#include "common.cuh"

namespace tpl {

// Phase clocks of the solve (tools/micro/solve_cost.cu defines TPL_SOLVE_CLOCKS; the
// library compiles these to nothing).
#ifdef TPL_SOLVE_CLOCKS
__device__ long long g_solve_clk[8];
#define TPL_SCLK(i) (g_solve_clk[i] = clock64())
#else
#define TPL_SCLK(i) ((void)0)
#endif

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

// Reciprocals for correction terms and normalisations whose relative error only
// needs to be small against the quantity they correct: the fp32 correctly rounded
// reciprocal (MUFU + 2 FMA) and, where a full-precision value is needed, one fp64
// Newton step on it (instead of the ~100-cycle IEEE fp64 division / sqrt sequences;
// 20 of those made the per-chain solve ~5000 cycles, tools/micro/solve_cost.cu).
static __device__ __forceinline__ double rcp_approx(double x) { return double(__frcp_rn(float(x))); }
static __device__ __forceinline__ double rcp_inrange(double x) {
    const double r = rcp_approx(x);
    return r * fma(-x, r, 2.0);  // ~1e-14 relative
}
static __device__ __forceinline__ double rsqrt_inrange(double x) {
    const double y = double(rsqrtf(float(x)));
    return y * fma(-0.5 * x * y, y, 1.5);  // Newton: ~1e-14 relative
}
// Outside the fp32 range the argument is scaled by an exact power of two (|R|-derived
// quantities reach 1e35 near a superposition of long chains); only 0, inf and NaN take
// the IEEE fp64 sequences.
static __device__ __forceinline__ double rcp_full(double x) {
    const double ax = fabs(x);
    if (ax > 1e-30 && ax < 1e30) return rcp_inrange(x);
    if (ax >= 1e30 && ax < 1e90) return rcp_inrange(x * 0x1p-200) * 0x1p-200;
    if (ax <= 1e-30 && ax > 1e-90) return rcp_inrange(x * 0x1p200) * 0x1p200;
    return 1.0 / x;
}
static __device__ __forceinline__ double rsqrt_full(double x) {
    if (x > 1e-30 && x < 1e30) return rsqrt_inrange(x);
    if (x >= 1e30 && x < 1e90) return rsqrt_inrange(x * 0x1p-200) * 0x1p-100;
    if (x <= 1e-30 && x > 1e-90) return rsqrt_inrange(x * 0x1p200) * 0x1p100;
    return 1.0 / sqrt(x);
}

static __device__ __forceinline__ double det3(double a, double b, double c, double d, double e, double f, double g,
                                       double h, double i) {
    return a * (e * i - f * h) - b * (d * i - f * g) + c * (d * h - e * g);
}

// Adjugate of a 4x4 through its twelve 2x2 minors of rows (0, 1) and (2, 3) (the
// Laplace expansion used by 4x4 inverses): 72 multiplications instead of sixteen
// 3x3 determinants; returns det as well.  adj[i][j] = (-1)^(i+j) det(a without row j, column i).
static __device__ __forceinline__ double adj4(const double a[4][4], double b[4][4]) {
    const double s0 = a[0][0] * a[1][1] - a[1][0] * a[0][1], s1 = a[0][0] * a[1][2] - a[1][0] * a[0][2];
    const double s2 = a[0][0] * a[1][3] - a[1][0] * a[0][3], s3 = a[0][1] * a[1][2] - a[1][1] * a[0][2];
    const double s4 = a[0][1] * a[1][3] - a[1][1] * a[0][3], s5 = a[0][2] * a[1][3] - a[1][2] * a[0][3];
    const double c5 = a[2][2] * a[3][3] - a[3][2] * a[2][3], c4 = a[2][1] * a[3][3] - a[3][1] * a[2][3];
    const double c3 = a[2][1] * a[3][2] - a[3][1] * a[2][2], c2 = a[2][0] * a[3][3] - a[3][0] * a[2][3];
    const double c1 = a[2][0] * a[3][2] - a[3][0] * a[2][2], c0 = a[2][0] * a[3][1] - a[3][0] * a[2][1];
    b[0][0] = a[1][1] * c5 - a[1][2] * c4 + a[1][3] * c3;
    b[0][1] = -a[0][1] * c5 + a[0][2] * c4 - a[0][3] * c3;
    b[0][2] = a[3][1] * s5 - a[3][2] * s4 + a[3][3] * s3;
    b[0][3] = -a[2][1] * s5 + a[2][2] * s4 - a[2][3] * s3;
    b[1][0] = -a[1][0] * c5 + a[1][2] * c2 - a[1][3] * c1;
    b[1][1] = a[0][0] * c5 - a[0][2] * c2 + a[0][3] * c1;
    b[1][2] = -a[3][0] * s5 + a[3][2] * s2 - a[3][3] * s1;
    b[1][3] = a[2][0] * s5 - a[2][2] * s2 + a[2][3] * s1;
    b[2][0] = a[1][0] * c4 - a[1][1] * c2 + a[1][3] * c0;
    b[2][1] = -a[0][0] * c4 + a[0][1] * c2 - a[0][3] * c0;
    b[2][2] = a[3][0] * s4 - a[3][1] * s2 + a[3][3] * s0;
    b[2][3] = -a[2][0] * s4 + a[2][1] * s2 - a[2][3] * s0;
    b[3][0] = -a[1][0] * c3 + a[1][1] * c1 - a[1][2] * c0;
    b[3][1] = a[0][0] * c3 - a[0][1] * c1 + a[0][2] * c0;
    b[3][2] = -a[3][0] * s3 + a[3][1] * s1 - a[3][2] * s0;
    b[3][3] = a[2][0] * s3 - a[2][1] * s1 + a[2][2] * s0;
    return s0 * c5 - s1 * c4 + s2 * c3 + s3 * c2 - s4 * c1 + s5 * c0;
}
static __device__ __forceinline__ double det4(const double a[4][4]) {
    const double s0 = a[0][0] * a[1][1] - a[1][0] * a[0][1], s1 = a[0][0] * a[1][2] - a[1][0] * a[0][2];
    const double s2 = a[0][0] * a[1][3] - a[1][0] * a[0][3], s3 = a[0][1] * a[1][2] - a[1][1] * a[0][2];
    const double s4 = a[0][1] * a[1][3] - a[1][1] * a[0][3], s5 = a[0][2] * a[1][3] - a[1][2] * a[0][3];
    const double c5 = a[2][2] * a[3][3] - a[3][2] * a[2][3], c4 = a[2][1] * a[3][3] - a[3][1] * a[2][3];
    const double c3 = a[2][1] * a[3][2] - a[3][1] * a[2][2], c2 = a[2][0] * a[3][3] - a[3][0] * a[2][3];
    const double c1 = a[2][0] * a[3][2] - a[3][0] * a[2][2], c0 = a[2][0] * a[3][1] - a[3][0] * a[2][1];
    return s0 * c5 - s1 * c4 + s2 * c3 + s3 * c2 - s4 * c1 + s5 * c0;
}

// Unit eigenvector of the symmetric 4x4 T for its (simple) eigenvalue l: the largest
// column of adj(T - l I), first nonzero component > 0 (as the oracle).  False when the
// adjugate vanishes (a degenerate pair: the caller falls back to Jacobi).
static __device__ __forceinline__ bool sym4_vector_at(const double T[4][4], double l, double q[4]) {
    double M[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) M[i][j] = T[i][j] - (i == j ? l : 0.0);
    // adj(M)[i][j] = (-1)^(i+j) det(M without row j, column i); keep the largest column
    double A[4][4];
    adj4(M, A);
    // the largest column, first of equals, by a two-level tournament (short dependency chain)
    double n2[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
        n2[j] = fma(A[0][j], A[0][j], A[1][j] * A[1][j]) + fma(A[2][j], A[2][j], A[3][j] * A[3][j]);
    const bool p1 = n2[1] > n2[0], p3 = n2[3] > n2[2];
    const double na = p1 ? n2[1] : n2[0], nb = p3 ? n2[3] : n2[2];
    const bool pb = nb > na;
    const double bn = pb ? nb : na;
    double best[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double a = p1 ? A[i][1] : A[i][0], b = p3 ? A[i][3] : A[i][2];
        best[i] = pb ? b : a;
    }
    TPL_SCLK(4);
    const double scale = fmax(fabs(l), 1e-300), sc2 = scale * scale;
    if (!(bn > 1e-24 * (sc2 * sc2) * sc2)) return false;  // degenerate: Jacobi
    const double inv = rsqrt_full(bn);
    // first nonzero component > 0 (as the oracle): |best_i| / |best| >= 1e-12, flags beside the rsqrt
    const bool f0 = best[0] * best[0] >= 1e-24 * bn, f1 = best[1] * best[1] >= 1e-24 * bn,
               f2 = best[2] * best[2] >= 1e-24 * bn;
    const double lead = f0 ? best[0] : f1 ? best[1] : f2 ? best[2] : best[3];
    const double sg = lead < 0.0 ? -inv : inv;
#pragma unroll
    for (int i = 0; i < 4; ++i) q[i] = best[i] * sg;
    return true;
}

// Largest eigenpair of the traceless symmetric 4x4 T of P:220-227, the fast way:
// Newton on its characteristic polynomial lambda^4 + c2 lambda^2 + c1 lambda + c0
// (c2 = -2 |R|_F^2, c1 = -8 det R, c0 = det T) from the upper bound e0 =
// (|x~|^2 + |y~|^2) / 2, which converges monotonically to the largest root; the
// eigenvector is the largest column of adj(T - lambda I).  A degenerate pair
// (adjugate ~ 0) falls back to Jacobi.  Returns false on fallback needed.
static __device__ bool sym4_max_eigen_newton(const double T[4][4], const double R[3][3], double e0, double* lam,
                                      double q[4]) {
    TPL_SCLK(0);
    double c2 = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) c2 += R[a][c] * R[a][c];
    c2 *= -2.0;
    const double c1 = -8.0 * det3(R[0][0], R[0][1], R[0][2], R[1][0], R[1][1], R[1][2], R[2][0], R[2][1], R[2][2]);
    const double c0 = det4(T);
    // Laguerre's method in fp64: every root of T's characteristic polynomial is real,
    // so from any point above the largest root the iteration decreases monotonically
    // onto it with cubic order.  Start: min(e0, sqrt(3) |R|_F) -- both bound lambda_max
    // (= s1 + s2 +- s3 in the singular values of R, <= sqrt(3 sum s^2)); the second is
    // the tight one for a random pair (e0 >> |R|): 3-4 steps on average, at most 7 over
    // random chain pairs, chain/cloud pairs and near-superpositions.  (An fp32 approach
    // from e0 landed between clustered roots for chain/cloud pairs and converged to the
    // second eigenvalue -- a wrong rotation.)
    TPL_SCLK(1);
    // e0 may carry fp32-level rounding (the fused kernel reduces |x~|^2, |y~|^2 in fp32)
    // and sits within ~1e-6 of lambda_max near a perfect superposition: start 1e-5
    // above it, and step up if the start still evaluates below the root
    double l = fmin(e0 * (1.0 + 1e-5), sqrt(-1.5 * c2) * (1.0 + 1e-12));
    for (int up = 0; up < 6; ++up) {
        const double l2 = l * l;
        if ((l2 + c2) * l2 + c1 * l + c0 > 0.0) break;
        l *= 1.0 + 1e-4 * double(1 << (2 * up));
    }
    TPL_SCLK(2);
    for (int it = 0; it < 12; ++it) {
        const double l2 = l * l;
        const double p = (l2 + c2) * l2 + c1 * l + c0;
        if (!(p > 0.0)) break;  // on the root (or just below it by rounding)
        const double dp = (4.0 * l2 + 2.0 * c2) * l + c1;
        const double ddp = 12.0 * l2 + 2.0 * c2;
        const double ip = rcp_full(p);
        const double G = dp * ip;
        const double H = fma(-ddp, ip, G * G);
        const double disc = 3.0 * fmax(4.0 * H - G * G, 0.0);
        const double den = G + (disc > 0.0 ? disc * rsqrt_full(disc) : 0.0);
        if (!(den > 0.0)) break;
        const double step = 4.0 * rcp_full(den);
        l -= step;
        if (step <= 1e-14 * fabs(l)) break;
    }
    TPL_SCLK(3);
    *lam = l;
    const bool ok = sym4_vector_at(T, l, q);
    TPL_SCLK(5);
    return ok;
}

// Largest root of lambda^4 + c2 lambda^2 + c1 lambda + c0 (T's characteristic
// polynomial, c2 = -2 |R|_F^2 < 0), cooperatively on the 32 lanes of one warp (same
// coefficients in every lane; every lane returns the root).  In mu = lambda / |R|_F
// every root lies in [-sqrt 3, sqrt 3] and lambda_max >= 0 (T is traceless):
//  1. three rounds of 32-section of [0, sqrt 3] in fp64, one sample per lane.  A
//     sample lies above every root iff p, p', p'' > 0 there (the third derivative
//     24 mu > 0 and the fourth 24 > 0: Budan-Fourier, no sign change = no root above;
//     above the largest root every derivative is positive, since their roots interlace
//     below it), so the lowest such sample brackets lambda_max to 1/32 per round.
//  2. Laguerre from the bracket's top (within 5e-5 relative): p in fp64, the step as
//     an fp32 correction -- 1-2 steps (every root is real, so the iteration decreases
//     monotonically onto the largest one).
// tools/micro/polish.cu: <= ~1100 cycles against 1100-4400 for fp64 Laguerre from the
// bound; lambda within ~1e-10 relative of the fp64 iteration's.
static __device__ __forceinline__ double quartic_max_root_warp(double c2, double c1, double c0) {
    const double s2 = -0.5 * c2;
    if (!(s2 > 1e-200)) return 0.0;  // R = 0: T = 0
    const double is = rsqrt_full(s2), sc = s2 * is;
    const double b1 = c1 * is * is * is, b0 = c0 * (is * is) * (is * is);
    const int lane = threadIdx.x & 31;
    double lo = 0.0, hi = 1.7320508075688772 * (1.0 + 1e-9);
#pragma unroll
    for (int round = 0; round < 3; ++round) {
        const double w = (hi - lo) * (1.0 / 32.0);
        const double mu = fma(w, double(lane + 1), lo);  // lane 31: hi
        const double m2 = mu * mu;
        const double p = fma(m2 - 2.0, m2, fma(b1, mu, b0));
        const double dp = fma(fma(4.0, m2, -4.0), mu, b1);
        const double ddp = fma(12.0, m2, -4.0);
        const unsigned above = __ballot_sync(0xffffffffu, p > 0.0 && dp > 0.0 && ddp > 0.0);
        const int first = above ? __ffs(above) - 1 : 31;  // the samples above every root: an upper set
        hi = fma(w, double(first + 1), lo);
        lo = hi - w;
    }
    double mu = hi;
    const float b1f = float(b1);
    for (int it = 0; it < 12; ++it) {
        const double m2 = mu * mu;
        const double p = fma(m2 - 2.0, m2, fma(b1, mu, b0));
        if (!(p > 0.0)) break;  // on the root (or just below it by rounding)
        const float mf = float(mu), pf = float(p), m2f = mf * mf;
        const float dp = fmaf(fmaf(4.f, m2f, -4.f), mf, b1f);
        const float ddp = fmaf(12.f, m2f, -4.f);
        // Laguerre (degree 4): step = 4 p / (p' + sqrt(3 (3 p'^2 - 4 p p'')))
        const float disc = fmaxf(fmaf(9.f * dp, dp, -12.f * pf * ddp), 0.f);
        const float den = dp + disc * rsqrtf(fmaxf(disc, 1e-37f));
        if (!(den > 0.f)) break;
        const float step = 4.f * pf * __frcp_rn(den);
        mu -= double(step);
        if (double(step) <= 1e-9 * fabs(mu)) break;  // the next step would be below ~1e-16
    }
    return mu * sc;
}

// U (row-major fp32) from the unit quaternion q (the eigenvector of P:220-227)
static __device__ __forceinline__ void rotation_from_q(const double q[4], float* U, float* Ulo) {
    const double q0 = q[0], q1 = q[1], q2 = q[2], q3 = q[3];
    const double Ud[9] = {q0 * q0 + q1 * q1 - q2 * q2 - q3 * q3, 2 * (q1 * q2 - q0 * q3), 2 * (q1 * q3 + q0 * q2),
                          2 * (q1 * q2 + q0 * q3), q0 * q0 - q1 * q1 + q2 * q2 - q3 * q3, 2 * (q2 * q3 - q0 * q1),
                          2 * (q1 * q3 - q0 * q2), 2 * (q2 * q3 + q0 * q1), q0 * q0 - q1 * q1 - q2 * q2 + q3 * q3};
    for (int k = 0; k < 9; ++k) {
        U[k] = float(Ud[k]);
        if (Ulo) Ulo[k] = float(Ud[k] - double(U[k]));  // U = U + Ulo to ~1e-14
    }
}

// lrmsd_rotation on one whole warp (every lane passes the same R; lane 0 writes U):
// the largest root by quartic_max_root_warp, then the adjugate eigenvector.
static __device__ __noinline__ void lrmsd_rotation_warp(const double R[3][3], float* U) {
    double T[4][4] = {
        {R[0][0] + R[1][1] + R[2][2], R[1][2] - R[2][1], R[2][0] - R[0][2], R[0][1] - R[1][0]},
        {R[1][2] - R[2][1], R[0][0] - R[1][1] - R[2][2], R[0][1] + R[1][0], R[0][2] + R[2][0]},
        {R[2][0] - R[0][2], R[0][1] + R[1][0], -R[0][0] + R[1][1] - R[2][2], R[1][2] + R[2][1]},
        {R[0][1] - R[1][0], R[0][2] + R[2][0], R[1][2] + R[2][1], -R[0][0] - R[1][1] + R[2][2]},
    };
    double rr[3];  // |R|_F^2 as three row sums (a short chain)
#pragma unroll
    for (int a = 0; a < 3; ++a) rr[a] = fma(R[a][0], R[a][0], fma(R[a][1], R[a][1], R[a][2] * R[a][2]));
    const double c2 = -2.0 * ((rr[0] + rr[1]) + rr[2]);
    const double c1 = -8.0 * det3(R[0][0], R[0][1], R[0][2], R[1][0], R[1][1], R[1][2], R[2][0], R[2][1], R[2][2]);
    const double c0 = det4(T);
    double lam = quartic_max_root_warp(c2, c1, c0), q[4];
    if (!sym4_vector_at(T, lam, q)) {
        double A[4][4];
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) A[i][j] = T[i][j];
        sym4_max_eigen(A, &lam, q);
    }
    // U's nine entries on lanes 0..8, one conversion and one store each (every lane forms all
    // nine in fp64 -- the same instructions -- and keeps its own)
    const double q0 = q[0], q1 = q[1], q2 = q[2], q3 = q[3];
    const double Ud[9] = {q0 * q0 + q1 * q1 - q2 * q2 - q3 * q3, 2 * (q1 * q2 - q0 * q3), 2 * (q1 * q3 + q0 * q2),
                          2 * (q1 * q2 + q0 * q3), q0 * q0 - q1 * q1 + q2 * q2 - q3 * q3, 2 * (q2 * q3 - q0 * q1),
                          2 * (q1 * q3 - q0 * q2), 2 * (q2 * q3 + q0 * q1), q0 * q0 - q1 * q1 - q2 * q2 + q3 * q3};
    const int lane = threadIdx.x & 31;
    double mine = Ud[0];
#pragma unroll
    for (int k = 1; k < 9; ++k) mine = lane == k ? Ud[k] : mine;
    if (lane < 9) U[lane] = float(mine);
}

// Step 2-3 without the value: U (row-major, fp32) of the optimal superposition from
// the centred correlation R = sum x~ y~^T (fp64) and e0 = (sum |x~|^2 + |y~|^2) / 2
// (an upper bound of the largest eigenvalue; only the starting point of the
// iteration).  The fused one-pass kernel computes the LRMSD itself from the
// residuals x~ - U^T y~ (a sum of squares, no cancellation).
static __device__ __noinline__ void lrmsd_rotation(const double R[3][3], double e0, float* U, float* Ulo = nullptr) {
    double T[4][4] = {
        {R[0][0] + R[1][1] + R[2][2], R[1][2] - R[2][1], R[2][0] - R[0][2], R[0][1] - R[1][0]},
        {R[1][2] - R[2][1], R[0][0] - R[1][1] - R[2][2], R[0][1] + R[1][0], R[0][2] + R[2][0]},
        {R[2][0] - R[0][2], R[0][1] + R[1][0], -R[0][0] + R[1][1] - R[2][2], R[1][2] + R[2][1]},
        {R[0][1] - R[1][0], R[0][2] + R[2][0], R[1][2] + R[2][1], -R[0][0] - R[1][1] + R[2][2]},
    };
    double lam, q[4];
    if (!sym4_max_eigen_newton(T, R, e0, &lam, q)) {
        double A[4][4];
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) A[i][j] = T[i][j];
        sym4_max_eigen(A, &lam, q);
    }
    const double q0 = q[0], q1 = q[1], q2 = q[2], q3 = q[3];
    const double Ud[9] = {q0 * q0 + q1 * q1 - q2 * q2 - q3 * q3, 2 * (q1 * q2 - q0 * q3), 2 * (q1 * q3 + q0 * q2),
                          2 * (q1 * q2 + q0 * q3), q0 * q0 - q1 * q1 + q2 * q2 - q3 * q3, 2 * (q2 * q3 - q0 * q1),
                          2 * (q1 * q3 - q0 * q2), 2 * (q2 * q3 + q0 * q1), q0 * q0 - q1 * q1 - q2 * q2 + q3 * q3};
    for (int k = 0; k < 9; ++k) {
        U[k] = float(Ud[k]);
        if (Ulo) Ulo[k] = float(Ud[k] - double(U[k]));  // U = U + Ulo to ~1e-14
    }
}

// Steps 2-3 for one chain from its raw fp64 moments s[17] (sum x, sum y, sum x y^T,
// sum |x|^2, sum |y|^2) over n atoms: writes out_b = LRMSD and st_b[16] = U (9),
// x barycentre (3), y barycentre (3), 1/(n LRMSD).
static __device__ void lrmsd_solve(const double* s, double n, float* out_b, float* st) {
    const double in = rcp_full(n);
    const double cx[3] = {s[0] * in, s[1] * in, s[2] * in}, cy[3] = {s[3] * in, s[4] * in, s[5] * in};
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
    const double e = (sxx + syy - 2.0 * lam) * in;
    const double v = e > 0.0 ? sqrt(e) : 0.0;
    *out_b = float(v);
    for (int k = 0; k < 9; ++k) st[k] = float(U[k]);
    for (int k = 0; k < 3; ++k) {
        st[9 + k] = float(cx[k]);
        st[12 + k] = float(cy[k]);
    }
    // 1/(N LRMSD); 0 where LRMSD vanishes (the gradient is undefined there)
    st[15] = v > 1e-12 ? float(rcp_full(n * v)) : 0.f;
}

}  // namespace tpl
