// lrmsd.cu -- batched LRMSD loss and its gradient (§4) on sm_100a.
//
// Per chain b (x = the structure that is differentiated, y = the reference;
// reading Q19 in DESIGN.md):
//   1. barycentres and the correlation R = sum_i x~_i y~_i^T
//      -- one pass over the atoms, fp64 raw moments (sum x, sum y, sum x y^T,
//      sum |x|^2, sum |y|^2) reduced over the block, centred afterwards;
//   2. the symmetric 4x4 T of P:220-227, its largest eigenpair (lambda, q) by
//      cyclic Jacobi rotations in fp64 (one thread; 4x4 is tiny);
//   3. U(q) as printed, LRMSD = sqrt((sum|x~|^2 + |y~|^2 - 2 lambda)/N);
//   4. backward: dLRMSD/dx_i = (x~_i - U^T y~_i) / (N LRMSD) (the printed
//      P:239-241 expression with its normalisation), times dL/dLRMSD.
// The loss is HBM-bound (24 B/atom read in the forward, 36 B/atom in the
// backward); everything per atom is a streaming pass.
#include "common.cuh"
#include "kernels.h"

namespace tpl {

constexpr int kLRThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
    return v;
}

// Largest eigenpair of a symmetric 4x4 (fp64, cyclic Jacobi).  Out of line: it is
// only the fallback for a degenerate pair, and its dynamically indexed arrays
// must not put the fast path on the stack.
__device__ __noinline__ void sym4_max_eigen(double A[4][4], double* lam, double q[4]) {
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

__device__ __forceinline__ double det3(double a, double b, double c, double d, double e, double f, double g,
                                       double h, double i) {
    return a * (e * i - f * h) - b * (d * i - f * g) + c * (d * h - e * g);
}

// Largest eigenpair of the traceless symmetric 4x4 T of P:220-227, the fast way:
// Newton on its characteristic polynomial lambda^4 + c2 lambda^2 + c1 lambda + c0
// (c2 = -2 |R|_F^2, c1 = -8 det R, c0 = det T) from the upper bound e0 =
// (|x~|^2 + |y~|^2) / 2, which converges monotonically to the largest root; the
// eigenvector is the largest column of adj(T - lambda I).  A degenerate pair
// (adjugate ~ 0) falls back to Jacobi.  Returns false on fallback needed.
__device__ bool sym4_max_eigen_newton(const double T[4][4], const double R[3][3], double e0, double* lam,
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
    double l = e0;
    for (int it = 0; it < 60; ++it) {
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

__global__ void __launch_bounds__(kLRThreads) lrmsd_forward_kernel(const float* __restrict__ x,
                                                                   const float* __restrict__ y,
                                                                   const int* __restrict__ n_atoms, int stride,
                                                                   float* __restrict__ out, float* __restrict__ state,
                                                                   unsigned* __restrict__ err) {
    __shared__ double s_red[kLRThreads / 32][17];
    pdl_wait();
    const int b = blockIdx.x;
    const int N = n_atoms[b];
    if (N < 1 || N > stride) {
        if (threadIdx.x == 0) atomicOr(err, ERR_LENGTH);
        return;
    }
    const float* xb = x + (size_t)b * stride * 3;
    const float* yb = y + (size_t)b * stride * 3;
    double m[17] = {0};  // sx(3) sy(3) sxy(9, row a = x_a, col c = y_c) sxx syy
    for (int i = threadIdx.x; i < N; i += kLRThreads) {
        const double x0 = __ldg(xb + 3 * i), x1 = __ldg(xb + 3 * i + 1), x2 = __ldg(xb + 3 * i + 2);
        const double y0 = __ldg(yb + 3 * i), y1 = __ldg(yb + 3 * i + 1), y2 = __ldg(yb + 3 * i + 2);
        m[0] += x0; m[1] += x1; m[2] += x2;
        m[3] += y0; m[4] += y1; m[5] += y2;
        m[6] += x0 * y0; m[7] += x0 * y1; m[8] += x0 * y2;
        m[9] += x1 * y0; m[10] += x1 * y1; m[11] += x1 * y2;
        m[12] += x2 * y0; m[13] += x2 * y1; m[14] += x2 * y2;
        m[15] += x0 * x0 + x1 * x1 + x2 * x2;
        m[16] += y0 * y0 + y1 * y1 + y2 * y2;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 17; ++k) {
        const double v = warp_sum(m[k]);
        if (lane == 0) s_red[warp][k] = v;
    }
    __syncthreads();
    __shared__ double s_tot[17];
    if (threadIdx.x < 17) {  // the warp partials, one moment per lane (fixed order)
        double v = 0.0;
#pragma unroll
        for (int w = 0; w < kLRThreads / 32; ++w) v += s_red[w][threadIdx.x];
        s_tot[threadIdx.x] = v;
    }
    __syncwarp();
    if (threadIdx.x != 0) return;
    double s[17];
#pragma unroll
    for (int k = 0; k < 17; ++k) s[k] = s_tot[k];
    const double n = double(N);
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
    out[b] = float(v);
    float* st = state + (size_t)b * 16;
    for (int k = 0; k < 9; ++k) st[k] = float(U[k]);
    for (int k = 0; k < 3; ++k) {
        st[9 + k] = float(cx[k]);
        st[12 + k] = float(cy[k]);
    }
    // 1/(N LRMSD); 0 where LRMSD vanishes (the gradient is undefined there)
    st[15] = v > 1e-12 ? float(1.0 / (n * v)) : 0.f;
}

__global__ void __launch_bounds__(kLRThreads) lrmsd_backward_kernel(const float* __restrict__ x,
                                                                    const float* __restrict__ y,
                                                                    const int* __restrict__ n_atoms, int stride,
                                                                    const float* __restrict__ state,
                                                                    const float* __restrict__ grad_out,
                                                                    float* __restrict__ grad_x,
                                                                    unsigned* __restrict__ err) {
    pdl_wait();
    const int b = blockIdx.y;
    const int N = n_atoms[b];
    if (N < 1 || N > stride) {
        if (threadIdx.x == 0 && blockIdx.x == 0) atomicOr(err, ERR_LENGTH);
        return;
    }
    const float* st = state + (size_t)b * 16;
    float U[9], cx[3], cy[3];
#pragma unroll
    for (int k = 0; k < 9; ++k) U[k] = __ldg(st + k);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        cx[k] = __ldg(st + 9 + k);
        cy[k] = __ldg(st + 12 + k);
    }
    const float scale = __ldg(st + 15) * __ldg(grad_out + b);
    const float* xb = x + (size_t)b * stride * 3;
    const float* yb = y + (size_t)b * stride * 3;
    float* gb = grad_x + (size_t)b * stride * 3;
    for (int i = blockIdx.x * kLRThreads + threadIdx.x; i < N; i += gridDim.x * kLRThreads) {
        const float yx = __ldg(yb + 3 * i) - cy[0], yy = __ldg(yb + 3 * i + 1) - cy[1], yz = __ldg(yb + 3 * i + 2) - cy[2];
        // (U^T y~)_a = sum_c U[c][a] y~_c
        const float u0 = fmaf(U[0], yx, fmaf(U[3], yy, U[6] * yz));
        const float u1 = fmaf(U[1], yx, fmaf(U[4], yy, U[7] * yz));
        const float u2 = fmaf(U[2], yx, fmaf(U[5], yy, U[8] * yz));
        gb[3 * i + 0] = scale * (__ldg(xb + 3 * i + 0) - cx[0] - u0);
        gb[3 * i + 1] = scale * (__ldg(xb + 3 * i + 1) - cx[1] - u1);
        gb[3 * i + 2] = scale * (__ldg(xb + 3 * i + 2) - cx[2] - u2);
    }
}

cudaError_t lrmsd_forward_launch(const LRArgs& a, cudaStream_t st) {
    return launch_pdl(lrmsd_forward_kernel, a.B, kLRThreads, 0, st, a.x, a.y, a.n_atoms, a.stride, a.out, a.state,
                      a.err);
}

cudaError_t lrmsd_backward_launch(const LRArgs& a, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    const int per_chain = (a.stride + kLRThreads * 4 - 1) / (kLRThreads * 4);  // ~4 atoms per thread
    cfg.gridDim = dim3(per_chain < 1 ? 1 : per_chain, a.B);
    cfg.blockDim = dim3(kLRThreads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, lrmsd_backward_kernel, a.x, a.y, a.n_atoms, a.stride, (const float*)a.state,
                              a.grad_out, a.grad_x, a.err);
}

}  // namespace tpl
