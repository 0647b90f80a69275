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
#include "lrmsd_math.cuh"

namespace tpl {

constexpr int kLRThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
    return v;
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
    lrmsd_solve(s, double(N), out + b, state + (size_t)b * 16);
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
