// precise.cu -- SURVEY §8(f) row f2: an fp64-internal backbone forward.
//
// The fp32 path keeps random chains at ~1e-4 A (profiles/r01_precision_profile.md)
// but regular structures reach hundreds to thousands of Angstrom, where fp32
// rounding alone crosses the 1e-3 A gate near atom 1000.  This kernel computes
// the same map (readings Q1/Q2) entirely in fp64 -- the theta/d
// constants from the paper's decimals, fp64 sincos, fp64 transforms and scan --
// and rounds only the output coordinates to fp32.  Layout and errors as
// tpl_backbone_forward; one CTA per chain, tiles of NT*RPT residues in order.
#include "common.cuh"
#include "kernels.h"

namespace tpl {

namespace {

struct AffD {
    double r00, r01, r02, t0;
    double r10, r11, r12, t1;
    double r20, r21, r22, t2;
};

__device__ __forceinline__ AffD affd_identity() { return {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0}; }

__device__ __forceinline__ AffD affd_compose(const AffD& A, const AffD& B) {
    AffD C;
    C.r00 = A.r00 * B.r00 + A.r01 * B.r10 + A.r02 * B.r20;
    C.r01 = A.r00 * B.r01 + A.r01 * B.r11 + A.r02 * B.r21;
    C.r02 = A.r00 * B.r02 + A.r01 * B.r12 + A.r02 * B.r22;
    C.t0 = A.r00 * B.t0 + A.r01 * B.t1 + A.r02 * B.t2 + A.t0;
    C.r10 = A.r10 * B.r00 + A.r11 * B.r10 + A.r12 * B.r20;
    C.r11 = A.r10 * B.r01 + A.r11 * B.r11 + A.r12 * B.r21;
    C.r12 = A.r10 * B.r02 + A.r11 * B.r12 + A.r12 * B.r22;
    C.t1 = A.r10 * B.t0 + A.r11 * B.t1 + A.r12 * B.t2 + A.t1;
    C.r20 = A.r20 * B.r00 + A.r21 * B.r10 + A.r22 * B.r20;
    C.r21 = A.r20 * B.r01 + A.r21 * B.r11 + A.r22 * B.r21;
    C.r22 = A.r20 * B.r02 + A.r21 * B.r12 + A.r22 * B.r22;
    C.t2 = A.r20 * B.t0 + A.r21 * B.t1 + A.r22 * B.t2 + A.t2;
    return C;
}

// M <- M * R(alpha, theta, d), the printed matrix of P:149-155 (27 flops, as aff_bond)
__device__ __forceinline__ void affd_bond(AffD& M, double ca, double sa, double ct, double st, double d) {
    const double u0 = ct * M.r00 - st * M.r02, u1 = ct * M.r10 - st * M.r12, u2 = ct * M.r20 - st * M.r22;
    const double w0 = st * M.r00 + ct * M.r02, w1 = st * M.r10 + ct * M.r12, w2 = st * M.r20 + ct * M.r22;
    const double n01 = ca * M.r01 + sa * w0, n02 = ca * w0 - sa * M.r01;
    const double n11 = ca * M.r11 + sa * w1, n12 = ca * w1 - sa * M.r11;
    const double n21 = ca * M.r21 + sa * w2, n22 = ca * w2 - sa * M.r21;
    M.t0 += d * u0;
    M.t1 += d * u1;
    M.t2 += d * u2;
    M.r00 = u0; M.r10 = u1; M.r20 = u2;
    M.r01 = n01; M.r11 = n11; M.r21 = n21;
    M.r02 = n02; M.r12 = n12; M.r22 = n22;
}

__device__ __forceinline__ AffD shfl_up_affd(const AffD& a, int d) {
    AffD b;
    const unsigned m = 0xffffffffu;
    b.r00 = __shfl_up_sync(m, a.r00, d); b.r01 = __shfl_up_sync(m, a.r01, d);
    b.r02 = __shfl_up_sync(m, a.r02, d); b.t0 = __shfl_up_sync(m, a.t0, d);
    b.r10 = __shfl_up_sync(m, a.r10, d); b.r11 = __shfl_up_sync(m, a.r11, d);
    b.r12 = __shfl_up_sync(m, a.r12, d); b.t1 = __shfl_up_sync(m, a.t1, d);
    b.r20 = __shfl_up_sync(m, a.r20, d); b.r21 = __shfl_up_sync(m, a.r21, d);
    b.r22 = __shfl_up_sync(m, a.r22, d); b.t2 = __shfl_up_sync(m, a.t2, d);
    return b;
}

constexpr int kPNT = 128, kPRPT = 4, kPTile = kPNT * kPRPT;

}  // namespace

// Slot constants in fp64 from the paper's decimals.
constexpr double kPi = 3.14159265358979323846;

__global__ void __launch_bounds__(kPNT) bb_forward_precise_kernel(const float* __restrict__ angles,
                                                                  const int* __restrict__ lengths, int B, int Lmax,
                                                                  float* __restrict__ coords,
                                                                  unsigned* __restrict__ err) {
    __shared__ AffD s_w[kPNT / 32];
    __shared__ AffD s_carry;
    const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int L = lengths[b];
    if (L < 1 || L > Lmax) {
        if (tid == 0) atomicOr(err, ERR_LENGTH);
        return;
    }
    const double th[3] = {kPi - 2.1186, kPi - 1.9391, kPi - 2.0610}, bd[3] = {1.330, 1.460, 1.525};
    const double ct[3] = {cos(th[0]), cos(th[1]), cos(th[2])};
    const double st[3] = {sin(th[0]), sin(th[1]), sin(th[2])};
    const float* ang = angles + (size_t)b * Lmax * 3;
    float* out = coords + (size_t)b * Lmax * 9;
    AffD carry = affd_identity();
    for (int r0 = 0; r0 < L; r0 += kPTile) {
        const int n = min(kPTile, L - r0);
        // pass 1: the thread's residues from the identity; positions in registers
        AffD M = affd_identity();
        double px[3 * kPRPT], py[3 * kPRPT], pz[3 * kPRPT];
#pragma unroll
        for (int q = 0; q < kPRPT; ++q) {
            const int rl = tid * kPRPT + q, j = r0 + rl;
            if (rl < n) {
                const double x[3] = {j > 0 ? double(ang[3 * j - 1]) : 0.0, double(ang[3 * j]), double(ang[3 * j + 1])};
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    if (k > 0 || j > 0) {
                        double s, c;
                        sincos(x[k], &s, &c);
                        affd_bond(M, c, s, ct[k], st[k], bd[k]);
                    }
                    px[3 * q + k] = M.t0; py[3 * q + k] = M.t1; pz[3 * q + k] = M.t2;
                }
            }
        }
        // block-wide exclusive scan of the thread aggregates (left operand = lower thread)
        AffD inc = M;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const AffD o = shfl_up_affd(inc, d);
            if (lane >= d) inc = affd_compose(o, inc);
        }
        if (lane == 31) s_w[warp] = inc;
        AffD ex = shfl_up_affd(inc, 1);
        if (lane == 0) ex = affd_identity();
        __syncthreads();
        AffD p = carry;
        for (int w = 0; w < warp; ++w) p = affd_compose(p, s_w[w]);
        const AffD P = affd_compose(p, ex);
        if (tid == kPNT - 1) s_carry = affd_compose(p, inc);
        // pass 2: global positions, rounded once to fp32
#pragma unroll
        for (int q = 0; q < kPRPT; ++q) {
            const int rl = tid * kPRPT + q, j = r0 + rl;
            if (rl < n) {
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const int a = 3 * q + k;
                    float* o = out + 9 * j + 3 * k;
                    o[0] = float(P.r00 * px[a] + P.r01 * py[a] + P.r02 * pz[a] + P.t0);
                    o[1] = float(P.r10 * px[a] + P.r11 * py[a] + P.r12 * pz[a] + P.t1);
                    o[2] = float(P.r20 * px[a] + P.r21 * py[a] + P.r22 * pz[a] + P.t2);
                }
            }
        }
        __syncthreads();
        carry = s_carry;
        __syncthreads();
    }
}

cudaError_t bb_forward_precise_launch(const BBArgs& a, cudaStream_t st) {
    bb_forward_precise_kernel<<<a.B, kPNT, 0, st>>>(a.angles, a.lengths, a.B, a.Lmax, a.coords, a.err);
    return cudaGetLastError();
}

}  // namespace tpl
