// paper_baseline.cu -- SURVEY §8(f) row f3: the paper's own GPU design for the
// backbone model, built on sm_100a as a measured comparison point.
// It is NOT the product path: the autograd layer and the bench's headline use
// backbone.cu.  What the paper describes, and what is reproduced here:
//
//   forward  "During the forward pass, we save the cumulative transformation
//            matrices for each atom: M_i = R_0 R_1 ... R_i": one
//            thread per chain walks the chain and stores every M_i (4x4 fp32,
//            64 B/atom) and r_i = M_i 0.
//   backward dr_i/dalpha_a = M_{a-1} dR_a/dalpha M_a^{-1} M_i 0,
//            "all derivatives simultaneously on GPU" with the inverse "computed
//            on the fly", and Eq. 2's sums over i without a reduction
//            (P:252): one thread per (chain, angle) loops over every
//            downstream atom -- O(L^2) work per chain.
//
// The transform table (Q1: R_0 = I; Q2: transform 3j carries omega_{j-1}) and
// the printed matrix R are the same as the product path's; only the
// algorithm differs.
#include "common.cuh"
#include "kernels.h"

namespace tpl {

namespace {

// The printed 4x4 of P:149-155, rows 0..2 (row 3 = 0 0 0 1).
struct M34 {
    float m[12];
};

__device__ __forceinline__ void printed_R(float ca, float sa, float ct, float st, float d, M34& R) {
    R.m[0] = ct;  R.m[1] = sa * st; R.m[2] = ca * st;  R.m[3] = d * ct;
    R.m[4] = 0.f; R.m[5] = ca;      R.m[6] = -sa;      R.m[7] = 0.f;
    R.m[8] = -st; R.m[9] = sa * ct; R.m[10] = ca * ct; R.m[11] = -d * st;
}
// dR/dalpha (the translation column does not depend on alpha)
__device__ __forceinline__ void printed_dR(float ca, float sa, float ct, float st, M34& D) {
    D.m[0] = 0.f; D.m[1] = ca * st; D.m[2] = -sa * st; D.m[3] = 0.f;
    D.m[4] = 0.f; D.m[5] = -sa;     D.m[6] = -ca;      D.m[7] = 0.f;
    D.m[8] = 0.f; D.m[9] = ca * ct; D.m[10] = -sa * ct; D.m[11] = 0.f;
}
// C = A B for affine 3x4 (implicit last row 0 0 0 1); tB = 1 keeps B's translation,
// tB = 0 treats B as linear (last row 0 0 0 0: used for dR, whose 4th row is 0)
__device__ __forceinline__ void mul34(const M34& A, const M34& B, M34& C, bool affineB) {
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c)
            C.m[4 * r + c] = A.m[4 * r] * B.m[c] + A.m[4 * r + 1] * B.m[4 + c] + A.m[4 * r + 2] * B.m[8 + c];
        C.m[4 * r + 3] = A.m[4 * r] * B.m[3] + A.m[4 * r + 1] * B.m[7] + A.m[4 * r + 2] * B.m[11] +
                         (affineB ? A.m[4 * r + 3] : 0.f);
    }
}
__device__ __forceinline__ void rigid_inverse(const M34& A, M34& I) {  // [R^T | -R^T t]
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) I.m[4 * r + c] = A.m[4 * c + r];
        I.m[4 * r + 3] = -(A.m[r] * A.m[3] + A.m[4 + r] * A.m[7] + A.m[8 + r] * A.m[11]);
    }
}

__device__ __forceinline__ void slot_constants(int k, float* ct, float* st, float* d) {
    constexpr float c0 = kBBct[0], c1 = kBBct[1], c2 = kBBct[2];
    constexpr float s0 = kBBst[0], s1 = kBBst[1], s2 = kBBst[2];
    constexpr float d0 = kBBd[0], d1 = kBBd[1], d2 = kBBd[2];
    *ct = k == 0 ? c0 : k == 1 ? c1 : c2;
    *st = k == 0 ? s0 : k == 1 ? s1 : s2;
    *d = k == 0 ? d0 : k == 1 ? d1 : d2;
}

__device__ __forceinline__ float angle_of(const float* ang, int i) {  // transform i's alpha (Q1, Q2)
    const int j = i / 3, k = i - 3 * j;
    return k == 0 ? ang[3 * (j - 1) + 2] : ang[3 * j + (k - 1)];
}

}  // namespace

// One thread per chain.  Msave [B][3*Lmax][16] row-major 4x4.
__global__ void paper_bb_forward_kernel(const float* __restrict__ angles, const int* __restrict__ lengths, int B,
                                        int Lmax, float* __restrict__ coords, float* __restrict__ Msave,
                                        unsigned* __restrict__ err) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const int L = lengths[b];
    if (L < 1 || L > Lmax) {
        atomicOr(err, ERR_LENGTH);
        return;
    }
    const float* ang = angles + (size_t)b * Lmax * 3;
    float* out = coords + (size_t)b * Lmax * 9;
    float* Ms = Msave + (size_t)b * Lmax * 48;
    M34 M;
    for (int q = 0; q < 12; ++q) M.m[q] = (q % 5 == 0) ? 1.f : 0.f;  // R_0 = I (Q1)
    for (int i = 0; i < 3 * L; ++i) {
        if (i > 0) {
            float ct, st, d, s, c;
            slot_constants(i % 3, &ct, &st, &d);
            tpl_sincos(angle_of(ang, i), &s, &c);
            M34 R, T;
            printed_R(c, s, ct, st, d, R);
            mul34(M, R, T, true);
            M = T;
        }
        float4* dst = reinterpret_cast<float4*>(Ms + (size_t)i * 16);
        dst[0] = make_float4(M.m[0], M.m[1], M.m[2], M.m[3]);
        dst[1] = make_float4(M.m[4], M.m[5], M.m[6], M.m[7]);
        dst[2] = make_float4(M.m[8], M.m[9], M.m[10], M.m[11]);
        dst[3] = make_float4(0.f, 0.f, 0.f, 1.f);
        out[3 * i + 0] = M.m[3];
        out[3 * i + 1] = M.m[7];
        out[3 * i + 2] = M.m[11];
    }
}

// One thread per (chain, angle transform a >= 1); grid (ceil(3*Lmax/NT), B).
// grad(alpha_a) = sum_{i >= a} g_i . (M_{a-1} dR_a M_a^{-1} M_i 0)   (Eq. 2)
__global__ void paper_bb_backward_kernel(const float* __restrict__ angles, const int* __restrict__ lengths, int B,
                                         int Lmax, const float* __restrict__ Msave,
                                         const float* __restrict__ grad_coords, float* __restrict__ grad_angles,
                                         unsigned* __restrict__ err) {
    const int b = blockIdx.y;
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    const int L = lengths[b];
    if (L < 1 || L > Lmax) {
        if (a == 0) atomicOr(err, ERR_LENGTH);
        return;
    }
    if (a >= 3 * L) return;
    const float* ang = angles + (size_t)b * Lmax * 3;
    const float* Ms = Msave + (size_t)b * Lmax * 48;
    const float* g = grad_coords + (size_t)b * Lmax * 9;
    float* go = grad_angles + (size_t)b * Lmax * 3;
    const int j = a / 3, k = a - 3 * j;
    float sum = 0.f;
    if (a > 0) {
        float ct, st, d, s, c;
        slot_constants(k, &ct, &st, &d);
        tpl_sincos(angle_of(ang, a), &s, &c);
        M34 Mprev, Ma, dR, Ia, T1, D;
        for (int q = 0; q < 12; ++q) {
            Mprev.m[q] = Ms[(size_t)(a - 1) * 16 + q];
            Ma.m[q] = Ms[(size_t)a * 16 + q];
        }
        printed_dR(c, s, ct, st, dR);
        rigid_inverse(Ma, Ia);
        mul34(Mprev, dR, T1, false);  // M_{a-1} dR (4th row of dR is 0: no translation carried)
        // D = T1 Ia, with T1 linear in homogeneous coordinates (its last row is 0)
        for (int r = 0; r < 3; ++r) {
            for (int cc = 0; cc < 3; ++cc)
                D.m[4 * r + cc] = T1.m[4 * r] * Ia.m[cc] + T1.m[4 * r + 1] * Ia.m[4 + cc] + T1.m[4 * r + 2] * Ia.m[8 + cc];
            D.m[4 * r + 3] = T1.m[4 * r] * Ia.m[3] + T1.m[4 * r + 1] * Ia.m[7] + T1.m[4 * r + 2] * Ia.m[11] +
                             T1.m[4 * r + 3];
        }
        // no reduction: this thread walks every downstream atom
        for (int i = a; i < 3 * L; ++i) {
            const float* Mi = Ms + (size_t)i * 16;
            const float x = __ldg(Mi + 3), y = __ldg(Mi + 7), z = __ldg(Mi + 11);
            const float dx = D.m[0] * x + D.m[1] * y + D.m[2] * z + D.m[3];
            const float dy = D.m[4] * x + D.m[5] * y + D.m[6] * z + D.m[7];
            const float dz = D.m[8] * x + D.m[9] * y + D.m[10] * z + D.m[11];
            sum += __ldg(g + 3 * i) * dx + __ldg(g + 3 * i + 1) * dy + __ldg(g + 3 * i + 2) * dz;
        }
    }
    // slot of transform a: 3j+1 -> phi_j, 3j+2 -> psi_j, 3j (j >= 1) -> omega_{j-1}
    if (k == 1) go[3 * j] = sum;
    else if (k == 2) go[3 * j + 1] = (j == L - 1) ? 0.f : sum;  // psi_{L-1} moves nothing (Q2)
    else if (j >= 1) go[3 * (j - 1) + 2] = sum;
    if (a == 3 * L - 1) go[3 * (L - 1) + 2] = 0.f;  // omega_{L-1} drives no transform (Q2)
}

cudaError_t paper_bb_forward_launch(const BBArgs& a, float* Msave, cudaStream_t st) {
    const int nt = 128;
    paper_bb_forward_kernel<<<(a.B + nt - 1) / nt, nt, 0, st>>>(a.angles, a.lengths, a.B, a.Lmax, a.coords, Msave,
                                                                a.err);
    return cudaGetLastError();
}

cudaError_t paper_bb_backward_launch(const BBArgs& a, const float* Msave, cudaStream_t st) {
    const int nt = 128;
    dim3 grid((3 * a.Lmax + nt - 1) / nt, a.B);
    paper_bb_backward_kernel<<<grid, nt, 0, st>>>(a.angles, a.lengths, a.B, a.Lmax, Msave, a.grad_coords,
                                                  a.grad_angles, a.err);
    return cudaGetLastError();
}

}  // namespace tpl
