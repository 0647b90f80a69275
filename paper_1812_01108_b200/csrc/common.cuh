// common.cuh -- device building blocks of the angles->coordinates kernels (sm_100a).
//
// Math (§2/§3):
//   * a rigid transform is kept as a 3x4 affine [R | t] (the 4x4 of P:149-155
//     with its constant last row dropped);
//   * bond transform R(alpha, theta, d) = R_y(theta) T_x(d) R_x(alpha),
//     columns c0 = (ct, 0, -st), c1 = (sa st, ca, sa ct), c2 = (ca st, -sa, ca ct),
//     t = (d ct, 0, -d st)   (the printed matrix P:149-155);
//   * M_i = M_{i-1} R_i is associative, so a chain is an
//     (ordered, non-commutative) prefix scan of affines.
// Memory movement: 1D TMA bulk copies (cp.async.bulk) global<->shared with
// mbarrier completion, head/tail handled by plain loads so any 4-byte aligned
// range can be staged.
#pragma once
#include <atomic>
#include <cstdint>
#include <mutex>

#include <cuda_runtime.h>

#include "kernels.h"

namespace tpl {

// ---------------------------------------------------------------------------
// 3x4 affine, row-major: r[row][col], t[row]
struct Aff {
    float r00, r01, r02, t0;
    float r10, r11, r12, t1;
    float r20, r21, r22, t2;
};

__device__ __forceinline__ Aff aff_identity() {
    Aff a;
    a.r00 = 1.f; a.r01 = 0.f; a.r02 = 0.f; a.t0 = 0.f;
    a.r10 = 0.f; a.r11 = 1.f; a.r12 = 0.f; a.t1 = 0.f;
    a.r20 = 0.f; a.r21 = 0.f; a.r22 = 1.f; a.t2 = 0.f;
    return a;
}

// A * B (A is the earlier segment of the chain): 36 FMA.
__device__ __forceinline__ Aff aff_compose(const Aff& A, const Aff& B) {
    Aff C;
    C.r00 = fmaf(A.r00, B.r00, fmaf(A.r01, B.r10, A.r02 * B.r20));
    C.r01 = fmaf(A.r00, B.r01, fmaf(A.r01, B.r11, A.r02 * B.r21));
    C.r02 = fmaf(A.r00, B.r02, fmaf(A.r01, B.r12, A.r02 * B.r22));
    C.t0  = fmaf(A.r00, B.t0,  fmaf(A.r01, B.t1,  fmaf(A.r02, B.t2, A.t0)));
    C.r10 = fmaf(A.r10, B.r00, fmaf(A.r11, B.r10, A.r12 * B.r20));
    C.r11 = fmaf(A.r10, B.r01, fmaf(A.r11, B.r11, A.r12 * B.r21));
    C.r12 = fmaf(A.r10, B.r02, fmaf(A.r11, B.r12, A.r12 * B.r22));
    C.t1  = fmaf(A.r10, B.t0,  fmaf(A.r11, B.t1,  fmaf(A.r12, B.t2, A.t1)));
    C.r20 = fmaf(A.r20, B.r00, fmaf(A.r21, B.r10, A.r22 * B.r20));
    C.r21 = fmaf(A.r20, B.r01, fmaf(A.r21, B.r11, A.r22 * B.r21));
    C.r22 = fmaf(A.r20, B.r02, fmaf(A.r21, B.r12, A.r22 * B.r22));
    C.t2  = fmaf(A.r20, B.t0,  fmaf(A.r21, B.t1,  fmaf(A.r22, B.t2, A.t2)));
    return C;
}


// M <- M * R(alpha, theta, d) specialised to the printed matrix (27 flops):
//   u  = ct m0 - st m2,  w = st m0 + ct m2,
//   m0' = u,  m1' = ca m1 + sa w,  m2' = ca w - sa m1,  t' = t + d u
// where m0, m1, m2 are the columns of M's rotation block.
__device__ __forceinline__ void aff_bond(Aff& M, float ca, float sa, const BondC& b) {
    // rows 0 and 1 packed (fma.rn.f32x2 / mul.rn.f32x2): per-element roundings as the scalar form
    const float2 c2 = make_float2(b.ct, b.ct), s2 = make_float2(b.st, b.st), ms2 = make_float2(-b.st, -b.st);
    const float2 ca2 = make_float2(ca, ca), sa2 = make_float2(sa, sa), msa2 = make_float2(-sa, -sa);
    const float2 m0 = make_float2(M.r00, M.r10), m1 = make_float2(M.r01, M.r11), m2 = make_float2(M.r02, M.r12);
    const float2 u = __ffma2_rn(c2, m0, __fmul2_rn(ms2, m2));
    const float2 w = __ffma2_rn(s2, m0, __fmul2_rn(c2, m2));
    const float2 n1 = __ffma2_rn(ca2, m1, __fmul2_rn(sa2, w));
    const float2 n2 = __ffma2_rn(ca2, w, __fmul2_rn(msa2, m1));
    const float2 t = __ffma2_rn(make_float2(b.d, b.d), u, make_float2(M.t0, M.t1));
    const float u2 = fmaf(b.ct, M.r20, -b.st * M.r22);
    const float w2 = fmaf(b.st, M.r20, b.ct * M.r22);
    const float n21 = fmaf(ca, M.r21, sa * w2), n22 = fmaf(ca, w2, -sa * M.r21);
    M.t2 = fmaf(b.d, u2, M.t2);
    M.t0 = t.x; M.t1 = t.y;
    M.r00 = u.x; M.r10 = u.y; M.r20 = u2;
    M.r01 = n1.x; M.r11 = n1.y; M.r21 = n21;
    M.r02 = n2.x; M.r12 = n2.y; M.r22 = n22;
}

// aff_bond with the backbone constants of transform kind k as immediates.
template <int k>
__device__ __forceinline__ void aff_bond_bb(Aff& M, float ca, float sa) {
    constexpr float ct = kBBct[k], st = kBBst[k], d = kBBd[k];
    float u0 = fmaf(ct, M.r00, -st * M.r02);
    float u1 = fmaf(ct, M.r10, -st * M.r12);
    float u2 = fmaf(ct, M.r20, -st * M.r22);
    float w0 = fmaf(st, M.r00, ct * M.r02);
    float w1 = fmaf(st, M.r10, ct * M.r12);
    float w2 = fmaf(st, M.r20, ct * M.r22);
    float n01 = fmaf(ca, M.r01, sa * w0), n02 = fmaf(ca, w0, -sa * M.r01);
    float n11 = fmaf(ca, M.r11, sa * w1), n12 = fmaf(ca, w1, -sa * M.r11);
    float n21 = fmaf(ca, M.r21, sa * w2), n22 = fmaf(ca, w2, -sa * M.r21);
    M.t0 = fmaf(d, u0, M.t0);
    M.t1 = fmaf(d, u1, M.t1);
    M.t2 = fmaf(d, u2, M.t2);
    M.r00 = u0; M.r10 = u1; M.r20 = u2;
    M.r01 = n01; M.r11 = n11; M.r21 = n21;
    M.r02 = n02; M.r12 = n12; M.r22 = n22;
}

// aff_bond_bb with rows 0 and 1 as packed pairs (fma.rn.f32x2 / mul.rn.f32x2):
// the same operations and roundings per element, two thirds of the issue slots.
template <int k>
__device__ __forceinline__ void aff_bond_bb_x2(Aff& M, float ca, float sa) {
    constexpr float ct = kBBct[k], st = kBBst[k], d = kBBd[k];
    const float2 c2 = make_float2(ct, ct), s2 = make_float2(st, st), ms2 = make_float2(-st, -st);
    const float2 ca2 = make_float2(ca, ca), sa2 = make_float2(sa, sa), msa2 = make_float2(-sa, -sa);
    const float2 m0 = make_float2(M.r00, M.r10), m1 = make_float2(M.r01, M.r11), m2 = make_float2(M.r02, M.r12);
    const float2 u = __ffma2_rn(c2, m0, __fmul2_rn(ms2, m2));
    const float2 w = __ffma2_rn(s2, m0, __fmul2_rn(c2, m2));
    const float2 n1 = __ffma2_rn(ca2, m1, __fmul2_rn(sa2, w));
    const float2 n2 = __ffma2_rn(ca2, w, __fmul2_rn(msa2, m1));
    const float2 t = __ffma2_rn(make_float2(d, d), u, make_float2(M.t0, M.t1));
    const float u2 = fmaf(ct, M.r20, -st * M.r22);
    const float w2 = fmaf(st, M.r20, ct * M.r22);
    const float n21 = fmaf(ca, M.r21, sa * w2), n22 = fmaf(ca, w2, -sa * M.r21);
    M.t2 = fmaf(d, u2, M.t2);
    M.t0 = t.x; M.t1 = t.y;
    M.r00 = u.x; M.r10 = u.y; M.r20 = u2;
    M.r01 = n1.x; M.r11 = n1.y; M.r21 = n21;
    M.r02 = n2.x; M.r12 = n2.y; M.r22 = n22;
}

// M <- M * R_x(beta) (the out-of-plane R' of P:48): columns m1, m2 rotate.
__device__ __forceinline__ void aff_rot_x(Aff& M, float cb, float sb) {
    float a1 = fmaf(cb, M.r01, sb * M.r02), a2 = fmaf(cb, M.r02, -sb * M.r01);
    float b1 = fmaf(cb, M.r11, sb * M.r12), b2 = fmaf(cb, M.r12, -sb * M.r11);
    float c1 = fmaf(cb, M.r21, sb * M.r22), c2 = fmaf(cb, M.r22, -sb * M.r21);
    M.r01 = a1; M.r02 = a2; M.r11 = b1; M.r12 = b2; M.r21 = c1; M.r22 = c2;
}

// M <- M * R(alpha, theta, d)^{-1} = M * R_x(-alpha) T_x(-d) R_y(-theta)
// (rigid inverse of one bond, used to walk a side-chain branch backwards).
__device__ __forceinline__ void aff_unbond(Aff& M, float ca, float sa, const BondC& b) {
    // columns after R_x(-alpha): m1' = ca m1 - sa m2, m2' = sa m1 + ca m2
    float p0 = fmaf(ca, M.r01, -sa * M.r02), q0 = fmaf(sa, M.r01, ca * M.r02);
    float p1 = fmaf(ca, M.r11, -sa * M.r12), q1 = fmaf(sa, M.r11, ca * M.r12);
    float p2 = fmaf(ca, M.r21, -sa * M.r22), q2 = fmaf(sa, M.r21, ca * M.r22);
    // T_x(-d): t -= d m0
    float t0 = fmaf(-b.d, M.r00, M.t0), t1 = fmaf(-b.d, M.r10, M.t1), t2 = fmaf(-b.d, M.r20, M.t2);
    // R_y(-theta): m0' = ct m0 + st m2, m2' = -st m0 + ct m2 (m2 = q after the x step)
    float a0 = fmaf(b.ct, M.r00, b.st * q0), c0 = fmaf(-b.st, M.r00, b.ct * q0);
    float a1 = fmaf(b.ct, M.r10, b.st * q1), c1 = fmaf(-b.st, M.r10, b.ct * q1);
    float a2 = fmaf(b.ct, M.r20, b.st * q2), c2 = fmaf(-b.st, M.r20, b.ct * q2);
    M.r00 = a0; M.r10 = a1; M.r20 = a2;
    M.r01 = p0; M.r11 = p1; M.r21 = p2;
    M.r02 = c0; M.r12 = c1; M.r22 = c2;
    M.t0 = t0; M.t1 = t1; M.t2 = t2;
}

// One Newton-Schulz step towards the nearest rotation: R <- R (3I - R^T R) / 2.
// fp32 products of rounded rotation entries drift in scale/shear; this keeps
// the scan's aggregates orthonormal.  ~50 flops.
__device__ __forceinline__ void aff_orthonormalize(Aff& A) {
    float g00 = fmaf(A.r00, A.r00, fmaf(A.r10, A.r10, A.r20 * A.r20));
    float g11 = fmaf(A.r01, A.r01, fmaf(A.r11, A.r11, A.r21 * A.r21));
    float g22 = fmaf(A.r02, A.r02, fmaf(A.r12, A.r12, A.r22 * A.r22));
    float g01 = fmaf(A.r00, A.r01, fmaf(A.r10, A.r11, A.r20 * A.r21));
    float g02 = fmaf(A.r00, A.r02, fmaf(A.r10, A.r12, A.r20 * A.r22));
    float g12 = fmaf(A.r01, A.r02, fmaf(A.r11, A.r12, A.r21 * A.r22));
    float h00 = fmaf(-0.5f, g00, 1.5f), h11 = fmaf(-0.5f, g11, 1.5f), h22 = fmaf(-0.5f, g22, 1.5f);
    float h01 = -0.5f * g01, h02 = -0.5f * g02, h12 = -0.5f * g12;
    float a0 = fmaf(A.r00, h00, fmaf(A.r01, h01, A.r02 * h02));
    float a1 = fmaf(A.r00, h01, fmaf(A.r01, h11, A.r02 * h12));
    float a2 = fmaf(A.r00, h02, fmaf(A.r01, h12, A.r02 * h22));
    float b0 = fmaf(A.r10, h00, fmaf(A.r11, h01, A.r12 * h02));
    float b1 = fmaf(A.r10, h01, fmaf(A.r11, h11, A.r12 * h12));
    float b2 = fmaf(A.r10, h02, fmaf(A.r11, h12, A.r12 * h22));
    float c0 = fmaf(A.r20, h00, fmaf(A.r21, h01, A.r22 * h02));
    float c1 = fmaf(A.r20, h01, fmaf(A.r21, h11, A.r22 * h12));
    float c2 = fmaf(A.r20, h02, fmaf(A.r21, h12, A.r22 * h22));
    A.r00 = a0; A.r01 = a1; A.r02 = a2;
    A.r10 = b0; A.r11 = b1; A.r12 = b2;
    A.r20 = c0; A.r21 = c1; A.r22 = c2;
}

// Accurate single-precision sincos for the dihedral angles.  Fast path for
// |x| <= 2^17: x = j (pi/2) + r with a 3-term FMA Cody-Waite reduction, minimax polynomials
// on [-pi/4, pi/4] (the Cephes/CUDA coefficient set, < 1.5 ulp), quadrant
// fix-up by swaps/sign flips.  Larger |x| falls back to sincosf
// (Payne-Hanek).  ~22 instructions; no MUFU, no fast-math.
// Returned by value: taking the address of the caller's registers would force
// them to the local-memory stack on the hot path.
static __device__ __noinline__ float2 tpl_sincos_slow(float x) {
    float2 r;
    sincosf(x, &r.x, &r.y);
    return r;
}

// Branch-free fast path (valid for |x| <= 2^17); callers batch several angles
// and take the (out-of-line) slow path only when one of them is huge, so the
// polynomial evaluations of independent angles interleave (ILP).
__device__ __forceinline__ void tpl_sincos_fast(float x, float* sp, float* cp) {
    // round-to-nearest-int of x*2/pi with the 1.5*2^23 magic constant: keeps
    // the quadrant in the low mantissa bits (no FRND / F2I on the XU pipe)
    const float jm = fmaf(x, 0.636619772f, 12582912.0f);
    const int q = __float_as_int(jm);
    const float j = jm - 12582912.0f;
    // pi/2 = C1 + C2 + C3 with C1 = fl32(pi/2), C2 = fl32(pi/2 - C1), C3 = fl32(pi/2 - C1 - C2);
    // each FMA forms j*Ck exactly (emulated: max 1.47 ulp over |x| <= 1e5).
    float r = fmaf(j, -1.570796371e+00f, x);
    r = fmaf(j, 4.371138829e-08f, r);
    r = fmaf(j, 1.715124510e-15f, r);
    const float r2 = r * r;
    float s = fmaf(fmaf(-1.95152959e-4f, r2, 8.33216087e-3f), r2, -1.66666546e-1f);
    s = fmaf(s * r2, r, r);
    float c = fmaf(fmaf(2.44331571e-5f, r2, -1.38873163e-3f), r2, 4.16666457e-2f);
    c = fmaf(fmaf(c, r2, -0.5f), r2, 1.0f);
    float sn = (q & 1) ? c : s;
    float cs = (q & 1) ? s : c;
    if (q & 2) sn = -sn;
    if ((q + 1) & 2) cs = -cs;
    *sp = sn;
    *cp = cs;
}

// sincos of N angles on the hot path: fast evaluations only, and the largest
// |x| folded into *maxabs.  Kernels OR "maxabs > kSinCosFastMax" over the
// block and redo the (rare) tile with tpl_sincos_n, so the hot loop carries
// no call and no branch.
constexpr float kSinCosFastMax = 131072.0f;
template <int N>
__device__ __forceinline__ void tpl_sincos_hot(const float (&x)[N], float (&s)[N], float (&c)[N], float* maxabs) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        tpl_sincos_fast(x[i], &s[i], &c[i]);
        *maxabs = fmaxf(*maxabs, fabsf(x[i]));
    }
}

// sincos of N angles: N independent fast evaluations, then one rare branch.
template <int N>
__device__ __forceinline__ void tpl_sincos_n(const float (&x)[N], float (&s)[N], float (&c)[N]) {
    float m = 0.f;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        tpl_sincos_fast(x[i], &s[i], &c[i]);
        m = fmaxf(m, fabsf(x[i]));
    }
    if (m > 131072.0f) {  // out of line: keeps the hot loops small in the I-cache
#pragma unroll
        for (int i = 0; i < N; ++i) {
            const float2 r = tpl_sincos_slow(x[i]);
            s[i] = r.x;
            c[i] = r.y;
        }
    }
}

__device__ __forceinline__ void tpl_sincos(float x, float* sp, float* cp) {
    float xs[1] = {x}, s[1], c[1];
    tpl_sincos_n<1>(xs, s, c);
    *sp = s[0];
    *cp = c[0];
}

__device__ __forceinline__ void apply(const Aff& M, float x, float y, float z, float& ox, float& oy, float& oz) {
    ox = fmaf(M.r00, x, fmaf(M.r01, y, fmaf(M.r02, z, M.t0)));
    oy = fmaf(M.r10, x, fmaf(M.r11, y, fmaf(M.r12, z, M.t1)));
    oz = fmaf(M.r20, x, fmaf(M.r21, y, fmaf(M.r22, z, M.t2)));
}

__device__ __forceinline__ Aff shfl_up_aff(const Aff& a, int delta) {
    Aff b;
    const unsigned m = 0xffffffffu;
    b.r00 = __shfl_up_sync(m, a.r00, delta); b.r01 = __shfl_up_sync(m, a.r01, delta);
    b.r02 = __shfl_up_sync(m, a.r02, delta); b.t0 = __shfl_up_sync(m, a.t0, delta);
    b.r10 = __shfl_up_sync(m, a.r10, delta); b.r11 = __shfl_up_sync(m, a.r11, delta);
    b.r12 = __shfl_up_sync(m, a.r12, delta); b.t1 = __shfl_up_sync(m, a.t1, delta);
    b.r20 = __shfl_up_sync(m, a.r20, delta); b.r21 = __shfl_up_sync(m, a.r21, delta);
    b.r22 = __shfl_up_sync(m, a.r22, delta); b.t2 = __shfl_up_sync(m, a.t2, delta);
    return b;
}

__device__ __forceinline__ void store_aff(float* s, const Aff& a) {
    s[0] = a.r00; s[1] = a.r01; s[2] = a.r02; s[3] = a.t0;
    s[4] = a.r10; s[5] = a.r11; s[6] = a.r12; s[7] = a.t1;
    s[8] = a.r20; s[9] = a.r21; s[10] = a.r22; s[11] = a.t2;
}
__device__ __forceinline__ Aff load_aff(const float* s) {
    Aff a;
    a.r00 = s[0]; a.r01 = s[1]; a.r02 = s[2]; a.t0 = s[3];
    a.r10 = s[4]; a.r11 = s[5]; a.r12 = s[6]; a.t1 = s[7];
    a.r20 = s[8]; a.r21 = s[9]; a.r22 = s[10]; a.t2 = s[11];
    return a;
}

// ---------------------------------------------------------------------------
// Block-wide EXCLUSIVE prefix scan of per-thread chunk aggregates (ordered by
// thread index, earlier on the left).  Returns carry * A_0 * ... * A_{t-1}
// for thread t and writes carry * A_0 * ... * A_{NT-1} to *total (smem,
// visible after the call).  scratch: NT/32 * 12 floats of smem.
// Newton-Schulz policy kNS: 0 = never, 1 = on the returned prefix and the
// total only, 2 = after every combine as well, 3 = as 1 plus on each warp
// total and after each cross-warp combine.  scratch: NW * 12 floats (NW <= 4) or 2 * NW * 12.
template <int NT, int kNS>
__device__ __forceinline__ Aff block_exclusive_scan(Aff a, const Aff& carry, float* scratch, float* total) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // warp inclusive scan (Kogge-Stone); left operand = lower lane.
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        Aff o = shfl_up_aff(a, d);
        if (lane >= d) {
            a = aff_compose(o, a);
            if (kNS == 2) aff_orthonormalize(a);
        }
    }
    if (lane == 31) {
        if (kNS == 3) {  // the warp totals feed the cross-warp combines: orthonormal first
            Aff w = a;
            aff_orthonormalize(w);
            store_aff(scratch + 12 * warp, w);
        } else {
            store_aff(scratch + 12 * warp, a);
        }
    }
    Aff ex = shfl_up_aff(a, 1);
    if (lane == 0) ex = aff_identity();
    __syncthreads();
    Aff p;
    if (NW > 4) {
        // wide blocks: warp 0 scans the NW warp totals in log2(NW) steps (instead of
        // up to NW - 1 sequential composes) and leaves each warp's prefix, carry
        // included, in scratch[NW + w]; needs 2 * NW * 12 floats of scratch
        if (warp == 0) {
            Aff t = lane < NW ? load_aff(scratch + 12 * lane) : aff_identity();
#pragma unroll
            for (int d = 1; d < NW; d <<= 1) {
                const Aff o = shfl_up_aff(t, d);
                if (lane >= d) {
                    t = aff_compose(o, t);
                    if (kNS >= 2) aff_orthonormalize(t);
                }
            }
            Aff e = shfl_up_aff(t, 1);
            if (lane == 0) e = aff_identity();
            Aff pw = aff_compose(carry, e);
            if (kNS >= 2) aff_orthonormalize(pw);
            if (lane < NW) store_aff(scratch + 12 * (NW + lane), pw);
        }
        __syncthreads();
        p = load_aff(scratch + 12 * (NW + warp));
    } else {
        // prefix over the warp totals of warps < warp, starting at the carry
        p = carry;
#pragma unroll
        for (int w = 0; w < NW - 1; ++w) {
            if (w < warp) {
                p = aff_compose(p, load_aff(scratch + 12 * w));
                if (kNS >= 2) aff_orthonormalize(p);
            }
        }
    }
    Aff res = aff_compose(p, ex);
    if (kNS >= 1) aff_orthonormalize(res);
    if (threadIdx.x == NT - 1) {
        Aff tot = aff_compose(p, a);
        if (kNS >= 1) aff_orthonormalize(tot);
        store_aff(total, tot);
    }
    __syncthreads();
    return res;
}

// Block-wide EXCLUSIVE suffix sum of a 6-vector (sum over threads > t) plus a
// carry (sum over later tiles).  scratch: (2 * NT/32 * 6 + 8) floats.
// kReuse = false: the caller never touches the scratch again (no trailing barrier).
template <int NT, bool kReuse = true>
__device__ __forceinline__ void block_exclusive_suffix6(float v[6], const float carry[6], float* scratch,
                                                        float out[6], float total[6]) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float inc[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) inc[k] = v[k];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            float o = __shfl_down_sync(0xffffffffu, inc[k], d);
            if (lane + d < 32) inc[k] += o;
        }
    }
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 6; ++k) scratch[6 * warp + k] = inc[k];
    }
    float ex[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        float o = __shfl_down_sync(0xffffffffu, inc[k], 1);
        ex[k] = lane == 31 ? 0.f : o;
    }
    __syncthreads();
    if (NW > 4) {
        // wide blocks: warp 0 suffix-scans the NW warp totals in log2(NW) steps and
        // leaves each warp's later sum (carry included) and the block total in
        // scratch, instead of every thread re-adding up to 2 NW totals
        if (warp == 0) {
            float t[6];
#pragma unroll
            for (int k = 0; k < 6; ++k) t[k] = lane < NW ? scratch[6 * lane + k] : 0.f;
#pragma unroll
            for (int d = 1; d < NW; d <<= 1) {
#pragma unroll
                for (int k = 0; k < 6; ++k) {
                    const float o = __shfl_down_sync(0xffffffffu, t[k], d);
                    if (lane + d < NW) t[k] += o;
                }
            }
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                const float o = __shfl_down_sync(0xffffffffu, t[k], 1);
                if (lane < NW) scratch[6 * NW + 6 * lane + k] = carry[k] + (lane + 1 < NW ? o : 0.f);
                if (lane == 0) scratch[12 * NW + k] = carry[k] + t[k];
            }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            out[k] = scratch[6 * NW + 6 * warp + k] + ex[k];
            total[k] = scratch[12 * NW + k];
        }
        __syncthreads();
        return;
    }
    float later[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) later[k] = carry[k];
    for (int w = NW - 1; w > warp; --w) {
#pragma unroll
        for (int k = 0; k < 6; ++k) later[k] += scratch[6 * w + k];
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) out[k] = later[k] + ex[k];
    // total over the tile and all later tiles
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        float s = carry[k];
        for (int w = NW - 1; w >= 0; --w) s += scratch[6 * w + k];
        total[k] = s;
    }
    if (kReuse) __syncthreads();
}

// Block-wide exclusive prefix sum of an int (plus carry); *total = carry + sum.
template <int NT>
__device__ __forceinline__ int block_exclusive_sum_int(int v, int carry, int* scratch, int* total) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
    }
    if (lane == 31) scratch[warp] = inc;
    __syncthreads();
    int before = carry;
    int all = carry;
    for (int w = 0; w < NW; ++w) {
        int s = scratch[w];
        if (w < warp) before += s;
        all += s;
    }
    *total = all;
    __syncthreads();
    return before + inc - v;
}

// ---------------------------------------------------------------------------
// Async-proxy (TMA bulk) staging.  A global range [g, g+n) (4-byte aligned)
// is mirrored in shared memory at sbase + (g & 15) so that the 16-byte
// aligned middle part moves with one cp.async.bulk and the <16-byte head and
// tail with plain loads/stores.

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// mbarrier.init visible to the async (TMA) proxy; CTA scope is enough here
// (no clusters), and far cheaper than fence.mbarrier_init.release.cluster.
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TPL_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TPL_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Thread-block clusters (the cluster-split kernels): rank, the cluster barrier
// (arrive by every thread; wait only where a remote access follows), and
// remote shared-memory stores / mbarrier arrivals through mapa addresses.
__device__ __forceinline__ unsigned cluster_ctarank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_aligned() {  // every thread of the CTA, converged
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ void fence_mbarrier_init_cluster() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, unsigned rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, float a, float b, float c, float d) {
    asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}
__device__ __forceinline__ void st_cluster_v2(uint32_t addr, float a, float b) {
    asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(a), "f"(b) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TPL_WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TPL_WAITC_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// Inter-CTA publication (decoupled tile carries): payload with plain stores,
// then a release store of the flag; the reader acquires the flag and reads the
// payload through L2 (.cg: L1 is not coherent across SMs).
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void wait_flag(const unsigned* p, unsigned v) {
    while (ld_acquire_gpu(p) != v) __nanosleep(32);
}

// Launch epoch of the workspace (header word 1): flags written by this launch
// carry epoch + 1, so stale flags of earlier launches never match.  The last
// CTA to finish (counter in header word 2) advances the epoch.
__device__ __forceinline__ unsigned launch_epoch(const unsigned* hdr) {
    return *reinterpret_cast<const volatile unsigned*>(hdr + 1);
}
__device__ __forceinline__ void finish_epoch(unsigned* hdr) {  // call once per CTA, thread 0, at exit
    __threadfence();
    const unsigned prev = atomicAdd(hdr + 2, 1u);
    if (prev == gridDim.x - 1) {
        *reinterpret_cast<volatile unsigned*>(hdr + 2) = 0u;
        __threadfence();
        atomicAdd(hdr + 1, 1u);
    }
}

// Programmatic dependent launch (PDL).  Kernels are launched with
// programmatic stream serialization: everything before pdl_wait() (CTA
// launch, shared-memory and mbarrier setup) may overlap the tail of the
// preceding kernel; no global memory is touched before it.  pdl_trigger()
// lets the next kernel start launching; its own pdl_wait() still waits for
// this grid to complete and flush, so it never sees partial results.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Host: per-device launch state.  Everything below is keyed by the current
// device (the C ABI enqueues on the caller's stream of the current device), so a
// process driving several GPUs sets attributes and reads occupancy per device.
constexpr int kMaxDevices = 64;
inline int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev >= 0 && dev < kMaxDevices ? dev : 0;
}
// SMs of the current device (cached per device).
inline int device_sm_count() {
    static std::atomic<int> sms[kMaxDevices] = {};
    const int dev = current_device();
    int n = sms[dev].load(std::memory_order_relaxed);
    if (n == 0) {
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
        sms[dev].store(n, std::memory_order_relaxed);
    }
    return n;
}

// Per kernel instance and device: the dynamic shared-memory opt-in, raised
// monotonically to the largest size requested so far, and the co-resident grid
// (resident CTAs per SM x SMs) at that size for the persistent kernels.
// Thread-safe; the attribute call happens on first use of a size on a device
// (outside graph capture in practice).
struct LaunchCfg {
    std::atomic<size_t> smem[kMaxDevices] = {};
    std::atomic<int> cap_[kMaxDevices] = {};
    std::mutex m;
    int cap_now() const { return cap_[current_device()].load(std::memory_order_relaxed); }
};
template <typename K>
inline cudaError_t ensure_launch_cfg(LaunchCfg& c, K kernel, int block, size_t smem) {
    const int dev = current_device();
    if (c.smem[dev].load(std::memory_order_acquire) >= smem && smem > 0) return cudaSuccess;
    std::lock_guard<std::mutex> g(c.m);
    if (c.smem[dev].load(std::memory_order_relaxed) >= smem && smem > 0) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    c.cap_[dev].store(per_sm * device_sm_count(), std::memory_order_relaxed);
    c.smem[dev].store(smem, std::memory_order_release);
    return cudaSuccess;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), int grid, int block, size_t smem, cudaStream_t st,
                              Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Cluster launch (cluster dimension cl along x), PDL attribute as launch_pdl.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_cluster(void (*kernel)(KArgs...), int grid, int cl, int block, size_t smem,
                                  cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = unsigned(cl);
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// L2 prefetch of a global range (bulk, no completion tracking).  Safe before
// griddepcontrol.wait even for data the preceding kernel writes: L2 is the point of
// coherence, a prefetched line the producer rewrites later just holds the new bytes;
// nothing is consumed before the wait.  It only moves a cold input's DRAM latency
// under the previous kernel's tail.
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// Only where the launch is latency-bound (at most two chains per SM, the PDL regime):
// in the throughput regime the load follows the prefetch at once and the prefetch is a
// second request for the same lines (config 5 backward +1.4%).
__device__ __forceinline__ bool prefetch_regime(int B) {
    unsigned nsm;
    asm("mov.u32 %0, %%nsmid;" : "=r"(nsm));
    return B <= 2 * int(nsm);
}

// Split of a byte range into (head | 16-aligned middle | tail).
struct Span {
    const char* g;  // global start
    int n;          // bytes (multiple of 4 for float data, any for bytes)
    int head;       // bytes before the aligned middle
    int mid;        // aligned middle bytes (multiple of 16, may be 0)
    __device__ __forceinline__ int tail() const { return n - head - mid; }
    __device__ __forceinline__ int mis() const { return int(reinterpret_cast<uintptr_t>(g) & 15); }
};

__device__ __forceinline__ Span make_span(const void* g, int n) {
    Span s;
    s.g = static_cast<const char*>(g);
    s.n = n;
    uintptr_t a = reinterpret_cast<uintptr_t>(g);
    uintptr_t lo = (a + 15) & ~uintptr_t(15);
    uintptr_t hi = (a + n) & ~uintptr_t(15);
    if (hi > lo) {
        s.head = int(lo - a);
        s.mid = int(hi - lo);
    } else {
        s.head = n;
        s.mid = 0;
    }
    return s;
}

// Issue (one elected thread) the bulk part of a load into sbase + mis.
__device__ __forceinline__ void span_load_bulk(const Span& s, char* sbase, uint64_t* bar) {
    if (s.mid > 0) bulk_g2s(sbase + s.mis() + s.head, s.g + s.head, unsigned(s.mid), bar);
}
// All threads: head/tail bytes with plain loads (4-byte words when aligned).
__device__ __forceinline__ void span_load_edges_f32(const Span& s, char* sbase) {
    float* d = reinterpret_cast<float*>(sbase + s.mis());
    const float* g = reinterpret_cast<const float*>(s.g);
    int nh = s.head >> 2, nt = s.tail() >> 2, off_t = (s.head + s.mid) >> 2;
    for (int k = threadIdx.x; k < nh + nt; k += blockDim.x) {
        int idx = k < nh ? k : off_t + (k - nh);
        d[idx] = __ldg(g + idx);
    }
}
__device__ __forceinline__ void span_load_edges_u8(const Span& s, char* sbase) {
    char* d = sbase + s.mis();
    const unsigned char* g = reinterpret_cast<const unsigned char*>(s.g);
    int nh = s.head, nt = s.tail(), off_t = s.head + s.mid;
    for (int k = threadIdx.x; k < nh + nt; k += blockDim.x) {
        int idx = k < nh ? k : off_t + (k - nh);
        d[idx] = static_cast<char>(__ldg(g + idx));
    }
}
// Stores: data already in sbase + mis; fence + barrier must precede.
__device__ __forceinline__ void span_store_bulk(const Span& s, const char* sbase) {
    if (s.mid > 0) bulk_s2g(const_cast<char*>(s.g) + s.head, sbase + s.mis() + s.head, unsigned(s.mid));
}
__device__ __forceinline__ void span_store_edges_f32(const Span& s, const char* sbase) {
    const float* d = reinterpret_cast<const float*>(sbase + s.mis());
    float* g = reinterpret_cast<float*>(const_cast<char*>(s.g));
    int nh = s.head >> 2, nt = s.tail() >> 2, off_t = (s.head + s.mid) >> 2;
    for (int k = threadIdx.x; k < nh + nt; k += blockDim.x) {
        int idx = k < nh ? k : off_t + (k - nh);
        g[idx] = d[idx];
    }
}

// Phase timestamps for latency studies (build with -DTPL_PROFILE_PHASES; the
// product build compiles these to nothing): thread 0 of every CTA writes
// %globaltimer (ns) at phase boundaries to g_tpl_stamps[blockIdx * 16 + i]
// (read back with tpl_debug_stamps, exported by that build only).
#ifdef TPL_PROFILE_PHASES
static __device__ unsigned long long g_tpl_stamps[1 << 16];
__device__ __forceinline__ unsigned long long tpl_globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TPL_STAMP(i)                                                                    \
    do {                                                                                \
        if (threadIdx.x == 0 && blockIdx.x < 4096) g_tpl_stamps[blockIdx.x * 16 + (i)] = tpl_globaltimer(); \
    } while (0)
#else
#define TPL_STAMP(i) \
    do {             \
    } while (0)
#endif

// Device error word (workspace[0]): bit 0 = a chain length outside [1, Lmax],
// bit 1 = a restype outside the table.  The offending chain is skipped.
enum : unsigned { ERR_LENGTH = 1u, ERR_RESTYPE = 2u, ERR_STRIDE = 4u };  // ERR_STRIDE: atoms > atom_stride

}  // namespace tpl
