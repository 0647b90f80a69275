// packed.cuh -- building blocks of the packed backbone kernels (packed.cu,
// fused_lrmsd.cu): pairs of 3x4 affines in the two lanes of f32x2 registers
// (fma.rn.f32x2 / mul.rn.f32x2 / add.rn.f32x2 on sm_100a), packed sincos, vector
// shared-memory runs, per-warp staging I/O, and the launch policy.
#pragma once
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace tpl {

// ---------------------------------------------------------------------------
// Packed pair of 3x4 affines (.x = run A, .y = run B).
struct Aff2 {
    float2 r00, r01, r02, t0;
    float2 r10, r11, r12, t1;
    float2 r20, r21, r22, t2;
};

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

// One row of M <- M R(alpha, theta, d) (common.cuh aff_bond_bb, per lane).
template <int k>
__device__ __forceinline__ void row_bond2(float2& m0, float2& m1, float2& m2, float2& t, float2 ca, float2 sa,
                                          float2 msa) {
    constexpr float ct = kBBct[k], st = kBBst[k], d = kBBd[k];
    const float2 u = __ffma2_rn(f2(ct), m0, __fmul2_rn(f2(-st), m2));
    const float2 w = __ffma2_rn(f2(st), m0, __fmul2_rn(f2(ct), m2));
    const float2 n1 = __ffma2_rn(ca, m1, __fmul2_rn(sa, w));
    const float2 n2 = __ffma2_rn(ca, w, __fmul2_rn(msa, m1));
    t = __ffma2_rn(f2(d), u, t);
    m0 = u;
    m1 = n1;
    m2 = n2;
}

template <int k>
__device__ __forceinline__ void aff2_bond(Aff2& M, float2 ca, float2 sa) {
    const float2 msa = make_float2(-sa.x, -sa.y);
    row_bond2<k>(M.r00, M.r01, M.r02, M.t0, ca, sa, msa);
    row_bond2<k>(M.r10, M.r11, M.r12, M.t1, ca, sa, msa);
    row_bond2<k>(M.r20, M.r21, M.r22, M.t2, ca, sa, msa);
}

// M = R(alpha, theta_k, d_k) itself: the bond update applied to the identity,
// with the same per-element results (products of one rounding each).
template <int k>
__device__ __forceinline__ void aff2_from_bond(Aff2& M, float2 ca, float2 sa) {
    constexpr float ct = kBBct[k], st = kBBst[k], d = kBBd[k];
    M.r00 = f2(ct);
    M.r10 = f2(0.f);
    M.r20 = f2(-st);
    M.r01 = __fmul2_rn(sa, f2(st));
    M.r11 = ca;
    M.r21 = __fmul2_rn(sa, f2(ct));
    M.r02 = __fmul2_rn(ca, f2(st));
    M.r12 = make_float2(-sa.x, -sa.y);
    M.r22 = __fmul2_rn(ca, f2(ct));
    M.t0 = f2(d * ct);
    M.t1 = f2(0.f);
    M.t2 = f2(-(d * st));
}

__device__ __forceinline__ Aff lane_x(const Aff2& M) {
    return Aff{M.r00.x, M.r01.x, M.r02.x, M.t0.x, M.r10.x, M.r11.x, M.r12.x, M.t1.x, M.r20.x, M.r21.x, M.r22.x, M.t2.x};
}
__device__ __forceinline__ Aff lane_y(const Aff2& M) {
    return Aff{M.r00.y, M.r01.y, M.r02.y, M.t0.y, M.r10.y, M.r11.y, M.r12.y, M.t1.y, M.r20.y, M.r21.y, M.r22.y, M.t2.y};
}
__device__ __forceinline__ void set_lane_x(Aff2& M, const Aff& a) {
    M.r00.x = a.r00; M.r01.x = a.r01; M.r02.x = a.r02; M.t0.x = a.t0;
    M.r10.x = a.r10; M.r11.x = a.r11; M.r12.x = a.r12; M.t1.x = a.t1;
    M.r20.x = a.r20; M.r21.x = a.r21; M.r22.x = a.r22; M.t2.x = a.t2;
}
__device__ __forceinline__ Aff2 pack2(const Aff& a, const Aff& b) {
    Aff2 M;
    M.r00 = make_float2(a.r00, b.r00); M.r01 = make_float2(a.r01, b.r01);
    M.r02 = make_float2(a.r02, b.r02); M.t0 = make_float2(a.t0, b.t0);
    M.r10 = make_float2(a.r10, b.r10); M.r11 = make_float2(a.r11, b.r11);
    M.r12 = make_float2(a.r12, b.r12); M.t1 = make_float2(a.t1, b.t1);
    M.r20 = make_float2(a.r20, b.r20); M.r21 = make_float2(a.r21, b.r21);
    M.r22 = make_float2(a.r22, b.r22); M.t2 = make_float2(a.t2, b.t2);
    return M;
}

// (x, y, z) <- M (x, y, z, 1) per lane (common.cuh apply).
__device__ __forceinline__ void apply2(const Aff2& M, float2 x, float2 y, float2 z, float2& ox, float2& oy,
                                       float2& oz) {
    ox = __ffma2_rn(M.r00, x, __ffma2_rn(M.r01, y, __ffma2_rn(M.r02, z, M.t0)));
    oy = __ffma2_rn(M.r10, x, __ffma2_rn(M.r11, y, __ffma2_rn(M.r12, z, M.t1)));
    oz = __ffma2_rn(M.r20, x, __ffma2_rn(M.r21, y, __ffma2_rn(M.r22, z, M.t2)));
}

// Packed fast sincos: tpl_sincos_fast per lane (common.cuh), the reduction and
// both polynomials as f32x2 operations, the quadrant fix-up per lane.
__device__ __forceinline__ void sincos2_fast(float2 x, float2& s, float2& c, float& maxabs) {
    const float2 jm = __ffma2_rn(x, f2(0.636619772f), f2(12582912.0f));
    const int qx = __float_as_int(jm.x), qy = __float_as_int(jm.y);
    const float2 j = __fadd2_rn(jm, f2(-12582912.0f));
    float2 r = __ffma2_rn(j, f2(-1.570796371e+00f), x);
    r = __ffma2_rn(j, f2(4.371138829e-08f), r);
    r = __ffma2_rn(j, f2(1.715124510e-15f), r);
    const float2 r2 = __fmul2_rn(r, r);
    float2 sp = __ffma2_rn(__ffma2_rn(f2(-1.95152959e-4f), r2, f2(8.33216087e-3f)), r2, f2(-1.66666546e-1f));
    sp = __ffma2_rn(__fmul2_rn(sp, r2), r, r);
    float2 cp = __ffma2_rn(__ffma2_rn(f2(2.44331571e-5f), r2, f2(-1.38873163e-3f)), r2, f2(4.16666457e-2f));
    cp = __ffma2_rn(__ffma2_rn(cp, r2, f2(-0.5f)), r2, f2(1.0f));
    float snx = (qx & 1) ? cp.x : sp.x, csx = (qx & 1) ? sp.x : cp.x;
    float sny = (qy & 1) ? cp.y : sp.y, csy = (qy & 1) ? sp.y : cp.y;
    // sign flips as sign-bit xors (quadrant bits 1 of q and q + 1)
    snx = __int_as_float(__float_as_int(snx) ^ ((qx & 2) << 30));
    csx = __int_as_float(__float_as_int(csx) ^ (((qx + 1) & 2) << 30));
    sny = __int_as_float(__float_as_int(sny) ^ ((qy & 2) << 30));
    csy = __int_as_float(__float_as_int(csy) ^ (((qy + 1) & 2) << 30));
    s = make_float2(snx, sny);
    c = make_float2(csx, csy);
    maxabs = fmaxf(maxabs, fmaxf(fabsf(x.x), fabsf(x.y)));
}
// Exact pair (Payne-Hanek for |x| > 2^17), out of line: returns (sin x, sin y, cos x, cos y).
static __device__ __noinline__ float4 sincos2_exact(float2 x) {
    float xs[2] = {x.x, x.y}, ss[2], cc[2];
    tpl_sincos_n<2>(xs, ss, cc);
    return make_float4(ss[0], ss[1], cc[0], cc[1]);
}
__device__ __forceinline__ void sincos2_slow(float2 x, float2& s, float2& c) {
    const float4 r = sincos2_exact(x);
    s = make_float2(r.x, r.y);
    c = make_float2(r.z, r.w);
}

// Pass 1 of the packed forward: runs A (.x lanes, residues [j0, j0+R))
// and B (.y lanes, [j0+R, j0+2R)) composed from the identity, the translation
// (atom position) after every bond kept.  Angles past Lmax read as 0 (they only
// move later residues, which are never stored); chain_start: run A begins at
// residue 0, whose omega bond is the identity (reading Q1).  A warp holding an
// |angle| > 2^17 evaluates all its sincos with the exact reduction.
template <int R>
__device__ __forceinline__ void bbp_pass1(const float* s_ang, int Lmax, int j0, bool chain_start,
                                          float2 (&px)[3 * R], float2 (&py)[3 * R], float2 (&pz)[3 * R], Aff2& M,
                                          bool has_pre = false) {
    // has_pre: s_ang[-1] holds omega of the residue before (a later tile of a chain)
    float maxabs = 0.f;
    auto angle = [&](int j, int k) -> float {  // omega_{j-1} (k=0), phi_j (1), psi_j (2); 0 past Lmax
        const int idx = 3 * j + k - 1;
        return (j < Lmax && (idx >= 0 || has_pre)) ? s_ang[idx] : 0.f;
    };
    auto pass1 = [&](auto slow) {
        constexpr bool kSlow = decltype(slow)::value;
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const int ja = j0 + q, jb = j0 + R + q;
            float2 c[3], s[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const float2 x = make_float2(angle(ja, k), angle(jb, k));
                if (kSlow) sincos2_slow(x, s[k], c[k]);
                else sincos2_fast(x, s[k], c[k], maxabs);
            }
            if (q == 0) {
                aff2_from_bond<0>(M, c[0], s[0]);
                if (chain_start) set_lane_x(M, aff_identity());  // R_0 = I (reading Q1)
            } else {
                aff2_bond<0>(M, c[0], s[0]);
            }
            px[3 * q] = M.t0; py[3 * q] = M.t1; pz[3 * q] = M.t2;
            aff2_bond<1>(M, c[1], s[1]);
            px[3 * q + 1] = M.t0; py[3 * q + 1] = M.t1; pz[3 * q + 1] = M.t2;
            aff2_bond<2>(M, c[2], s[2]);
            px[3 * q + 2] = M.t0; py[3 * q + 2] = M.t1; pz[3 * q + 2] = M.t2;
        }
    };
    if (__all_sync(0xffffffffu, j0 >= Lmax)) {  // the warp's residues are all past the chain (ragged batches)
        M.r00 = M.r11 = M.r22 = f2(1.f);
        M.r01 = M.r02 = M.r10 = M.r12 = M.r20 = M.r21 = f2(0.f);
        M.t0 = M.t1 = M.t2 = f2(0.f);
        return;
    }
    pass1(std::false_type{});
    if (__any_sync(0xffffffffu, maxabs > kSinCosFastMax)) pass1(std::true_type{});  // rare: huge angles
}

// ---------------------------------------------------------------------------
// Rigid transforms as (unit quaternion, translation): 7 floats.  The block scan of
// the packed forward composes thread aggregates in this form and renormalises the
// quaternion after every combine, so every rotation that carries a long
// translation is orthonormal to fp32 precision (a 3x4 scan re-orthonormalises only
// its results: a warp total that is off-orthogonal by 1e-6 moves a 2800 A
// translation by 3e-3 A -- extended chains of 769-1024 residues missed the 1e-3 A
// gate that way).  Fewer shuffles too: 7 floats per KS level instead of 12.
struct QT {
    float w, x, y, z;  // rotation q = w + x i + y j + z k, |q| = 1
    float tx, ty, tz;  // translation
};

__device__ __forceinline__ QT qt_identity() { return QT{1.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}; }

// |q| is within ~1e-6 of 1 here (products of unit quaternions, or Shepperd's
// conversion): one Newton step q (3 - |q|^2) / 2 renormalises to O(eps^2) without
// a MUFU rsqrt in the scan's dependency chain.
__device__ __forceinline__ void qt_normalize(QT& a) {
    const float n2 = fmaf(a.w, a.w, fmaf(a.x, a.x, fmaf(a.y, a.y, a.z * a.z)));
    const float r = fmaf(-0.5f, n2, 1.5f);
    a.w *= r; a.x *= r; a.y *= r; a.z *= r;
}

// A then B in A's frame (the affine product A B): (qA qB, tA + R(qA) tB), renormalised.
__device__ __forceinline__ QT qt_compose(const QT& A, const QT& B) {
    QT C;
    C.w = fmaf(A.w, B.w, -fmaf(A.x, B.x, fmaf(A.y, B.y, A.z * B.z)));
    C.x = fmaf(A.w, B.x, fmaf(A.x, B.w, fmaf(A.y, B.z, -A.z * B.y)));
    C.y = fmaf(A.w, B.y, fmaf(-A.x, B.z, fmaf(A.y, B.w, A.z * B.x)));
    C.z = fmaf(A.w, B.z, fmaf(A.x, B.y, fmaf(-A.y, B.x, A.z * B.w)));
    // R(qA) tB = v + w c + u x c with c = 2 u x v
    const float cx = 2.f * fmaf(A.y, B.tz, -A.z * B.ty);
    const float cy = 2.f * fmaf(A.z, B.tx, -A.x * B.tz);
    const float cz = 2.f * fmaf(A.x, B.ty, -A.y * B.tx);
    C.tx = A.tx + fmaf(A.w, cx, fmaf(A.y, cz, fmaf(-A.z, cy, B.tx)));
    C.ty = A.ty + fmaf(A.w, cy, fmaf(A.z, cx, fmaf(-A.x, cz, B.ty)));
    C.tz = A.tz + fmaf(A.w, cz, fmaf(A.x, cy, fmaf(-A.y, cx, B.tz)));
    qt_normalize(C);
    return C;
}

// 3x4 affine with an orthonormal rotation -> QT (Shepperd: the largest of the four
// quaternion-component candidates sets the divisor; branch-free selects).
__device__ __forceinline__ QT qt_from_aff(const Aff& m) {
    const float tr = m.r00 + m.r11 + m.r22;
    const float v0 = 1.f + tr, v1 = 1.f + m.r00 - m.r11 - m.r22, v2 = 1.f - m.r00 + m.r11 - m.r22,
                v3 = 1.f - m.r00 - m.r11 + m.r22;
    const float d21 = m.r21 - m.r12, d02 = m.r02 - m.r20, d10 = m.r10 - m.r01;
    const float s01 = m.r01 + m.r10, s02 = m.r02 + m.r20, s12 = m.r12 + m.r21;
    QT q;
    const int k = (v0 >= v1 && v0 >= v2 && v0 >= v3) ? 0 : (v1 >= v2 && v1 >= v3) ? 1 : (v2 >= v3) ? 2 : 3;
    const float v = k == 0 ? v0 : k == 1 ? v1 : k == 2 ? v2 : v3;
    const float h = 0.5f * rsqrtf(v);  // 1 / (4 * component)
    const float big = v * h;           // 0.5 sqrt(v) = the large component
    if (k == 0) { q.w = big; q.x = d21 * h; q.y = d02 * h; q.z = d10 * h; }
    else if (k == 1) { q.w = d21 * h; q.x = big; q.y = s01 * h; q.z = s02 * h; }
    else if (k == 2) { q.w = d02 * h; q.x = s01 * h; q.y = big; q.z = s12 * h; }
    else { q.w = d10 * h; q.x = s02 * h; q.y = s12 * h; q.z = big; }
    qt_normalize(q);
    q.tx = m.t0; q.ty = m.t1; q.tz = m.t2;
    return q;
}

__device__ __forceinline__ Aff aff_from_qt(const QT& q) {
    const float x2 = q.x + q.x, y2 = q.y + q.y, z2 = q.z + q.z;
    const float xx = q.x * x2, yy = q.y * y2, zz = q.z * z2, xy = q.x * y2, xz = q.x * z2, yz = q.y * z2;
    const float wx = q.w * x2, wy = q.w * y2, wz = q.w * z2;
    Aff a;
    a.r00 = 1.f - (yy + zz); a.r01 = xy - wz; a.r02 = xz + wy; a.t0 = q.tx;
    a.r10 = xy + wz; a.r11 = 1.f - (xx + zz); a.r12 = yz - wx; a.t1 = q.ty;
    a.r20 = xz - wy; a.r21 = yz + wx; a.r22 = 1.f - (xx + yy); a.t2 = q.tz;
    return a;
}

__device__ __forceinline__ QT shfl_up_qt(const QT& a, int d) {
    const unsigned m = 0xffffffffu;
    return QT{__shfl_up_sync(m, a.w, d), __shfl_up_sync(m, a.x, d), __shfl_up_sync(m, a.y, d),
              __shfl_up_sync(m, a.z, d), __shfl_up_sync(m, a.tx, d), __shfl_up_sync(m, a.ty, d),
              __shfl_up_sync(m, a.tz, d)};
}
__device__ __forceinline__ void store_qt(float* s, const QT& a) {
    s[0] = a.w; s[1] = a.x; s[2] = a.y; s[3] = a.z; s[4] = a.tx; s[5] = a.ty; s[6] = a.tz;
}
__device__ __forceinline__ QT load_qt(const float* s) { return QT{s[0], s[1], s[2], s[3], s[4], s[5], s[6]}; }

// Block-wide EXCLUSIVE scan of the thread aggregates in (quaternion, translation)
// form (one tile, carry = identity); returns the thread's prefix as a 3x4 affine.
// scratch: NW * 8 floats.  Aggregates must be orthonormal (policy >= 1).
template <int NT>
__device__ __forceinline__ Aff block_exclusive_scan_qt(const Aff& agg, float* scratch) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    QT a = qt_from_aff(agg);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const QT o = shfl_up_qt(a, d);
        if (lane >= d) a = qt_compose(o, a);
    }
    if (lane == 31) store_qt(scratch + 8 * warp, a);
    QT ex = shfl_up_qt(a, 1);
    if (lane == 0) ex = qt_identity();
    __syncthreads();
    QT p = load_qt(scratch);  // the warp totals before this warp (warp 0 uses none)
#pragma unroll
    for (int w = 1; w < NW - 1; ++w)
        if (w < warp) p = qt_compose(p, load_qt(scratch + 8 * w));
    const QT res = warp > 0 ? qt_compose(p, ex) : ex;
    // no trailing barrier: the single-tile callers never reuse the scratch
    return aff_from_qt(res);
}

// As block_exclusive_scan_qt with a carry: returns carry (x) the thread's exclusive
// prefix and replaces carry by carry (x) the block's total (the next tile's carry).
// scratch: NW * 8 + 8 floats ((2 NW + 1) * 8 for NW > 4).
template <int NT>
__device__ __forceinline__ Aff block_exclusive_scan_qt_carry(const Aff& agg, float* scratch, QT& carry) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    QT a = qt_from_aff(agg);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const QT o = shfl_up_qt(a, d);
        if (lane >= d) a = qt_compose(o, a);
    }
    if (lane == 31) store_qt(scratch + 8 * warp, a);
    QT ex = shfl_up_qt(a, 1);
    if (lane == 0) ex = qt_identity();
    __syncthreads();
    QT p = carry;
    if (NW > 4) {
        // wide blocks: warp 0 scans the NW warp totals in log2(NW) steps (a serial chain of
        // NW - 1 combines cost the 512-thread full-atom forward 9%) and parks each warp's
        // prefix, carry included, at scratch[8 (NW + 1 + w)]; scratch: (2 NW + 1) 8 floats
        if (warp == 0) {
            QT t = lane < NW ? load_qt(scratch + 8 * lane) : qt_identity();
#pragma unroll
            for (int d = 1; d < NW; d <<= 1) {
                const QT o = shfl_up_qt(t, d);
                if (lane >= d) t = qt_compose(o, t);
            }
            QT e = shfl_up_qt(t, 1);
            if (lane == 0) e = qt_identity();
            if (lane < NW) store_qt(scratch + 8 * (NW + 1 + lane), qt_compose(carry, e));
        }
        __syncthreads();
        p = load_qt(scratch + 8 * (NW + 1 + warp));
    } else {
#pragma unroll
        for (int w = 0; w < NW - 1; ++w)
            if (w < warp) p = qt_compose(p, load_qt(scratch + 8 * w));
    }
    const QT res = qt_compose(p, ex);
    if (threadIdx.x == NT - 1) store_qt(scratch + 8 * NW, qt_compose(p, a));
    __syncthreads();
    carry = load_qt(scratch + 8 * NW);
    __syncthreads();  // scratch is free again
    return aff_from_qt(res);
}

// Block-wide EXCLUSIVE suffix sum of N floats per thread (sum over threads > t)
// and the block total, NT = 32 NW threads; scratch: 2 NW N + N floats.  The
// association order is fixed (deterministic).
template <int NT, int N>
__device__ __forceinline__ void block_exclusive_suffix_n(const float (&v)[N], float* scratch, float (&out)[N],
                                                         float (&total)[N]) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float inc[N];
#pragma unroll
    for (int k = 0; k < N; ++k) inc[k] = v[k];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
        for (int k = 0; k < N; ++k) {
            const float o = __shfl_down_sync(0xffffffffu, inc[k], d);
            if (lane + d < 32) inc[k] += o;
        }
    }
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < N; ++k) scratch[N * warp + k] = inc[k];
    }
    float ex[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        const float o = __shfl_down_sync(0xffffffffu, inc[k], 1);
        ex[k] = lane == 31 ? 0.f : o;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < N; ++k) {
        float later = 0.f, all = 0.f;
#pragma unroll
        for (int w = NW - 1; w >= 0; --w) {
            const float t = scratch[N * w + k];
            if (w > warp) later += t;
            all += t;
        }
        out[k] = later + ex[k];
        total[k] = all;
    }
    __syncthreads();
}

// Launch shape of the packed kernels for chains of up to Lmax residues: NT threads
// x 2R residues per thread.  Runs of R = 3 residues from 513 residues on (a 3-residue
// run of a periodic chain need not be a pure translation, so per-run rounding does
// not add up coherently along an extended chain the way it does for R = 4: extended
// L = 1000 had 1.2e-2 A with 128 x 4, tools/regular_sweep.py).
struct BBPShape {
    int nt, r;
};
constexpr int kBBPMaxL = 2 * 3 * 192;
inline BBPShape bbp_shape(int Lmax) {
    if (Lmax <= 256) return {128, 1};
    if (Lmax <= 512) return {128, 2};
    if (Lmax <= 768) return {128, 3};
    return {192, 3};
}

// N consecutive floats between registers and shared memory, as 8-byte accesses
// where the address allows (a thread's runs sit 216 R bytes apart: 64-bit accesses
// of a half-warp then hit distinct bank pairs).
template <int N>
__device__ __forceinline__ void sts_run(float* p, const float (&v)[N]) {
    if ((reinterpret_cast<uintptr_t>(p) & 7) == 0) {
#pragma unroll
        for (int i = 0; i + 1 < N; i += 2) *reinterpret_cast<float2*>(p + i) = make_float2(v[i], v[i + 1]);
        if (N & 1) p[N - 1] = v[N - 1];
    } else {
        p[0] = v[0];
#pragma unroll
        for (int i = 1; i + 1 < N; i += 2) *reinterpret_cast<float2*>(p + i) = make_float2(v[i], v[i + 1]);
        if (!(N & 1)) p[N - 1] = v[N - 1];
    }
}
template <int N>
__device__ __forceinline__ void lds_run(const float* p, float (&v)[N]) {
    if ((reinterpret_cast<uintptr_t>(p) & 7) == 0) {
#pragma unroll
        for (int i = 0; i + 1 < N; i += 2) {
            const float2 t = *reinterpret_cast<const float2*>(p + i);
            v[i] = t.x;
            v[i + 1] = t.y;
        }
        if (N & 1) v[N - 1] = p[N - 1];
    } else {
        v[0] = p[0];
#pragma unroll
        for (int i = 1; i + 1 < N; i += 2) {
            const float2 t = *reinterpret_cast<const float2*>(p + i);
            v[i] = t.x;
            v[i + 1] = t.y;
        }
        if (!(N & 1)) v[N - 1] = p[N - 1];
    }
}

// Head/tail bytes of a span with plain loads by the 32 lanes of one warp.
__device__ __forceinline__ void span_load_edges_warp(const Span& s, char* sbase, int lane) {
    float* d = reinterpret_cast<float*>(sbase + s.mis());
    const float* g = reinterpret_cast<const float*>(s.g);
    const int nh = s.head >> 2, nt = s.tail() >> 2, off_t = (s.head + s.mid) >> 2;
    for (int k = lane; k < nh + nt; k += 32) {
        const int idx = k < nh ? k : off_t + (k - nh);
        d[idx] = __ldg(g + idx);
    }
}

// A warp's staged output chunk to global memory: 16-byte vector stores for the aligned
// middle (each warp instruction writes 512 contiguous bytes), plain stores for the
// <16-byte head and tail.  Shared and global addresses share their 16-byte phase.
// (Measured against one cp.async.bulk store per warp: the CTA then has to wait for the
// TMA engine to read the staging before it may exit -- 13% of the forward's warp
// samples sat in that wait.)
__device__ __forceinline__ void store_warp_chunk(float* gdst, const float* ssrc, int bytes, int lane) {
    const Span sw = make_span(gdst, bytes);
    const char* src = reinterpret_cast<const char*>(ssrc);
    char* dst = const_cast<char*>(sw.g);
    for (int i = lane; i < (sw.mid >> 4); i += 32) {
        const float4 v = *reinterpret_cast<const float4*>(src + sw.head + 16 * i);
        *reinterpret_cast<float4*>(dst + sw.head + 16 * i) = v;
    }
    const int nh = sw.head >> 2, ntl = sw.tail() >> 2, off_t = (sw.head + sw.mid) >> 2;
    for (int e = lane; e < nh + ntl; e += 32) {
        const int idx = e < nh ? e : off_t + (e - nh);
        reinterpret_cast<float*>(dst)[idx] = ssrc[idx];
    }
}

// TPL_BBP_MINSMEM=<bytes>: pad the packed kernels' shared memory (tuning: caps the
// CTAs per SM, e.g. to keep early-launched dependents from piling onto idle SMs)
inline size_t bbp_min_smem() {
    static long v = -1;
    if (v < 0) {
        const char* e = std::getenv("TPL_BBP_MINSMEM");
        v = e ? std::atol(e) : 0;
    }
    return size_t(v);
}

// Launch policy of the packed kernels.  With at most 2 chains per SM the step is
// latency-bound and every kernel boundary costs ~0.8 us between the last CTA of one
// kernel and the first of the next (tools/step_gaps.py).  These kernels are then
// launched with programmatic stream serialization (each CTA waits on
// griddepcontrol.wait before its first global access and triggers the next grid
// at once), so consecutive tpl kernels overlap launch with the previous tail; and
// their shared memory is padded so that at most ceil(B / SMs) CTAs of either
// kernel fit on an SM -- otherwise the early-launched dependents pile onto the SMs
// that finish first (measured: 256 x 700 step 12.4 us without PDL, 13.3 us with
// PDL unpadded, 11.3 us with PDL padded to 2 CTAs/SM).  TPL_BBP_PDL=0 disables.
struct BBPLaunch {
    size_t smem;
    bool pdl;
};
inline BBPLaunch bbp_policy(int B, size_t smem) {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("TPL_BBP_PDL");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    BBPLaunch l{std::max(smem, bbp_min_smem()), false};
    const int sms = device_sm_count();
    if (v == 1 && B <= 2 * sms) {
        const int per_sm = (B + sms - 1) / sms;                         // 1 or 2
        const size_t cap = per_sm == 1 ? 118 * 1024 : 80 * 1024;        // > 228 KB / (per_sm + 1)
        l.smem = std::max(l.smem, cap);
        l.pdl = true;
    }
    return l;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_bbp(void (*kernel)(KArgs...), int grid, int block, const BBPLaunch& l, cudaStream_t st,
                              Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = l.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = l.pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace tpl
