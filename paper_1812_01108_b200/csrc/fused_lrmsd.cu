// fused_lrmsd.cu -- SURVEY §8(f) f1 in one pass: dihedral angles -> backbone
// coordinates (PAPER §3) -> LRMSD to a target (PAPER §4)
// -> dLRMSD/dalpha (Eq. 2, through dLRMSD/dx of P:233-236 with the
// normalisation of reading Q19), one CTA per chain, with no coordinate
// round-trip through HBM: angles (12 B/res) and the target (36 B/res) in,
// dLRMSD/dalpha (12 B/res) out, coordinates (36 B/res) only when asked for.
//
// Per chain (the packed layout of packed.cu: thread t owns residues
// [2Rt, 2Rt + 2R), run A in the .x lanes, run B in the .y lanes):
//   1. forward: pass 1, block scan in (quaternion, translation) form, pass 2 ->
//      atom positions x in registers (and staged in shared memory for the
//      neighbours' axes);
//   2. step 1 of §4: barycentres of x and y (x_0 = 0 by reading Q1, y about its
//      first atom), then the centred correlation R -- fp32 per thread (18 atoms),
//      fp64 across threads (warp sums by recursive halving, then across warps);
//   3. steps 2-3 (lrmsd_math.cuh, warp 0): T, its largest eigenpair (the root
//      bracketed across the lanes), U; the value is the residuals' sum of squares;
//   4. backward: g_i = (x~_i - U^T y~_i) / (N LRMSD) formed on the fly,
//      S = sum_{later} g, T = sum_{later} x x g, one block suffix sum, and
//      dLRMSD/dalpha_a = e_a . (T_a - x_a x S_a) per atom (as packed.cu).
// The autograd backward scales the saved dLRMSD/dalpha by dL/dLRMSD
// (tpl_chain_scale).
#include <cstdio>

#include "common.cuh"
#include "kernels.h"
#include "lrmsd_math.cuh"
#include "packed.cuh"

namespace tpl {

// Warp sum of S (a power of two, 8 or 16) doubles per lane by recursive halving: at
// each level a lane sends the half of its slots its partner keeps and adds the half it
// receives (S - 1 + 1 double shuffles instead of 5 S for a tree per value).  Returns the
// warp total of slot lane / (32 / S) (every 32 / S consecutive lanes hold the same slot).
template <int S>
__device__ __forceinline__ double warp_sum_halving(double (&v)[S]) {
    static_assert(S == 8 || S == 16, "8 or 16 slots");
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int off = 16, h = S / 2; h >= 1; off >>= 1, h >>= 1) {
        const bool up = (lane & off) != 0;  // keeps the upper half of its slots
#pragma unroll
        for (int k = 0; k < h; ++k) {
            const double send = up ? v[k] : v[k + h];
            const double keep = up ? v[k + h] : v[k];
            v[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
    // S slots over 32 lanes: the remaining 32 / S lanes per slot still hold partial sums
#pragma unroll
    for (int off = 16 / S; off >= 1; off >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
    return v[0];
}

template <int NT, int R, int kNS>
__global__ void __launch_bounds__(NT, NT > 128 ? 1 : 2) bbp_lrmsd_kernel(const float* __restrict__ angles,
                                                                       const int* __restrict__ lengths, int B,
                                                                       int Lmax, const float* __restrict__ target,
                                                                       float* __restrict__ coords,
                                                                       float* __restrict__ loss_out,
                                                                       float* __restrict__ state_out,
                                                                       float* __restrict__ grad_angles,
                                                                       unsigned* __restrict__ err) {
    constexpr int TILE = 2 * R * NT;
    constexpr int NW = NT / 32;
    constexpr int WRES = 64 * R;
    constexpr int XB = (16 + 36 * TILE + 16 + 15) & ~15;
    extern __shared__ __align__(16) char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);                  // [0] angles, [1 + w] target pieces
    double* s_red = reinterpret_cast<double*>(smem + 8 * (NW + 1) + 8);  // 6 NW barycentre + 9 NW R sums (+ pad)
    float* s_sol = reinterpret_cast<float*>(s_red + NW * 17 + 1);       // 16 state + value
    float* scratch = s_sol + 32;                                         // 2 NW 12 + 12 (affine scan)
    float* s_total = scratch + 2 * NW * 12;
    float* s_suf = s_total + 12;                                         // 2 NW 7 + 16 (suffix sums)
    char* s_ang_base = smem + ((reinterpret_cast<char*>(s_suf + 2 * NW * 7 + 16) - smem + 15) & ~15);
    char* s_y_base = s_ang_base + ((16 + 12 * TILE + 16 + 15) & ~15);
    char* s_x_base = s_y_base + XB;
    char* s_go_base = s_x_base + XB;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b = blockIdx.x;
    TPL_STAMP(0);
    const size_t cbase = (size_t)b * 3 * Lmax * 3;
    const Span sa = make_span(angles + (size_t)b * Lmax * 3, Lmax * 12);
    const int w0 = warp * WRES;
    const Span syw = make_span(target + cbase + 9 * (size_t)w0, max(0, min(WRES, Lmax - w0)) * 36);
    if (prefetch_regime(B)) {
        if (tid == 0 && sa.mid > 0) prefetch_l2(sa.g + sa.head, unsigned(sa.mid));
        if (lane == 0 && syw.mid > 0) prefetch_l2(syw.g + syw.head, unsigned(syw.mid));
    }
    pdl_wait();
    pdl_trigger();
    if (tid == 0) {
        mbar_init(bar, 1);
        fence_barrier_init();
        mbar_arrive_expect_tx(bar, unsigned(sa.mid));
        span_load_bulk(sa, s_ang_base, bar);
    }
    if (lane == 0) {  // each warp's own target piece
        mbar_init(bar + 1 + warp, 1);
        fence_barrier_init();
        mbar_arrive_expect_tx(bar + 1 + warp, unsigned(syw.mid));
        span_load_bulk(syw, s_y_base + 36 * w0, bar + 1 + warp);
    }
    const int L = __ldg(lengths + b);
    const float y0x = __ldg(target + cbase), y0y = __ldg(target + cbase + 1), y0z = __ldg(target + cbase + 2);
    span_load_edges_f32(sa, s_ang_base);
    span_load_edges_warp(syw, s_y_base + 36 * w0, lane);
    __syncthreads();  // barriers initialised, edges in place
    mbar_wait(bar, 0);
    const float* s_ang = reinterpret_cast<const float*>(s_ang_base + sa.mis());
    const bool ok = L >= 1 && L <= Lmax;
    const int Lv = ok ? L : 0;
    TPL_STAMP(1);

    // ---- 1. forward: positions of runs A / B
    const int j0 = 2 * R * tid;
    float2 X[3 * R], Y[3 * R], Z[3 * R];
    {
        Aff2 M;
        bbp_pass1<R>(s_ang, Lmax, j0, tid == 0, X, Y, Z, M);
        const Aff A = lane_x(M);
        Aff agg = aff_compose(A, lane_y(M));
        if (kNS >= 2) aff_orthonormalize(agg);  // policy 1: the quaternion extraction renormalises
        const Aff P = kNS == 1 ? block_exclusive_scan_qt<NT>(agg, scratch)
                               : block_exclusive_scan<NT, kNS>(agg, aff_identity(), scratch, s_total);
        const Aff2 P2 = pack2(P, aff_compose(P, A));
#pragma unroll
        for (int a = 0; a < 3 * R; ++a) apply2(P2, X[a], Y[a], Z[a], X[a], Y[a], Z[a]);
    }
    // atoms past the chain: 0 (pads may hold anything; they must not reach the sums)
#pragma unroll
    for (int a = 0; a < 3 * R; ++a) {
        if (j0 + a / 3 >= Lv) { X[a].x = 0.f; Y[a].x = 0.f; Z[a].x = 0.f; }
        if (j0 + R + a / 3 >= Lv) { X[a].y = 0.f; Y[a].y = 0.f; Z[a].y = 0.f; }
    }
    // stage x (the axes of the neighbours' first atoms; the optional coordinate output)
    const int xmis = coords ? int(reinterpret_cast<uintptr_t>(coords + cbase) & 15) : 0;
    float* s_x = reinterpret_cast<float*>(s_x_base + xmis);
    {
        float fa[9 * R], fb[9 * R];
#pragma unroll
        for (int a = 0; a < 3 * R; ++a) {
            fa[3 * a] = X[a].x; fa[3 * a + 1] = Y[a].x; fa[3 * a + 2] = Z[a].x;
            fb[3 * a] = X[a].y; fb[3 * a + 1] = Y[a].y; fb[3 * a + 2] = Z[a].y;
        }
        sts_run<9 * R>(s_x + 9 * j0, fa);
        sts_run<9 * R>(s_x + 9 * j0 + 9 * R, fb);
    }
    __syncwarp();
    if (coords && ok) {
        const int wn = min(WRES, L - w0);
        if (wn > 0) store_warp_chunk(coords + cbase + 9 * (size_t)w0, s_x + 9 * w0, wn * 36, lane);
    }
    TPL_STAMP(2);

    // ---- 2. moments of (x, y - y0) over the valid atoms (x_0 = 0: no shift for x)
    mbar_wait(bar + 1 + warp, 0);
    TPL_STAMP(7);
    float* s_y = reinterpret_cast<float*>(s_y_base + int(reinterpret_cast<uintptr_t>(target + cbase) & 15));
    {
        const int f0 = 9 * max(Lv, w0), f1 = 9 * (w0 + WRES);  // target atoms past the chain: 0
        for (int f = f0 + lane; f < f1; f += 32) s_y[f] = 0.f;
    }
    __syncwarp();
    // target atom i of runs A (.x) and B (.y)
    auto load_y = [&](int i, float2& u, float2& w, float2& t) {
        const float* pa = s_y + 9 * j0 + 3 * i;
        const float* pb = pa + 9 * R;
        u = make_float2(pa[0], pb[0]);
        w = make_float2(pa[1], pb[1]);
        t = make_float2(pa[2], pb[2]);
    };
    // validity of the runs' atoms: run A residues j0.., run B j0 + R..
    auto valid2 = [&](int q) { return make_float2(j0 + q < Lv ? 1.f : 0.f, j0 + R + q < Lv ? 1.f : 0.f); };
    const double n = 3.0 * (Lv > 0 ? Lv : 1);
    // ---- 2a. barycentres of x and of y - y0 (fp32 per thread and warp, fp64 across warps)
    float cx, cy, cz, dcx, dcy, dcz;     // barycentres (x; y about y0), rounded to fp32
    float lx, ly, lz, ky, kyy, kz;       // their rounding remainders, and y's absolute barycentre's
    {
        float2 m[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) m[k] = f2(0.f);
#pragma unroll
        for (int i = 0; i < 3 * R; ++i) {
            const float2 v = valid2(i / 3);
            float2 u, w, t;
            load_y(i, u, w, t);
            m[0] = __fadd2_rn(m[0], X[i]); m[1] = __fadd2_rn(m[1], Y[i]); m[2] = __fadd2_rn(m[2], Z[i]);
            m[3] = __ffma2_rn(__fadd2_rn(u, f2(-y0x)), v, m[3]);
            m[4] = __ffma2_rn(__fadd2_rn(w, f2(-y0y)), v, m[4]);
            m[5] = __ffma2_rn(__fadd2_rn(t, f2(-y0z)), v, m[5]);
        }
        // fp64 from the thread partials on: an fp32 warp sum leaves the barycentre ~3e-6 A
        // off, a shift every residual carries coherently into the suffix sums (1e-2 of the
        // gradient near a perfect superposition)
        double c[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) c[k] = k < 6 ? double(m[k].x) + double(m[k].y) : 0.0;
        const double tot = warp_sum_halving<8>(c);  // slot lane / 4
        if ((lane & 3) == 0 && (lane >> 2) < 6) s_red[6 * warp + (lane >> 2)] = tot;
        TPL_STAMP(8);
        __syncthreads();
        TPL_STAMP(9);
        double cs[6];
        const double inv_n = rcp_full(n);
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            double v = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) v += s_red[6 * w + k];
            cs[k] = v * inv_n;
        }
        cx = float(cs[0]); cy = float(cs[1]); cz = float(cs[2]);
        lx = float(cs[0] - double(cx)); ly = float(cs[1] - double(cy)); lz = float(cs[2] - double(cz));
        // y's barycentre y0 + cs[3..5] as a float pair (hi, lo): centring with both halves
        // leaves no coherent rounding bias in the residuals (a 2e-6 A bias summed over
        // 2100 atoms is 2e-3 of the suffix sums near a perfect superposition)
        const double ay0 = double(y0x) + cs[3], ay1 = double(y0y) + cs[4], ay2 = double(y0z) + cs[5];
        dcx = float(ay0); dcy = float(ay1); dcz = float(ay2);
        ky = float(ay0 - double(dcx)); kyy = float(ay1 - double(dcy)); kz = float(ay2 - double(dcz));
    }
    // x~ and y~ (centred) of atom i of both runs, 0 past the chain
    auto centred = [&](int i, float2& ax, float2& ay, float2& az, float2& bx, float2& by, float2& bz) {
        const float2 v = valid2(i / 3);
        float2 u, w, t;
        load_y(i, u, w, t);
        ax = __fmul2_rn(__fadd2_rn(__fadd2_rn(X[i], f2(-cx)), f2(-lx)), v);
        ay = __fmul2_rn(__fadd2_rn(__fadd2_rn(Y[i], f2(-cy)), f2(-ly)), v);
        az = __fmul2_rn(__fadd2_rn(__fadd2_rn(Z[i], f2(-cz)), f2(-lz)), v);
        bx = __fmul2_rn(__fadd2_rn(__fadd2_rn(u, f2(-dcx)), f2(-ky)), v);
        by = __fmul2_rn(__fadd2_rn(__fadd2_rn(w, f2(-dcy)), f2(-kyy)), v);
        bz = __fmul2_rn(__fadd2_rn(__fadd2_rn(t, f2(-dcz)), f2(-kz)), v);
    };
    // ---- 2b. centred correlation R = sum x~ y~^T (step 1 of §4)
    {
        float2 m[9];
#pragma unroll
        for (int k = 0; k < 9; ++k) m[k] = f2(0.f);
#pragma unroll
        for (int i = 0; i < 3 * R; ++i) {
            float2 ax, ay, az, bx, by, bz;
            centred(i, ax, ay, az, bx, by, bz);
            m[0] = __ffma2_rn(ax, bx, m[0]); m[1] = __ffma2_rn(ax, by, m[1]); m[2] = __ffma2_rn(ax, bz, m[2]);
            m[3] = __ffma2_rn(ay, bx, m[3]); m[4] = __ffma2_rn(ay, by, m[4]); m[5] = __ffma2_rn(ay, bz, m[5]);
            m[6] = __ffma2_rn(az, bx, m[6]); m[7] = __ffma2_rn(az, by, m[7]); m[8] = __ffma2_rn(az, bz, m[8]);
        }
        // fp64 from the thread partials on: R's rounding sets U's, and near a perfect
        // superposition the gradient's residuals x~ - U^T y~ are tiny (fp32 warp sums
        // cost 4e-3 of gradient accuracy at a 0.05 A jitter)
        double c[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) c[k] = k < 9 ? double(m[k].x) + double(m[k].y) : 0.0;
        const double tot = warp_sum_halving<16>(c);  // slot lane / 2
        TPL_STAMP(10);
        // after the barycentre sums (s_red[0, 6 NW)): no barrier between
        if ((lane & 1) == 0 && (lane >> 1) < 9) s_red[6 * NW + 9 * warp + (lane >> 1)] = tot;
    }
    __syncthreads();
    TPL_STAMP(3);
    // ---- 3. steps 2-3 of §4 on warp 0 (fp64): T, its largest eigenpair (the root
    //      bracketed across the lanes), U.  The moments are centred, so the barycentres
    //      handed to the solver are 0.
    if (warp == 0) {
        double Rm[3][3];
        for (int k = 0; k < 9; ++k) {
            double v = 0.0;
            for (int w = 0; w < NW; ++w) v += s_red[6 * NW + 9 * w + k];
            Rm[k / 3][k % 3] = v;
        }
        lrmsd_rotation_warp(Rm, s_sol);  // U in s_sol[0..8]
    }
    __syncthreads();
    TPL_STAMP(4);
    float U[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) U[k] = s_sol[k];
    // r = x~ - U^T y~ of atom i of both runs (0 past the chain): dLRMSD/dx = r / (N LRMSD)
    auto resid = [&](int i, float2& gx, float2& gy, float2& gz) {
        float2 ax, ay, az, bx, by, bz;
        centred(i, ax, ay, az, bx, by, bz);
        gx = __ffma2_rn(f2(-U[0]), bx, __ffma2_rn(f2(-U[3]), by, __ffma2_rn(f2(-U[6]), bz, ax)));
        gy = __ffma2_rn(f2(-U[1]), bx, __ffma2_rn(f2(-U[4]), by, __ffma2_rn(f2(-U[7]), bz, ay)));
        gz = __ffma2_rn(f2(-U[2]), bx, __ffma2_rn(f2(-U[5]), by, __ffma2_rn(f2(-U[8]), bz, az)));
    };

    // ---- 4. backward pass 1: (S, T) of the residuals about the origin (= atom 0), and
    //      E = sum |r|^2, the LRMSD's numerator as a sum of squares (no cancellation)
    float2 S0 = f2(0.f), S1 = f2(0.f), S2 = f2(0.f), T0 = f2(0.f), T1 = f2(0.f), T2 = f2(0.f), E2 = f2(0.f);
#pragma unroll
    for (int i = 0; i < 3 * R; ++i) {
        float2 gx, gy, gz;
        resid(i, gx, gy, gz);
        const float2 px = X[i], py = Y[i], pz = Z[i];
        E2 = __ffma2_rn(gx, gx, __ffma2_rn(gy, gy, __ffma2_rn(gz, gz, E2)));
        S0 = __fadd2_rn(S0, gx); S1 = __fadd2_rn(S1, gy); S2 = __fadd2_rn(S2, gz);
        T0 = __fadd2_rn(T0, __ffma2_rn(py, gz, __fmul2_rn(make_float2(-pz.x, -pz.y), gy)));
        T1 = __fadd2_rn(T1, __ffma2_rn(pz, gx, __fmul2_rn(make_float2(-px.x, -px.y), gz)));
        T2 = __fadd2_rn(T2, __ffma2_rn(px, gy, __fmul2_rn(make_float2(-py.x, -py.y), gx)));
    }
    float v7[7] = {S0.x + S0.y, S1.x + S1.y, S2.x + S2.y, T0.x + T0.y, T1.x + T1.y, T2.x + T2.y, E2.x + E2.y};
    float ext[7], tot7[7];
    block_exclusive_suffix_n<NT, 7>(v7, s_suf, ext, tot7);
    S0 = make_float2(ext[0] + S0.y, ext[0]); S1 = make_float2(ext[1] + S1.y, ext[1]);
    S2 = make_float2(ext[2] + S2.y, ext[2]); T0 = make_float2(ext[3] + T0.y, ext[3]);
    T1 = make_float2(ext[4] + T1.y, ext[4]); T2 = make_float2(ext[5] + T2.y, ext[5]);
    // the value from the fp32 sum of squares in fp32 (correctly rounded division and sqrt)
    const float nf = float(n);
    const float lr = sqrtf(fmaxf(tot7[6], 0.f) / nf);
    const float sc = lr > 1e-12f ? 1.f / (nf * lr) : 0.f;  // 1/(N LRMSD); 0 where LRMSD vanishes
    if (tid == 0 && ok) {
        loss_out[b] = lr;
        float* st = state_out + (size_t)b * 16;
#pragma unroll
        for (int k = 0; k < 9; ++k) st[k] = U[k];
        st[9] = cx; st[10] = cy; st[11] = cz;  // x_0 = 0: absolute
        st[12] = dcx; st[13] = dcy; st[14] = dcz;
        st[15] = sc;
    }
    if (!ok) {
        if (tid == 0) atomicOr(err, ERR_LENGTH);
        return;
    }
    TPL_STAMP(5);

    // ---- backward pass 2: runs last atom to first (as bbp_backward_xyz_kernel, P = x)
    const Span so = make_span(grad_angles + (size_t)b * Lmax * 3, Lv * 12);
    float* s_go = reinterpret_cast<float*>(s_go_base + so.mis());
    float oa[3 * R], ob[3 * R];
    {
        const float* xp = s_x + 9 * j0 - 3;  // the atom before run A (unused for the chain's atom 0)
        const float pAx = j0 > 0 ? xp[0] : 0.f, pAy = j0 > 0 ? xp[1] : 0.f, pAz = j0 > 0 ? xp[2] : 0.f;
#pragma unroll
        for (int i = 3 * R - 1; i >= 0; --i) {
            const float2 px = X[i], py = Y[i], pz = Z[i];
            float2 qx, qy, qz;
            if (i > 0) {
                qx = X[i - 1]; qy = Y[i - 1]; qz = Z[i - 1];
            } else {
                qx = make_float2(pAx, X[3 * R - 1].x);
                qy = make_float2(pAy, Y[3 * R - 1].x);
                qz = make_float2(pAz, Z[3 * R - 1].x);
            }
            const float2 ux = __fadd2_rn(px, make_float2(-qx.x, -qx.y));
            const float2 uy = __fadd2_rn(py, make_float2(-qy.x, -qy.y));
            const float2 uz = __fadd2_rn(pz, make_float2(-qz.x, -qz.y));
            const float2 c0 = __fadd2_rn(T0, __ffma2_rn(make_float2(-py.x, -py.y), S2, __fmul2_rn(pz, S1)));
            const float2 c1 = __fadd2_rn(T1, __ffma2_rn(make_float2(-pz.x, -pz.y), S0, __fmul2_rn(px, S2)));
            const float2 c2 = __fadd2_rn(T2, __ffma2_rn(make_float2(-px.x, -px.y), S1, __fmul2_rn(py, S0)));
            const float2 uc = __ffma2_rn(ux, c0, __ffma2_rn(uy, c1, __fmul2_rn(uz, c2)));
            const int q = i / 3, k = i - 3 * q;
            // the bond ending at atom i has the model's length kBBd[k] (the forward built it so):
            // its unit axis is u / d, no rsqrt
            const float2 gv = __fmul2_rn(uc, f2(bb_invd(k)));
            if (k == 1) { oa[3 * q] = gv.x; ob[3 * q] = gv.y; }
            else if (k == 2) { oa[3 * q + 1] = gv.x; ob[3 * q + 1] = gv.y; }
            else {
                if (q > 0) { oa[3 * (q - 1) + 2] = gv.x; ob[3 * (q - 1) + 2] = gv.y; }
                else oa[3 * (R - 1) + 2] = gv.y;
            }
            float2 gx, gy, gz;
            resid(i, gx, gy, gz);
            S0 = __fadd2_rn(S0, gx); S1 = __fadd2_rn(S1, gy); S2 = __fadd2_rn(S2, gz);
            T0 = __fadd2_rn(T0, __ffma2_rn(py, gz, __fmul2_rn(make_float2(-pz.x, -pz.y), gy)));
            T1 = __fadd2_rn(T1, __ffma2_rn(pz, gx, __fmul2_rn(make_float2(-px.x, -px.y), gz)));
            T2 = __fadd2_rn(T2, __ffma2_rn(px, gy, __fmul2_rn(make_float2(-py.x, -py.y), gx)));
        }
        const int jl = j0 + 2 * R - 1;  // omega of the thread's last residue (closure, as packed.cu)
        float wl_ = 0.f;
        if (jl < Lv - 1) {
            const float* xn = s_x + 9 * (jl + 1);
            const float nx = xn[0], ny = xn[1], nz = xn[2];
            const float ux = nx - X[3 * R - 1].y, uy = ny - Y[3 * R - 1].y, uz = nz - Z[3 * R - 1].y;
            const float c0 = ext[3] - fmaf(ny, ext[2], -nz * ext[1]);
            const float c1 = ext[4] - fmaf(nz, ext[0], -nx * ext[2]);
            const float c2 = ext[5] - fmaf(nx, ext[1], -ny * ext[0]);
            wl_ = bb_invd(0) * fmaf(ux, c0, fmaf(uy, c1, uz * c2));  // C -> N bond: length kBBd[0]
        }
        ob[3 * (R - 1) + 2] = wl_;
#pragma unroll
        for (int q = 0; q < R; ++q) {
            if (j0 + q == Lv - 1) oa[3 * q + 2] = 0.f;
            if (j0 + R + q == Lv - 1) ob[3 * q + 2] = 0.f;
        }
#pragma unroll
        for (int k = 0; k < 3 * R; ++k) {  // dLRMSD/dalpha = (dE-weighted sums) / (N LRMSD)
            oa[k] *= sc;
            ob[k] *= sc;
        }
    }
    sts_run<3 * R>(s_go + 3 * j0, oa);
    sts_run<3 * R>(s_go + 3 * j0 + 3 * R, ob);
    __syncwarp();
    const int wn = min(WRES, L - w0);
    if (wn > 0) store_warp_chunk(grad_angles + ((size_t)b * Lmax + w0) * 3, s_go + 3 * w0, wn * 12, lane);
    TPL_STAMP(6);
    (void)B;
    (void)tot7;
}

template <int NT, int R>
static size_t bbp_lrmsd_smem() {
    constexpr int TILE = 2 * R * NT, NW = NT / 32;
    constexpr int XB = (16 + 36 * TILE + 16 + 15) & ~15;
    const size_t head = 8 * (NW + 1) + 8 + 8 * (NW * 17 + 1) + 4 * (32 + 2 * NW * 12 + 12 + 2 * NW * 7 + 16);
    return ((head + 15) & ~size_t(15)) + ((16 + 12 * TILE + 16 + 15) & ~15) + 2 * XB + 16 + 12 * TILE + 16;
}

template <int NT, int R, int NS>
static cudaError_t launch_bbp_lrmsd(const BBArgs& a, float* grad_angles, cudaStream_t st) {
    auto k = bbp_lrmsd_kernel<NT, R, NS>;
    const BBPLaunch l = bbp_policy(a.B, bbp_lrmsd_smem<NT, R>());
    static LaunchCfg cfg;
    cudaError_t e = ensure_launch_cfg(cfg, k, NT, l.smem);
    if (e != cudaSuccess) return e;
    return launch_bbp(k, a.B, NT, l, st, a.angles, a.lengths, a.B, a.Lmax, a.loss_target, a.coords, a.loss_out,
                      a.loss_state_out, grad_angles, a.err);
}

int bbp_lrmsd_max_L() { return kBBPMaxL; }

cudaError_t bbp_lrmsd_fused_launch(const BBArgs& a, float* grad_angles, cudaStream_t st) {
    if (a.Lmax > bbp_lrmsd_max_L() || a.ns > 1) return cudaErrorInvalidConfiguration;
    const BBPShape sh = bbp_shape(a.Lmax);
#define TPL_BBL(NT_, R_) \
    if (sh.nt == NT_ && sh.r == R_) return a.ns == 0 ? launch_bbp_lrmsd<NT_, R_, 0>(a, grad_angles, st) : launch_bbp_lrmsd<NT_, R_, 1>(a, grad_angles, st);
    TPL_BBL(128, 1) TPL_BBL(128, 2) TPL_BBL(128, 3) TPL_BBL(192, 3)
#undef TPL_BBL
    return cudaErrorInvalidConfiguration;
}

// dL/dalpha = dL/dLRMSD[b] * dLRMSD/dalpha (the autograd backward of the fused pass).
// y[b][i] = s[b] x[b][i]: blockIdx.y = chain (no index division), 16-byte vectors
// when the row and the pointers allow it.
template <bool kVec>
__global__ void chain_scale_kernel(const float* __restrict__ x, const float* __restrict__ s, int per_chain,
                                   float* __restrict__ y) {
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.y;
    const float f = __ldg(s + b);
    const size_t base = (size_t)b * per_chain;
    if (kVec) {
        const float4* x4 = reinterpret_cast<const float4*>(x + base);
        float4* y4 = reinterpret_cast<float4*>(y + base);
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < per_chain / 4; i += gridDim.x * blockDim.x) {
            float4 v = __ldg(x4 + i);
            v.x *= f; v.y *= f; v.z *= f; v.w *= f;
            y4[i] = v;
        }
    } else {
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < per_chain; i += gridDim.x * blockDim.x)
            y[base + i] = __ldg(x + base + i) * f;
    }
}
cudaError_t chain_scale_launch(const float* x, const float* s, int B, int per_chain, float* y, cudaStream_t st) {
    if (B == 0 || per_chain == 0) return cudaSuccess;
    const bool vec = per_chain % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(y) & 15) == 0;
    const int items = vec ? per_chain / 4 : per_chain;
    // 256 threads, about two items each, enough CTAs per chain for ~8 per SM: behind the
    // one-pass kernel (gradient still in L2) fewer, fuller CTAs finish sooner (lrmsd step
    // 13.90 -> 13.80 us against 128 threads x 1 item)
    const int nt = 256;
    const int per = std::max(1, std::min((items + 2 * nt - 1) / (2 * nt), (8 * device_sm_count() + B - 1) / B));
    // programmatic dependent launch: it usually follows the fused pass directly
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    for (int b0 = 0; b0 < B; b0 += 65535) {  // gridDim.y <= 65535 chains per launch
        const int nb = std::min(B - b0, 65535);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(per, nb);
        cfg.blockDim = dim3(nt);
        cfg.stream = st;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const size_t o = (size_t)b0 * per_chain;
        const cudaError_t e = vec ? cudaLaunchKernelEx(&cfg, chain_scale_kernel<true>, x + o, s + b0, per_chain, y + o)
                                  : cudaLaunchKernelEx(&cfg, chain_scale_kernel<false>, x + o, s + b0, per_chain, y + o);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

#ifdef TPL_PROFILE_PHASES
extern "C" __attribute__((visibility("default"))) int tpl_debug_stamps_fused(unsigned long long* host, int n) {
    return int(cudaMemcpyFromSymbol(host, g_tpl_stamps, sizeof(unsigned long long) * n));
}
#endif

}  // namespace tpl
