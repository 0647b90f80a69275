// packed.cu -- backbone kernels with two residue runs per thread in the two
// lanes of packed fp32 pairs (sm_100a fma.rn.f32x2 / mul.rn.f32x2), for chains
// that fit one CTA tile (§3).
//
// Forward (M_i = M_{i-1} R_i): thread t owns residues
// [2Rt, 2Rt + 2R) as two runs of R, run A = [2Rt, 2Rt + R) in the .x lanes and
// run B = [2Rt + R, 2Rt + 2R) in the .y lanes.  Both runs are composed from the
// identity at once -- every bond update R(alpha, theta, d) (the printed matrix
// P:149-155, 27 flops) and every sincos is one packed instruction stream for
// the pair, so a thread's serial chain is R residues while the block scan sees
// 2R residues per thread.  The thread's aggregate A B enters the block-wide
// exclusive scan of 3x4 affines (common.cuh); run A is placed with the prefix P,
// run B with P A.  Each element keeps the rounding of the scalar kernels
// (same operations per element, FMA contraction as written).
//
// Latency cuts for few chains (the 256 x 700 headline has <= 2 chains per SM):
// the tile is bulk-loaded for Lmax residues before the chain's length is known
// (residues past the length only influence later residues, which are never
// stored), so the length load overlaps the whole computation; each warp
// bulk-stores its own contiguous residues.
#include <cstdio>
#include <cstdlib>
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "packed.cuh"

namespace tpl {

// ---------------------------------------------------------------------------
// Forward, one CTA per chain, NT threads x 2R residues (tile TILE = 2 R NT >= Lmax).
template <int NT, int R, int kNS>
__global__ void __launch_bounds__(NT, NT * R >= 512 ? 384 / NT : 512 / NT) bbp_forward_kernel(const float* __restrict__ angles,
                                                                             const int* __restrict__ lengths, int B,
                                                                             int Lmax, float* __restrict__ coords,
                                                                             unsigned* __restrict__ err) {
    constexpr int TILE = 2 * R * NT;
    constexpr int NW = NT / 32;
    extern __shared__ __align__(16) char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    float* scratch = reinterpret_cast<float*>(smem + 16);             // 2 NW 12 floats
    float* s_total = scratch + 2 * NW * 12;                            // 12 floats
    char* s_ang_base = smem + 16 + (2 * NW * 12 + 16) * 4;             // 16 + 12 TILE bytes (+ head slack)
    char* s_out_base = s_ang_base + ((16 + 12 * TILE + 16 + 15) & ~15);  // 16 + 36 TILE bytes

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b = blockIdx.x;
    TPL_STAMP(0);
    const Span sa = make_span(angles + (size_t)b * Lmax * 3, Lmax * 12);
    if (tid == 0 && sa.mid > 0 && prefetch_regime(B)) prefetch_l2(sa.g + sa.head, unsigned(sa.mid));  // under the previous kernel's tail
    pdl_wait();     // programmatic dependent launch: nothing global is read before this
    pdl_trigger();  // every CTA is resident: the next kernel may start launching
    if (tid == 0) {
        mbar_init(bar, 1);
        fence_barrier_init();
        mbar_arrive_expect_tx(bar, unsigned(sa.mid));
        span_load_bulk(sa, s_ang_base, bar);
    }
    const int L = __ldg(lengths + b);  // consumed only by the store
    span_load_edges_f32(sa, s_ang_base);
    __syncthreads();  // barrier initialised, edges in place
    TPL_STAMP(1);
    mbar_wait(bar, 0);
    TPL_STAMP(2);
    const float* s_ang = reinterpret_cast<const float*>(s_ang_base + sa.mis());

    // ---- pass 1: runs A (.x) and B (.y) from the identity; atom positions kept
    const int j0 = 2 * R * tid;  // first residue of run A; run B starts at j0 + R
    float2 px[3 * R], py[3 * R], pz[3 * R];
    Aff2 M;
    bbp_pass1<R>(s_ang, Lmax, j0, tid == 0, px, py, pz, M);
    const Aff A = lane_x(M);
    Aff agg = aff_compose(A, lane_y(M));
    if (kNS >= 2) aff_orthonormalize(agg);  // policy 1: the quaternion extraction renormalises
    TPL_STAMP(3);

    // ---- block scan of the thread aggregates (carry: identity, one tile); policy 1
    //      (default) scans in (quaternion, translation) form, renormalised every combine
    const Aff P = kNS == 1 ? block_exclusive_scan_qt<NT>(agg, scratch)
                           : block_exclusive_scan<NT, kNS>(agg, aff_identity(), scratch, s_total);
    const Aff PB = aff_compose(P, A);
    const Aff2 P2 = pack2(P, PB);
    TPL_STAMP(4);

    // ---- pass 2: positions to the output staging (run A then run B)
    const int ok = L >= 1 && L <= Lmax;
    const Span so = make_span(coords + (size_t)b * 3 * Lmax * 3, (ok ? L : 0) * 36);
    float* s_out = reinterpret_cast<float*>(s_out_base + so.mis());
    {
        float fa[9 * R], fb[9 * R];
#pragma unroll
        for (int a = 0; a < 3 * R; ++a) {
            float2 ox, oy, oz;
            apply2(P2, px[a], py[a], pz[a], ox, oy, oz);
            fa[3 * a] = ox.x; fa[3 * a + 1] = oy.x; fa[3 * a + 2] = oz.x;
            fb[3 * a] = ox.y; fb[3 * a + 1] = oy.y; fb[3 * a + 2] = oz.y;
        }
        sts_run<9 * R>(s_out + 9 * j0, fa);
        sts_run<9 * R>(s_out + 9 * j0 + 9 * R, fb);
    }
    TPL_STAMP(5);
    if (!ok) {
        if (tid == 0) atomicOr(err, ERR_LENGTH);
        return;
    }
    // ---- per-warp stores of the warp's contiguous residues (same 16-byte phase in shared
    //      and global memory: a warp's chunk starts 36 * 64 * R bytes apart)
    __syncwarp();
    const int w0 = warp * 64 * R, wn = min(64 * R, L - w0);
    if (wn > 0) store_warp_chunk(coords + ((size_t)b * 3 * Lmax + 3 * (size_t)w0) * 3, s_out + 9 * w0, wn * 36, lane);
    TPL_STAMP(7);
    (void)B;
    (void)NW;
}

// Forward for chains longer than one tile (the ragged / long-chain configs): one CTA
// per chain walks its tiles first to last with the chain prefix as a carry in
// (quaternion, translation) form; tile t + 1's angles (with the residue before, for its
// omega) are bulk-loaded into the other buffer while tile t is computed.  Policy 1.
template <int NT, int R>
__global__ void __launch_bounds__(NT, NT * R >= 512 ? 384 / NT : 512 / NT) bbp_forward_tiles_kernel(
    const float* __restrict__ angles, const int* __restrict__ lengths, int B, int Lmax, float* __restrict__ coords,
    unsigned* __restrict__ err) {
    constexpr int TILE = 2 * R * NT;
    constexpr int NW = NT / 32;
    constexpr int ANG = (16 + 12 * (TILE + 1) + 16 + 15) & ~15;
    extern __shared__ __align__(16) char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);    // one per angle buffer
    float* scratch = reinterpret_cast<float*>(smem + 16);  // NW * 8 + 8 floats
    char* s_ang_buf = smem + 16 + ((NW * 8 + 8) * 4 + 15) / 16 * 16;
    char* s_out_base = s_ang_buf + 2 * ANG;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b = blockIdx.x;
    pdl_wait();
    pdl_trigger();
    const int L = __ldg(lengths + b);
    if (L < 1 || L > Lmax) {
        if (tid == 0) atomicOr(err, ERR_LENGTH);
        return;
    }
    const int nt = (L + TILE - 1) / TILE;
    auto tile_span = [&](int t) {
        const int r0 = t * TILE, pre = t > 0 ? 1 : 0, n = min(TILE, L - r0);
        return make_span(angles + ((size_t)b * Lmax + r0 - pre) * 3, (n + pre) * 12);
    };
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        fence_barrier_init();
        const Span s0 = tile_span(0);
        mbar_arrive_expect_tx(bar, unsigned(s0.mid));
        span_load_bulk(s0, s_ang_buf, bar);
    }
    span_load_edges_f32(tile_span(0), s_ang_buf);
    __syncthreads();
    QT carry = qt_identity();
    unsigned phases = 0;
    const int j0 = 2 * R * tid;
    for (int t = 0; t < nt; ++t) {
        const int buf = t & 1, r0 = t * TILE, n = min(TILE, L - r0), pre = t > 0 ? 1 : 0;
        if (t + 1 < nt) {  // prefetch the next tile (its buffer was consumed two tiles ago)
            const Span sn = tile_span(t + 1);
            if (tid == 0) {
                mbar_arrive_expect_tx(bar + (buf ^ 1), unsigned(sn.mid));
                span_load_bulk(sn, s_ang_buf + (buf ^ 1) * ANG, bar + (buf ^ 1));
            }
            span_load_edges_f32(sn, s_ang_buf + (buf ^ 1) * ANG);
        }
        mbar_wait(bar + buf, (phases >> buf) & 1u);
        phases ^= 1u << buf;
        const Span sa = tile_span(t);
        const float* s_ang = reinterpret_cast<const float*>(s_ang_buf + buf * ANG + sa.mis()) + 3 * pre;
        float2 px[3 * R], py[3 * R], pz[3 * R];
        Aff2 M;
        bbp_pass1<R>(s_ang, n, j0, t == 0 && tid == 0, px, py, pz, M, t > 0);
        const Aff A = lane_x(M);
        Aff agg = aff_compose(A, lane_y(M));
        // no Newton-Schulz step: the quaternion extraction renormalises (reading Q25)
        const Aff P = block_exclusive_scan_qt_carry<NT>(agg, scratch, carry);
        const Aff2 P2 = pack2(P, aff_compose(P, A));
        float* gout = coords + ((size_t)b * 3 * Lmax + 3 * (size_t)r0) * 3;
        float* s_out = reinterpret_cast<float*>(s_out_base + int(reinterpret_cast<uintptr_t>(gout) & 15));
        if (warp * 64 * R < n) {  // warps past the chain's end have nothing to place
            float fa[9 * R], fb[9 * R];
#pragma unroll
            for (int a = 0; a < 3 * R; ++a) {
                float2 ox, oy, oz;
                apply2(P2, px[a], py[a], pz[a], ox, oy, oz);
                fa[3 * a] = ox.x; fa[3 * a + 1] = oy.x; fa[3 * a + 2] = oz.x;
                fb[3 * a] = ox.y; fb[3 * a + 1] = oy.y; fb[3 * a + 2] = oz.y;
            }
            sts_run<9 * R>(s_out + 9 * j0, fa);
            sts_run<9 * R>(s_out + 9 * j0 + 9 * R, fb);
        }
        __syncwarp();
        const int w0 = warp * 64 * R, wn = min(64 * R, n - w0);
        if (wn > 0) store_warp_chunk(gout + 9 * (size_t)w0, s_out + 9 * w0, wn * 36, lane);
        // the staging and this tile's angle buffer are reused after the next tile's scan barrier
    }
    (void)B;
}

template <int NT, int R>
static size_t bbp_fwd_tiles_smem() {
    constexpr int TILE = 2 * R * NT, NW = NT / 32;
    constexpr int ANG = (16 + 12 * (TILE + 1) + 16 + 15) & ~15;
    return 16 + ((NW * 8 + 8) * 4 + 15) / 16 * 16 + 2 * ANG + 16 + 36 * TILE + 16;
}

template <int NT, int R>
static size_t bbp_fwd_smem() {
    constexpr int TILE = 2 * R * NT, NW = NT / 32;
    return 16 + (2 * NW * 12 + 16) * 4 + ((16 + 12 * TILE + 16 + 15) & ~15) + 16 + 36 * TILE + 16;
}

template <int NT, int R, int NS>
static cudaError_t launch_bbp_fwd(const BBArgs& a, cudaStream_t st) {
    auto k = bbp_forward_kernel<NT, R, NS>;
    const BBPLaunch l = bbp_policy(a.B, bbp_fwd_smem<NT, R>());
    static LaunchCfg cfg;
    cudaError_t e = ensure_launch_cfg(cfg, k, NT, l.smem);
    if (e != cudaSuccess) return e;
    return launch_bbp(k, a.B, NT, l, st, a.angles, a.lengths, a.B, a.Lmax, a.coords, a.err);
}

// TPL_PACKED=0 disables the packed kernels (A/B against the chain-serial ones).
bool bbp_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("TPL_PACKED");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

int bbp_forward_max_L() { return kBBPMaxL; }

template <int NT, int R>
static cudaError_t launch_bbp_fwd_ns(const BBArgs& a, cudaStream_t st) {
    if (a.ns == 0) return launch_bbp_fwd<NT, R, 0>(a, st);
    if (a.ns == 1) return launch_bbp_fwd<NT, R, 1>(a, st);
    return launch_bbp_fwd<NT, R, 2>(a, st);
}

template <int NT, int R>
static cudaError_t launch_bbp_fwd_tiles(const BBArgs& a, cudaStream_t st) {
    auto k = bbp_forward_tiles_kernel<NT, R>;
    const BBPLaunch l = bbp_policy(a.B, bbp_fwd_tiles_smem<NT, R>());
    static LaunchCfg cfg;
    cudaError_t e = ensure_launch_cfg(cfg, k, NT, l.smem);
    if (e != cudaSuccess) return e;
    return launch_bbp(k, a.B, NT, l, st, a.angles, a.lengths, a.B, a.Lmax, a.coords, a.err);
}

// Multi-tile chains (Lmax > kBBPMaxL): TPL_BBPT=NTxR forces the tile shape (tuning).
cudaError_t bbp_forward_tiles_launch(const BBArgs& a, cudaStream_t st) {
    static int env_nt = -1, env_r = 0;
    if (env_nt < 0) {
        env_nt = 0;
        if (const char* e = std::getenv("TPL_BBPT")) {
            if (std::sscanf(e, "%dx%d", &env_nt, &env_r) != 2) env_nt = 0;
        }
    }
    if (env_nt == 192 && env_r == 3) return launch_bbp_fwd_tiles<192, 3>(a, st);
    if (env_nt == 128 && env_r == 2) return launch_bbp_fwd_tiles<128, 2>(a, st);
    if (env_nt == 64 && env_r == 3) return launch_bbp_fwd_tiles<64, 3>(a, st);
    if (env_nt == 96 && env_r == 3) return launch_bbp_fwd_tiles<96, 3>(a, st);
    return launch_bbp_fwd_tiles<128, 3>(a, st);
}

cudaError_t bbp_forward_launch(const BBArgs& a, cudaStream_t st) {
    if (a.ns > 2) return cudaErrorInvalidConfiguration;
    static int env_nt = -1, env_r = 0;  // TPL_BBP=NTxR forces a shape (tuning)
    if (env_nt < 0) {
        env_nt = 0;
        if (const char* e = std::getenv("TPL_BBP")) {
            if (std::sscanf(e, "%dx%d", &env_nt, &env_r) != 2) env_nt = 0;
        }
    }
    BBPShape sh = bbp_shape(a.Lmax);
    if (env_nt > 0 && 2 * env_nt * env_r >= a.Lmax) sh = {env_nt, env_r};
    const int nt = sh.nt, r = sh.r;
#define TPL_BBP(NT_, R_) \
    if (nt == NT_ && r == R_) return launch_bbp_fwd_ns<NT_, R_>(a, st);
    TPL_BBP(128, 1) TPL_BBP(128, 2) TPL_BBP(128, 3) TPL_BBP(128, 4) TPL_BBP(192, 3)
#undef TPL_BBP
    return cudaErrorInvalidConfiguration;
}

// ---------------------------------------------------------------------------
// Coordinate backward (Eq. 2, via the rotation-axis identity; reading
// Q23), one CTA per chain, runs as the forward: thread t owns residues
// [2Rt, 2Rt + 2R), run A in the .x lanes, run B in the .y lanes.  With atoms
// a = 3j + k (N, CA, C), S_a = sum_{b>a} g_b and T_a = sum_{b>a} (x_b - c) x g_b
// about the chain's first atom c,
//     dL/dalpha_a = e_a . (T_a - (x_a - c) x S_a),   e_a = unit(x_a - x_{a-1}),
// alpha_{3j+1} = phi_j, alpha_{3j+2} = psi_j, alpha_{3j} = omega_{j-1}.
// Pass 1 reduces (S, T) of each run (kept: x - c of every atom); one block-wide
// exclusive suffix sum gives each run the sums of all later atoms; pass 2 walks
// each run last to first.  omega of a thread's last residue is closed from the
// next thread's first atom N (its own lever arm about N is zero), so every
// thread writes only its own residues and each warp bulk-stores its residues
// without a block barrier.  The tile is loaded in one TMA piece per warp (each
// warp starts on its own data), for Lmax residues before the length is known;
// atoms past the length are zeroed in shared memory (they add nothing).
template <int NT, int R>
__global__ void __launch_bounds__(NT, NT * R >= 512 ? 2 : (R >= 3 ? 3 : 4)) bbp_backward_xyz_kernel(const float* __restrict__ coords,
                                                                        const int* __restrict__ lengths, int B,
                                                                        int Lmax,
                                                                        const float* __restrict__ grad_coords,
                                                                        float* __restrict__ grad_angles,
                                                                        unsigned* __restrict__ err) {
    constexpr int TILE = 2 * R * NT;
    constexpr int NW = NT / 32;
    constexpr int WRES = 64 * R;                       // residues per warp
    constexpr int XB = (16 + 36 * TILE + 16 + 15) & ~15;  // coordinate / dL/dr staging (+ slack)
    extern __shared__ __align__(16) char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);                         // NW barriers
    float* s_suf = reinterpret_cast<float*>(smem + 8 * NW + 8);                // 2 NW 6 + 8 floats
    char* s_x_base = smem + ((8 * NW + 8 + (2 * NW * 6 + 8) * 4 + 15) & ~15);
    char* s_g_base = s_x_base + XB;
    char* s_go_base = s_g_base + XB;                                            // 16 + 12 TILE bytes

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b = blockIdx.x;
    TPL_STAMP(8);
    const size_t cbase = (size_t)b * 3 * Lmax * 3;
    const int w0 = warp * WRES;                       // the warp's first residue
    const int wl = max(0, min(WRES, Lmax - w0));      // residues of the warp's piece (speculative: Lmax)
    const Span sxw = make_span(coords + cbase + 9 * (size_t)w0, wl * 36);
    const Span sgw = make_span(grad_coords + cbase + 9 * (size_t)w0, wl * 36);
    if (lane == 0 && sgw.mid > 0 && prefetch_regime(B)) prefetch_l2(sgw.g + sgw.head, unsigned(sgw.mid));  // dL/dr is cold
    pdl_wait();
    pdl_trigger();
    if (lane == 0) {  // each warp initialises its own barrier and issues its own piece
        mbar_init(bar + warp, 1);
        fence_barrier_init();
        mbar_arrive_expect_tx(bar + warp, unsigned(sxw.mid + sgw.mid));
        span_load_bulk(sxw, s_x_base + 36 * w0, bar + warp);
        span_load_bulk(sgw, s_g_base + 36 * w0, bar + warp);
    }
    const int L = __ldg(lengths + b);
    const float* c0p = coords + cbase;
    const float cx = __ldg(c0p), cy = __ldg(c0p + 1), cz = __ldg(c0p + 2);  // reference point: atom 0
    const int mis = int(reinterpret_cast<uintptr_t>(coords + cbase) & 15);   // same for dL/dr (checked on host)
    float* s_x = reinterpret_cast<float*>(s_x_base + mis);
    float* s_g = reinterpret_cast<float*>(s_g_base + mis);
    span_load_edges_warp(sxw, s_x_base + 36 * w0, lane);
    span_load_edges_warp(sgw, s_g_base + 36 * w0, lane);
    __syncwarp();  // the warp's barrier initialised, its edges in place
    const bool ok = L >= 1 && L <= Lmax;
    const int Lv = ok ? L : 0;
    TPL_STAMP(9);
    mbar_wait(bar + warp, 0);
    // zero the warp's atoms at and past the chain's end (pads and unloaded slack)
    {
        const int f0 = 9 * max(Lv, w0), f1 = 9 * (w0 + WRES);
        for (int f = f0 + lane; f < f1; f += 32) {
            s_x[f] = 0.f;
            s_g[f] = 0.f;
        }
    }
    __syncwarp();
    TPL_STAMP(10);

    // ---- pass 1: (S, T) of runs A and B; P = x - c of every atom kept
    const int j0 = 2 * R * tid;
    float2 Px[3 * R], Py[3 * R], Pz[3 * R];
    float2 S0 = f2(0.f), S1 = f2(0.f), S2 = f2(0.f), T0 = f2(0.f), T1 = f2(0.f), T2 = f2(0.f);
    if (__any_sync(0xffffffffu, j0 < Lv)) {  // warps past the chain's end add nothing
        float xa[9 * R], xb[9 * R], ga[9 * R], gb[9 * R];
        lds_run<9 * R>(s_x + 9 * j0, xa);
        lds_run<9 * R>(s_x + 9 * j0 + 9 * R, xb);
        lds_run<9 * R>(s_g + 9 * j0, ga);
        lds_run<9 * R>(s_g + 9 * j0 + 9 * R, gb);
        const float2 c2x = f2(cx), c2y = f2(cy), c2z = f2(cz);
#pragma unroll
        for (int i = 0; i < 3 * R; ++i) {
            const float2 px = __fadd2_rn(make_float2(xa[3 * i], xb[3 * i]), make_float2(-c2x.x, -c2x.y));
            const float2 py = __fadd2_rn(make_float2(xa[3 * i + 1], xb[3 * i + 1]), make_float2(-c2y.x, -c2y.y));
            const float2 pz = __fadd2_rn(make_float2(xa[3 * i + 2], xb[3 * i + 2]), make_float2(-c2z.x, -c2z.y));
            const float2 gx = make_float2(ga[3 * i], gb[3 * i]);
            const float2 gy = make_float2(ga[3 * i + 1], gb[3 * i + 1]);
            const float2 gz = make_float2(ga[3 * i + 2], gb[3 * i + 2]);
            Px[i] = px; Py[i] = py; Pz[i] = pz;
            S0 = __fadd2_rn(S0, gx); S1 = __fadd2_rn(S1, gy); S2 = __fadd2_rn(S2, gz);
            T0 = __fadd2_rn(T0, __ffma2_rn(py, gz, __fmul2_rn(make_float2(-pz.x, -pz.y), gy)));
            T1 = __fadd2_rn(T1, __ffma2_rn(pz, gx, __fmul2_rn(make_float2(-px.x, -px.y), gz)));
            T2 = __fadd2_rn(T2, __ffma2_rn(px, gy, __fmul2_rn(make_float2(-py.x, -py.y), gx)));
        }
    }
    TPL_STAMP(11);

    // ---- block-wide exclusive suffix sum of the thread totals (runs A + B)
    float v6[6] = {S0.x + S0.y, S1.x + S1.y, S2.x + S2.y, T0.x + T0.y, T1.x + T1.y, T2.x + T2.y};
    const float zero6[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float ext[6], tot6[6];
    block_exclusive_suffix6<NT, false>(v6, zero6, s_suf, ext, tot6);
    // running suffix state: lane y = after run B (= ext), lane x = after run A (= ext + run B)
    S0 = make_float2(ext[0] + S0.y, ext[0]); S1 = make_float2(ext[1] + S1.y, ext[1]);
    S2 = make_float2(ext[2] + S2.y, ext[2]); T0 = make_float2(ext[3] + T0.y, ext[3]);
    T1 = make_float2(ext[4] + T1.y, ext[4]); T2 = make_float2(ext[5] + T2.y, ext[5]);
    TPL_STAMP(12);

    // ---- pass 2: runs last atom to first
    const Span so = make_span(grad_angles + (size_t)b * Lmax * 3, Lv * 12);
    float* s_go = reinterpret_cast<float*>(s_go_base + so.mis());
    float oa[3 * R], ob[3 * R];  // (phi, psi, omega) of the run's residues
    const bool wact = __any_sync(0xffffffffu, j0 < Lv);
    if (wact) {
        float ga[9 * R], gb[9 * R];
        lds_run<9 * R>(s_g + 9 * j0, ga);
        lds_run<9 * R>(s_g + 9 * j0 + 9 * R, gb);
        // the atom before run A (previous thread's last atom; unused for atom 0 of the chain)
        const float* xp = s_x + 9 * j0 - 3;
        const float2 prevA = j0 > 0 ? make_float2(xp[0] - cx, 0.f) : f2(0.f);
        const float prevAy = j0 > 0 ? xp[1] - cy : 0.f, prevAz = j0 > 0 ? xp[2] - cz : 0.f;
#pragma unroll
        for (int i = 3 * R - 1; i >= 0; --i) {
            const float2 px = Px[i], py = Py[i], pz = Pz[i];
            float2 qx, qy, qz;  // the previous atom's P
            if (i > 0) {
                qx = Px[i - 1]; qy = Py[i - 1]; qz = Pz[i - 1];
            } else {
                qx = make_float2(prevA.x, Px[3 * R - 1].x);
                qy = make_float2(prevAy, Py[3 * R - 1].x);
                qz = make_float2(prevAz, Pz[3 * R - 1].x);
            }
            const float2 ux = __fadd2_rn(px, make_float2(-qx.x, -qx.y));
            const float2 uy = __fadd2_rn(py, make_float2(-qy.x, -qy.y));
            const float2 uz = __fadd2_rn(pz, make_float2(-qz.x, -qz.y));
            // c = T - P x S
            const float2 c0 = __fadd2_rn(T0, __ffma2_rn(make_float2(-py.x, -py.y), S2, __fmul2_rn(pz, S1)));
            const float2 c1 = __fadd2_rn(T1, __ffma2_rn(make_float2(-pz.x, -pz.y), S0, __fmul2_rn(px, S2)));
            const float2 c2 = __fadd2_rn(T2, __ffma2_rn(make_float2(-px.x, -px.y), S1, __fmul2_rn(py, S0)));
            const float2 uc = __ffma2_rn(ux, c0, __ffma2_rn(uy, c1, __fmul2_rn(uz, c2)));
            const int q = i / 3, k = i - 3 * q;
            // the bond ending at atom i has the model's length kBBd[k] (the forward built it so):
            // its unit axis is u / d, no rsqrt
            const float2 gv = __fmul2_rn(uc, f2(bb_invd(k)));
            if (k == 1) { oa[3 * q] = gv.x; ob[3 * q] = gv.y; }            // phi
            else if (k == 2) { oa[3 * q + 1] = gv.x; ob[3 * q + 1] = gv.y; }  // psi
            else {                                                            // omega of the residue before
                if (q > 0) { oa[3 * (q - 1) + 2] = gv.x; ob[3 * (q - 1) + 2] = gv.y; }
                else oa[3 * (R - 1) + 2] = gv.y;  // run B's first N closes run A's last omega
            }
            const float2 gx = make_float2(ga[3 * i], gb[3 * i]);
            const float2 gy = make_float2(ga[3 * i + 1], gb[3 * i + 1]);
            const float2 gz = make_float2(ga[3 * i + 2], gb[3 * i + 2]);
            S0 = __fadd2_rn(S0, gx); S1 = __fadd2_rn(S1, gy); S2 = __fadd2_rn(S2, gz);
            T0 = __fadd2_rn(T0, __ffma2_rn(py, gz, __fmul2_rn(make_float2(-pz.x, -pz.y), gy)));
            T1 = __fadd2_rn(T1, __ffma2_rn(pz, gx, __fmul2_rn(make_float2(-px.x, -px.y), gz)));
            T2 = __fadd2_rn(T2, __ffma2_rn(px, gy, __fmul2_rn(make_float2(-py.x, -py.y), gx)));
        }
        // omega of the thread's last residue jl: axis C_jl -> N_{jl+1} (next thread's first atom),
        // sums over the atoms after the thread (ext); structural zero for the chain's last residue
        const int jl = j0 + 2 * R - 1;
        float wl_ = 0.f;
        if (jl < Lv - 1) {
            const float* xn = s_x + 9 * (jl + 1);
            const float nx = xn[0] - cx, ny = xn[1] - cy, nz = xn[2] - cz;
            const float ux = nx - Px[3 * R - 1].y, uy = ny - Py[3 * R - 1].y, uz = nz - Pz[3 * R - 1].y;
            const float c0 = ext[3] - fmaf(ny, ext[2], -nz * ext[1]);
            const float c1 = ext[4] - fmaf(nz, ext[0], -nx * ext[2]);
            const float c2 = ext[5] - fmaf(nx, ext[1], -ny * ext[0]);
            wl_ = bb_invd(0) * fmaf(ux, c0, fmaf(uy, c1, uz * c2));  // C -> N bond: length kBBd[0]
        }
        ob[3 * (R - 1) + 2] = wl_;
        // omega_{L-1} is a structural zero wherever the chain ends inside a run
#pragma unroll
        for (int q = 0; q < R; ++q) {
            if (j0 + q == Lv - 1) oa[3 * q + 2] = 0.f;
            if (j0 + R + q == Lv - 1) ob[3 * q + 2] = 0.f;
        }
        sts_run<3 * R>(s_go + 3 * j0, oa);
        sts_run<3 * R>(s_go + 3 * j0 + 3 * R, ob);
    }
    TPL_STAMP(13);
    if (!ok) {
        if (tid == 0) atomicOr(err, ERR_LENGTH);
        return;
    }
    // ---- per-warp stores (a warp's chunk starts 12 * 64 R bytes apart: same 16-byte phase)
    __syncwarp();
    const int wn = min(WRES, L - w0);
    if (wn > 0) store_warp_chunk(grad_angles + ((size_t)b * Lmax + w0) * 3, s_go + 3 * w0, wn * 12, lane);
    TPL_STAMP(15);
    (void)B;
    (void)tot6;
}

// Coordinate backward for chains longer than one tile: one CTA per chain walks its
// tiles last to first; the (S, T) of the later tiles is carried about the current
// tile's first atom (T_c = T_c' + (c' - c) x S), and omega of a tile's last residue is
// closed with the next tile's first atom.  Tile t - 1 (coordinates with the atom before
// it, dL/dr) is bulk-loaded into the other buffer while tile t is computed.
template <int NT, int R, int NB>
__global__ void __launch_bounds__(NT, NT * R >= 512 ? 2 : (R >= 3 ? 3 : 4)) bbp_backward_xyz_tiles_kernel(
    const float* __restrict__ coords, const int* __restrict__ lengths, int B, int Lmax,
    const float* __restrict__ grad_coords, float* __restrict__ grad_angles, unsigned* __restrict__ err) {
    constexpr int TILE = 2 * R * NT;
    constexpr int NW = NT / 32;
    constexpr int WRES = 64 * R;
    constexpr int XB = (16 + 36 * TILE + 12 + 16 + 15) & ~15;
    extern __shared__ __align__(16) char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);  // one per buffer
    float* s_suf = reinterpret_cast<float*>(smem + 16);  // 2 NW 6 + 8 floats
    char* s_x_buf = smem + ((16 + (2 * NW * 6 + 8) * 4 + 15) & ~15);
    char* s_g_buf = s_x_buf + NB * XB;
    char* s_go_base = s_g_buf + NB * XB;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b = blockIdx.x;
    pdl_wait();
    pdl_trigger();
    const int L = __ldg(lengths + b);
    if (L < 1 || L > Lmax) {
        if (tid == 0) atomicOr(err, ERR_LENGTH);
        return;
    }
    const int nt = (L + TILE - 1) / TILE;
    const size_t cb = (size_t)b * 3 * Lmax * 3;
    auto spans = [&](int t, Span& sx, Span& sg) {
        const int r0 = t * TILE, pre = t > 0 ? 1 : 0, n = min(TILE, L - r0);
        sx = make_span(coords + cb + 9 * (size_t)r0 - 3 * pre, (3 * n + pre) * 12);
        sg = make_span(grad_coords + cb + 9 * (size_t)r0, n * 36);
    };
    auto issue = [&](int t, int buf) {
        Span sx, sg;
        spans(t, sx, sg);
        if (tid == 0) {
            mbar_arrive_expect_tx(bar + buf, unsigned(sx.mid + sg.mid));
            span_load_bulk(sx, s_x_buf + buf * XB, bar + buf);
            span_load_bulk(sg, s_g_buf + buf * XB, bar + buf);
        }
        span_load_edges_f32(sx, s_x_buf + buf * XB);
        span_load_edges_f32(sg, s_g_buf + buf * XB);
    };
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        fence_barrier_init();
    }
    __syncthreads();
    issue(nt - 1, NB == 2 ? (nt - 1) & 1 : 0);
    float carry6[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float cpx = 0.f, cpy = 0.f, cpz = 0.f;
    unsigned phases = 0;
    const int j0 = 2 * R * tid;
    for (int t = nt - 1; t >= 0; --t) {
        const int buf = NB == 2 ? t & 1 : 0, r0 = t * TILE, n = min(TILE, L - r0), pre = t > 0 ? 1 : 0;
        if (NB == 2 && t > 0) issue(t - 1, buf ^ 1);  // its buffer was consumed two tiles ago
        mbar_wait(bar + buf, (phases >> buf) & 1u);
        phases ^= 1u << buf;
        Span sx, sg;
        spans(t, sx, sg);
        float* s_x = reinterpret_cast<float*>(s_x_buf + buf * XB + sx.mis()) + 3 * pre;  // atom 3 r0
        float* s_g = reinterpret_cast<float*>(s_g_buf + buf * XB + sg.mis());
        if (t == nt - 1) {  // the chain ends in this tile: atoms past it add nothing
            for (int f = 9 * n + tid; f < 9 * TILE; f += NT) {
                s_x[f] = 0.f;
                s_g[f] = 0.f;
            }
        }
        __syncthreads();  // edges and zero fill visible
        const float cx = s_x[0], cy = s_x[1], cz = s_x[2];  // the tile's reference point
        if (t < nt - 1) {  // the later tiles' moment about this tile's reference
            const float dx = cpx - cx, dy = cpy - cy, dz = cpz - cz;
            carry6[3] += fmaf(dy, carry6[2], -dz * carry6[1]);
            carry6[4] += fmaf(dz, carry6[0], -dx * carry6[2]);
            carry6[5] += fmaf(dx, carry6[1], -dy * carry6[0]);
        }
        cpx = cx; cpy = cy; cpz = cz;
        // ---- pass 1: (S, T) of runs A and B; P = x - c of every atom kept
        float2 Px[3 * R], Py[3 * R], Pz[3 * R];
        float2 S0 = f2(0.f), S1 = f2(0.f), S2 = f2(0.f), T0 = f2(0.f), T1 = f2(0.f), T2 = f2(0.f);
        if (warp * WRES < n) {  // warps past the chain's end add nothing
            float xa[9 * R], xb[9 * R], ga[9 * R], gb[9 * R];
            lds_run<9 * R>(s_x + 9 * j0, xa);
            lds_run<9 * R>(s_x + 9 * j0 + 9 * R, xb);
            lds_run<9 * R>(s_g + 9 * j0, ga);
            lds_run<9 * R>(s_g + 9 * j0 + 9 * R, gb);
            const float2 c2x = f2(cx), c2y = f2(cy), c2z = f2(cz);
    #pragma unroll
            for (int i = 0; i < 3 * R; ++i) {
                const float2 px = __fadd2_rn(make_float2(xa[3 * i], xb[3 * i]), make_float2(-c2x.x, -c2x.y));
                const float2 py = __fadd2_rn(make_float2(xa[3 * i + 1], xb[3 * i + 1]), make_float2(-c2y.x, -c2y.y));
                const float2 pz = __fadd2_rn(make_float2(xa[3 * i + 2], xb[3 * i + 2]), make_float2(-c2z.x, -c2z.y));
                const float2 gx = make_float2(ga[3 * i], gb[3 * i]);
                const float2 gy = make_float2(ga[3 * i + 1], gb[3 * i + 1]);
                const float2 gz = make_float2(ga[3 * i + 2], gb[3 * i + 2]);
                Px[i] = px; Py[i] = py; Pz[i] = pz;
                S0 = __fadd2_rn(S0, gx); S1 = __fadd2_rn(S1, gy); S2 = __fadd2_rn(S2, gz);
                T0 = __fadd2_rn(T0, __ffma2_rn(py, gz, __fmul2_rn(make_float2(-pz.x, -pz.y), gy)));
                T1 = __fadd2_rn(T1, __ffma2_rn(pz, gx, __fmul2_rn(make_float2(-px.x, -px.y), gz)));
                T2 = __fadd2_rn(T2, __ffma2_rn(px, gy, __fmul2_rn(make_float2(-py.x, -py.y), gx)));
            }
        }

        // ---- block-wide exclusive suffix sum of the thread totals (runs A + B)
        float v6[6] = {S0.x + S0.y, S1.x + S1.y, S2.x + S2.y, T0.x + T0.y, T1.x + T1.y, T2.x + T2.y};
        float ext[6], tot6[6];
        block_exclusive_suffix6<NT>(v6, carry6, s_suf, ext, tot6);
        // running suffix state: lane y = after run B (= ext), lane x = after run A (= ext + run B)
        S0 = make_float2(ext[0] + S0.y, ext[0]); S1 = make_float2(ext[1] + S1.y, ext[1]);
        S2 = make_float2(ext[2] + S2.y, ext[2]); T0 = make_float2(ext[3] + T0.y, ext[3]);
        T1 = make_float2(ext[4] + T1.y, ext[4]); T2 = make_float2(ext[5] + T2.y, ext[5]);

        // ---- pass 2: runs last atom to first
        float* gdst = grad_angles + ((size_t)b * Lmax + r0) * 3;
        float* s_go = reinterpret_cast<float*>(s_go_base + int(reinterpret_cast<uintptr_t>(gdst) & 15));
        float oa[3 * R], ob[3 * R];  // (phi, psi, omega) of the run's residues
        if (warp * WRES < n) {
            float ga[9 * R], gb[9 * R];
            lds_run<9 * R>(s_g + 9 * j0, ga);
            lds_run<9 * R>(s_g + 9 * j0 + 9 * R, gb);
            // the atom before run A (previous thread's last atom; unused for atom 0 of the chain)
            const float* xp = s_x + 9 * j0 - 3;
            const bool hp = j0 > 0 || t > 0;  // the atom before exists (previous thread, or the tile's pre atom)
            const float2 prevA = hp ? make_float2(xp[0] - cx, 0.f) : f2(0.f);
            const float prevAy = hp ? xp[1] - cy : 0.f, prevAz = hp ? xp[2] - cz : 0.f;
    #pragma unroll
            for (int i = 3 * R - 1; i >= 0; --i) {
                const float2 px = Px[i], py = Py[i], pz = Pz[i];
                float2 qx, qy, qz;  // the previous atom's P
                if (i > 0) {
                    qx = Px[i - 1]; qy = Py[i - 1]; qz = Pz[i - 1];
                } else {
                    qx = make_float2(prevA.x, Px[3 * R - 1].x);
                    qy = make_float2(prevAy, Py[3 * R - 1].x);
                    qz = make_float2(prevAz, Pz[3 * R - 1].x);
                }
                const float2 ux = __fadd2_rn(px, make_float2(-qx.x, -qx.y));
                const float2 uy = __fadd2_rn(py, make_float2(-qy.x, -qy.y));
                const float2 uz = __fadd2_rn(pz, make_float2(-qz.x, -qz.y));
                // c = T - P x S
                const float2 c0 = __fadd2_rn(T0, __ffma2_rn(make_float2(-py.x, -py.y), S2, __fmul2_rn(pz, S1)));
                const float2 c1 = __fadd2_rn(T1, __ffma2_rn(make_float2(-pz.x, -pz.y), S0, __fmul2_rn(px, S2)));
                const float2 c2 = __fadd2_rn(T2, __ffma2_rn(make_float2(-px.x, -px.y), S1, __fmul2_rn(py, S0)));
                const float2 uc = __ffma2_rn(ux, c0, __ffma2_rn(uy, c1, __fmul2_rn(uz, c2)));
                const int q = i / 3, k = i - 3 * q;
                // the bond ending at atom i has the model's length kBBd[k] (the forward built it so):
                // its unit axis is u / d, no rsqrt
                const float2 gv = __fmul2_rn(uc, f2(bb_invd(k)));
                if (k == 1) { oa[3 * q] = gv.x; ob[3 * q] = gv.y; }            // phi
                else if (k == 2) { oa[3 * q + 1] = gv.x; ob[3 * q + 1] = gv.y; }  // psi
                else {                                                            // omega of the residue before
                    if (q > 0) { oa[3 * (q - 1) + 2] = gv.x; ob[3 * (q - 1) + 2] = gv.y; }
                    else oa[3 * (R - 1) + 2] = gv.y;  // run B's first N closes run A's last omega
                }
                const float2 gx = make_float2(ga[3 * i], gb[3 * i]);
                const float2 gy = make_float2(ga[3 * i + 1], gb[3 * i + 1]);
                const float2 gz = make_float2(ga[3 * i + 2], gb[3 * i + 2]);
                S0 = __fadd2_rn(S0, gx); S1 = __fadd2_rn(S1, gy); S2 = __fadd2_rn(S2, gz);
                T0 = __fadd2_rn(T0, __ffma2_rn(py, gz, __fmul2_rn(make_float2(-pz.x, -pz.y), gy)));
                T1 = __fadd2_rn(T1, __ffma2_rn(pz, gx, __fmul2_rn(make_float2(-px.x, -px.y), gz)));
                T2 = __fadd2_rn(T2, __ffma2_rn(px, gy, __fmul2_rn(make_float2(-py.x, -py.y), gx)));
            }
            // omega of the thread's last residue jl: axis C_jl -> N_{jl+1} (next thread's first atom),
            // sums over the atoms after the thread (ext); structural zero for the chain's last residue
            const int jl = j0 + 2 * R - 1;
            float wl_ = 0.f;
            if (r0 + jl < L - 1) {  // N_{jl+1}: in this tile, or the next tile's first atom (global)
                const float* xn = jl + 1 < n ? s_x + 9 * (jl + 1) : coords + ((size_t)b * 3 * Lmax + 3 * (size_t)(r0 + n)) * 3;
                const float nx = xn[0] - cx, ny = xn[1] - cy, nz = xn[2] - cz;
                const float ux = nx - Px[3 * R - 1].y, uy = ny - Py[3 * R - 1].y, uz = nz - Pz[3 * R - 1].y;
                const float c0 = ext[3] - fmaf(ny, ext[2], -nz * ext[1]);
                const float c1 = ext[4] - fmaf(nz, ext[0], -nx * ext[2]);
                const float c2 = ext[5] - fmaf(nx, ext[1], -ny * ext[0]);
                wl_ = bb_invd(0) * fmaf(ux, c0, fmaf(uy, c1, uz * c2));  // C -> N bond: length kBBd[0]
            }
            ob[3 * (R - 1) + 2] = wl_;
            // omega_{L-1} is a structural zero wherever the chain ends inside a run
    #pragma unroll
            for (int q = 0; q < R; ++q) {
                if (r0 + j0 + q == L - 1) oa[3 * q + 2] = 0.f;
                if (r0 + j0 + R + q == L - 1) ob[3 * q + 2] = 0.f;
            }
            sts_run<3 * R>(s_go + 3 * j0, oa);
            sts_run<3 * R>(s_go + 3 * j0 + 3 * R, ob);
        }


        __syncwarp();
        const int w0 = warp * WRES, wn = min(WRES, n - w0);
        if (wn > 0) store_warp_chunk(gdst + 3 * w0, s_go + 3 * w0, wn * 12, lane);
#pragma unroll
        for (int q = 0; q < 6; ++q) carry6[q] = tot6[q];
        __syncthreads();  // this tile's buffers and the staging are free again
        if (NB == 1 && t > 0) issue(t - 1, 0);  // single buffer: refill now (other CTAs overlap it)
    }
    (void)B;
}

template <int NT, int R, int NB>
static size_t bbp_bwd_tiles_smem() {
    constexpr int TILE = 2 * R * NT, NW = NT / 32;
    constexpr int XB = (16 + 36 * TILE + 12 + 16 + 15) & ~15;
    return ((16 + (2 * NW * 6 + 8) * 4 + 15) & ~15) + 2 * NB * XB + 16 + 12 * TILE + 16;
}

template <int NT, int R, int NB>
static cudaError_t launch_bbp_bwd_xyz_tiles(const BBArgs& a, cudaStream_t st) {
    auto k = bbp_backward_xyz_tiles_kernel<NT, R, NB>;
    const BBPLaunch l = bbp_policy(a.B, bbp_bwd_tiles_smem<NT, R, NB>());
    static LaunchCfg cfg;
    cudaError_t e = ensure_launch_cfg(cfg, k, NT, l.smem);
    if (e != cudaSuccess) return e;
    return launch_bbp(k, a.B, NT, l, st, static_cast<const float*>(a.coords), a.lengths, a.B, a.Lmax,
                      a.grad_coords, a.grad_angles, a.err);
}

// TPL_BBPXT=NTxRxNB forces the shape and buffering (tuning).  Default: single-buffered
// 128 x 3 -- double buffering takes 2 x 55 KB of staging per CTA and left one CTA per
// SM (config 4 backward 175 us vs 86 us for the chain-serial kernel).
cudaError_t bbp_backward_xyz_tiles_launch(const BBArgs& a, cudaStream_t st) {
    static int nt = -1, r = 0, nb = 0;
    if (nt < 0) {
        nt = 0;
        if (const char* e = std::getenv("TPL_BBPXT")) {
            if (std::sscanf(e, "%dx%dx%d", &nt, &r, &nb) != 3) nt = 0;
        }
    }
    if (nt == 128 && r == 3 && nb == 2) return launch_bbp_bwd_xyz_tiles<128, 3, 2>(a, st);
    if (nt == 128 && r == 2 && nb == 1) return launch_bbp_bwd_xyz_tiles<128, 2, 1>(a, st);
    if (nt == 64 && r == 3 && nb == 1) return launch_bbp_bwd_xyz_tiles<64, 3, 1>(a, st);
    return launch_bbp_bwd_xyz_tiles<128, 3, 1>(a, st);
}

template <int NT, int R>
static size_t bbp_bwd_smem() {
    constexpr int TILE = 2 * R * NT, NW = NT / 32;
    constexpr int XB = (16 + 36 * TILE + 16 + 15) & ~15;
    return ((8 * NW + 8 + (2 * NW * 6 + 8) * 4 + 15) & ~15) + 2 * XB + 16 + 12 * TILE + 16;
}

template <int NT, int R>
static cudaError_t launch_bbp_bwd_xyz(const BBArgs& a, cudaStream_t st) {
    auto k = bbp_backward_xyz_kernel<NT, R>;
    const BBPLaunch l = bbp_policy(a.B, bbp_bwd_smem<NT, R>());
    static LaunchCfg cfg;
    cudaError_t e = ensure_launch_cfg(cfg, k, NT, l.smem);
    if (e != cudaSuccess) return e;
    return launch_bbp(k, a.B, NT, l, st, static_cast<const float*>(a.coords), a.lengths, a.B, a.Lmax,
                      a.grad_coords, a.grad_angles, a.err);
}

// coords and dL/dr must share their 16-byte phase (the staging mirrors both at one offset)
bool bbp_backward_xyz_ok(const BBArgs& a) {
    return a.Lmax <= kBBPMaxL &&
           ((reinterpret_cast<uintptr_t>(a.coords) ^ reinterpret_cast<uintptr_t>(a.grad_coords)) & 15) == 0 &&
           (size_t(a.Lmax) * 36) % 16 == 0;
}

cudaError_t bbp_backward_xyz_launch(const BBArgs& a, cudaStream_t st) {
    static int env_r = -1;  // TPL_BBPX=R forces the residues per run (tuning)
    if (env_r < 0) {
        const char* e = std::getenv("TPL_BBPX");
        env_r = e ? std::atoi(e) : 0;
    }
    BBPShape sh = bbp_shape(a.Lmax);
    if (env_r > 0 && 2 * 128 * env_r >= a.Lmax) sh = {128, env_r};
    if (sh.nt == 192) return launch_bbp_bwd_xyz<192, 3>(a, st);
    if (sh.r == 1) return launch_bbp_bwd_xyz<128, 1>(a, st);
    if (sh.r == 2) return launch_bbp_bwd_xyz<128, 2>(a, st);
    if (sh.r == 3) return launch_bbp_bwd_xyz<128, 3>(a, st);
    return launch_bbp_bwd_xyz<128, 4>(a, st);
}

#ifdef TPL_PROFILE_PHASES
// the stamp array is per translation unit: this file's copy
extern "C" __attribute__((visibility("default"))) int tpl_debug_stamps_packed(unsigned long long* host, int n) {
    return int(cudaMemcpyFromSymbol(host, g_tpl_stamps, sizeof(unsigned long long) * n));
}
#endif

}  // namespace tpl
