// backbone.cu -- batched backbone model (§3) on sm_100a.
//
// Forward: atom i of a chain sits at r_i = M_i 0 with
// M_i = R_0 R_1 ... R_i; transform 3j carries omega_{j-1} (C-N), 3j+1 phi_j
// (N-CA), 3j+2 psi_j (CA-C), R_0 = I (readings Q1, Q2 in DESIGN.md).
// Instead of the paper's saved M_i (64 B/atom) we compute M_i with a block-wide
// prefix scan of 3x4 affines and store only r_i (12 B/atom).
//
// Backward (Eq. 2): dr_j/dalpha_i = e_i x (r_j - r_i) for j > i
// (e_i = x-axis of frame M_i, the rotation axis of R_x(alpha_i)), hence
//   dL/dalpha_i = e_i . (T_i - r_i x S_i),  S_i = sum_{j>i} g_j,  T_i = sum_{j>i} r_j x g_j,
// one reverse suffix sum per chain: O(L) instead of the paper's O(L^2).
// The forward frames are recomputed from the angles (no saved state).
//
// Work decomposition: one CTA per chain; a tile of NT*RPT residues per CTA
// iteration; each thread owns RPT consecutive residues (3*RPT transforms).
// Longer chains loop over tiles carrying the prefix transform (forward) or,
// in backward, run a prefix pre-pass (phase A, tile prefixes to the
// workspace) then walk tiles last-to-first carrying the suffix sums.
#include "common.cuh"
#include "kernels.h"

namespace tpl {

template <int NT>
struct BBSmem {
    static constexpr int NW = NT / 32;
    static constexpr int kBar = 0;                        // uint64 mbarrier (16 B slot)
    static constexpr int kScratch = 16;                   // NW*12 floats
    static constexpr int kTotal = kScratch + NW * 12 * 4;  // 12 floats (+ misc)
    static constexpr int kMisc = kTotal + 48;             // 16 floats of misc
    static constexpr int kData = ((kMisc + 64 + 15) / 16) * 16;
};

__host__ __device__ constexpr int round16(int x) { return (x + 15) & ~15; }

// Transform i of the chain (atom i): angle index into the staged tile.
// s_ang points at local residue 0 of the tile; s_ang[-1] (omega of the
// previous residue) is staged whenever the tile does not start the chain.

template <int NT, int RPT, bool kOrtho>
__global__ void __launch_bounds__(NT) bb_forward_kernel(const float* __restrict__ angles,
                                                        const int* __restrict__ lengths, int Lmax,
                                                        float* __restrict__ coords, unsigned* __restrict__ err,
                                                        BBConst K) {
    constexpr int TILE = NT * RPT;
    constexpr int APT = 3 * RPT;
    using S = BBSmem<NT>;
    extern __shared__ __align__(16) char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::kBar);
    float* scratch = reinterpret_cast<float*>(smem + S::kScratch);
    float* s_total = reinterpret_cast<float*>(smem + S::kTotal);
    char* s_ang_base = smem + S::kData;
    char* s_out_base = s_ang_base + round16(16 + 12 * (TILE + 1));

    const int b = blockIdx.x;
    const int tid = threadIdx.x;
    const int L = lengths[b];
    if (L < 1 || L > Lmax) {
        if (tid == 0) atomicOr(err, ERR_LENGTH);
        return;
    }
    if (tid == 0) {
        mbar_init(bar, 1);
        fence_barrier_init();
    }
    __syncthreads();

    Aff carry = aff_identity();
    unsigned phase = 0;
    for (int r0 = 0; r0 < L; r0 += TILE) {
        const int n = min(TILE, L - r0);
        const int pre = r0 > 0 ? 1 : 0;
        // ---- stage angles [r0-pre, r0+n) with one bulk copy (+ edges)
        const Span sa = make_span(angles + ((size_t)b * Lmax + r0 - pre) * 3, (n + pre) * 12);
        if (tid == 0) {
            bulk_wait_read_all();  // previous tile's output staging may still be read by TMA
            mbar_arrive_expect_tx(bar, unsigned(sa.mid));
            span_load_bulk(sa, s_ang_base, bar);
        }
        span_load_edges_f32(sa, s_ang_base);
        mbar_wait(bar, phase);
        phase ^= 1u;
        __syncthreads();
        const float* s_ang = reinterpret_cast<const float*>(s_ang_base + sa.mis()) + 3 * pre;

        // ---- per-thread chunk: sequential compose from identity
        Aff M = aff_identity();
        float px[APT], py[APT], pz[APT];
        const int rl0 = tid * RPT;
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int rl = rl0 + q;
            const int j = r0 + rl;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                if (rl < n && (j | k) != 0) {
                    const float a = (k == 0) ? s_ang[3 * rl - 1] : s_ang[3 * rl + k - 1];
                    float s, c;
                    sincosf(a, &s, &c);
                    aff_bond(M, c, s, K.b[k]);
                }
                px[3 * q + k] = M.t0;
                py[3 * q + k] = M.t1;
                pz[3 * q + k] = M.t2;
            }
        }
        if (kOrtho) aff_orthonormalize(M);
        const Aff P = block_exclusive_scan<NT, kOrtho>(M, carry, scratch, s_total);
        carry = load_aff(s_total);

        // ---- global positions into the output staging buffer, then bulk store
        const Span so = make_span(coords + ((size_t)b * 3 * Lmax + 3 * (size_t)r0) * 3, n * 36);
        float* s_out = reinterpret_cast<float*>(s_out_base + so.mis());
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int rl = rl0 + q;
            if (rl < n) {
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    float x, y, z;
                    apply(P, px[3 * q + k], py[3 * q + k], pz[3 * q + k], x, y, z);
                    s_out[9 * rl + 3 * k + 0] = x;
                    s_out[9 * rl + 3 * k + 1] = y;
                    s_out[9 * rl + 3 * k + 2] = z;
                }
            }
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            span_store_bulk(so, s_out_base);
            bulk_commit();
        }
        span_store_edges_f32(so, s_out_base);
    }
    if (tid == 0) bulk_wait_all();
}

template <int NT, int RPT, bool kOrtho>
__global__ void __launch_bounds__(NT) bb_backward_kernel(const float* __restrict__ angles,
                                                         const int* __restrict__ lengths, int Lmax,
                                                         const float* __restrict__ grad_coords,
                                                         float* __restrict__ grad_angles, unsigned* __restrict__ err,
                                                         float* __restrict__ ws_prefix, int max_tiles, BBConst K) {
    constexpr int TILE = NT * RPT;
    constexpr int APT = 3 * RPT;
    using S = BBSmem<NT>;
    extern __shared__ __align__(16) char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::kBar);
    float* scratch = reinterpret_cast<float*>(smem + S::kScratch);
    float* s_total = reinterpret_cast<float*>(smem + S::kTotal);
    float* s_misc = reinterpret_cast<float*>(smem + S::kMisc);
    char* s_ang_base = smem + S::kData;
    char* s_g_base = s_ang_base + round16(16 + 12 * (TILE + 1));
    char* s_go_base = s_g_base + round16(16 + 36 * TILE);

    const int b = blockIdx.x;
    const int tid = threadIdx.x;
    const int L = lengths[b];
    if (L < 1 || L > Lmax) {
        if (tid == 0) atomicOr(err, ERR_LENGTH);
        return;
    }
    if (tid == 0) {
        mbar_init(bar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    const int n_tiles = (L + TILE - 1) / TILE;
    unsigned phase = 0;
    const int rl0 = tid * RPT;
    float* pref = ws_prefix + (size_t)b * max_tiles * 12;

    // ---- phase A: prefix transform at the start of every tile but the first
    if (n_tiles > 1) {
        Aff carry = aff_identity();
        for (int t = 0; t + 1 < n_tiles; ++t) {
            const int r0 = t * TILE;
            const int pre = r0 > 0 ? 1 : 0;
            const Span sa = make_span(angles + ((size_t)b * Lmax + r0 - pre) * 3, (TILE + pre) * 12);
            if (tid == 0) {
                mbar_arrive_expect_tx(bar, unsigned(sa.mid));
                span_load_bulk(sa, s_ang_base, bar);
            }
            span_load_edges_f32(sa, s_ang_base);
            mbar_wait(bar, phase);
            phase ^= 1u;
            __syncthreads();
            const float* s_ang = reinterpret_cast<const float*>(s_ang_base + sa.mis()) + 3 * pre;
            Aff M = aff_identity();
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const int rl = rl0 + q;
                const int j = r0 + rl;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    if ((j | k) != 0) {
                        const float a = (k == 0) ? s_ang[3 * rl - 1] : s_ang[3 * rl + k - 1];
                        float s, c;
                        sincosf(a, &s, &c);
                        aff_bond(M, c, s, K.b[k]);
                    }
                }
            }
            if (kOrtho) aff_orthonormalize(M);
            block_exclusive_scan<NT, kOrtho>(M, carry, scratch, s_total);
            carry = load_aff(s_total);
            if (tid < 12) pref[(t + 1) * 12 + tid] = s_total[tid];
        }
        __syncthreads();
    }

    // ---- phase B: tiles last to first
    float carry6[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float omega_next = 0.f;  // dL/d omega of the tile's last residue (from the later tile)
    for (int t = n_tiles - 1; t >= 0; --t) {
        const int r0 = t * TILE;
        const int n = min(TILE, L - r0);
        const int pre = r0 > 0 ? 1 : 0;
        const Aff carry = (t == 0) ? aff_identity() : load_aff(pref + t * 12);
        const Span sa = make_span(angles + ((size_t)b * Lmax + r0 - pre) * 3, (n + pre) * 12);
        const Span sg = make_span(grad_coords + ((size_t)b * 3 * Lmax + 3 * (size_t)r0) * 3, n * 36);
        if (tid == 0) {
            bulk_wait_read_all();
            mbar_arrive_expect_tx(bar, unsigned(sa.mid + sg.mid));
            span_load_bulk(sa, s_ang_base, bar);
            span_load_bulk(sg, s_g_base, bar);
        }
        span_load_edges_f32(sa, s_ang_base);
        span_load_edges_f32(sg, s_g_base);
        mbar_wait(bar, phase);
        phase ^= 1u;
        __syncthreads();
        const float* s_ang = reinterpret_cast<const float*>(s_ang_base + sa.mis()) + 3 * pre;
        const float* s_g = reinterpret_cast<const float*>(s_g_base + sg.mis());

        // local chunk: positions and rotation axes (x-axis of each frame)
        Aff M = aff_identity();
        float px[APT], py[APT], pz[APT], ex[APT], ey[APT], ez[APT];
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int rl = rl0 + q;
            const int j = r0 + rl;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                if (rl < n && (j | k) != 0) {
                    const float a = (k == 0) ? s_ang[3 * rl - 1] : s_ang[3 * rl + k - 1];
                    float s, c;
                    sincosf(a, &s, &c);
                    aff_bond(M, c, s, K.b[k]);
                }
                px[3 * q + k] = M.t0;
                py[3 * q + k] = M.t1;
                pz[3 * q + k] = M.t2;
                ex[3 * q + k] = M.r00;
                ey[3 * q + k] = M.r10;
                ez[3 * q + k] = M.r20;
            }
        }
        if (kOrtho) aff_orthonormalize(M);
        const Aff P = block_exclusive_scan<NT, kOrtho>(M, carry, scratch, s_total);

        // global r, e; per-thread sums S = sum g, T = sum r x g
        float sum6[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int a = 0; a < APT; ++a) {
            const int rl = rl0 + a / 3;
            float x, y, z;
            apply(P, px[a], py[a], pz[a], x, y, z);
            px[a] = x; py[a] = y; pz[a] = z;
            const float e0 = fmaf(P.r00, ex[a], fmaf(P.r01, ey[a], P.r02 * ez[a]));
            const float e1 = fmaf(P.r10, ex[a], fmaf(P.r11, ey[a], P.r12 * ez[a]));
            const float e2 = fmaf(P.r20, ex[a], fmaf(P.r21, ey[a], P.r22 * ez[a]));
            ex[a] = e0; ey[a] = e1; ez[a] = e2;
            if (rl < n) {
                const float g0 = s_g[9 * rl + 3 * (a % 3) + 0];
                const float g1 = s_g[9 * rl + 3 * (a % 3) + 1];
                const float g2 = s_g[9 * rl + 3 * (a % 3) + 2];
                sum6[0] += g0; sum6[1] += g1; sum6[2] += g2;
                sum6[3] += fmaf(y, g2, -z * g1);
                sum6[4] += fmaf(z, g0, -x * g2);
                sum6[5] += fmaf(x, g1, -y * g0);
            }
        }
        float suf[6], tot6[6];
        block_exclusive_suffix6<NT>(sum6, carry6, scratch, suf, tot6);

        // walk atoms last to first: grad alpha_i = e_i . (T - r_i x S)
        const Span so = make_span(grad_angles + ((size_t)b * Lmax + r0) * 3, n * 12);
        float* s_go = reinterpret_cast<float*>(s_go_base + so.mis());
#pragma unroll
        for (int a = APT - 1; a >= 0; --a) {
            const int q = a / 3, k = a % 3;
            const int rl = rl0 + q;
            const int j = r0 + rl;
            if (rl < n) {
                const float x = px[a], y = py[a], z = pz[a];
                const float c0 = suf[3] - fmaf(y, suf[2], -z * suf[1]);
                const float c1 = suf[4] - fmaf(z, suf[0], -x * suf[2]);
                const float c2 = suf[5] - fmaf(x, suf[1], -y * suf[0]);
                const float ga = fmaf(ex[a], c0, fmaf(ey[a], c1, ez[a] * c2));
                if (k == 1) s_go[3 * rl + 0] = ga;        // phi_j
                else if (k == 2) s_go[3 * rl + 1] = ga;   // psi_j
                else if (j > 0) {                          // omega_{j-1}
                    if (rl > 0) s_go[3 * (rl - 1) + 2] = ga;
                    else s_misc[0] = ga;                   // belongs to the previous tile
                }
                const float g0 = s_g[9 * rl + 3 * k + 0];
                const float g1 = s_g[9 * rl + 3 * k + 1];
                const float g2 = s_g[9 * rl + 3 * k + 2];
                suf[0] += g0; suf[1] += g1; suf[2] += g2;
                suf[3] += fmaf(y, g2, -z * g1);
                suf[4] += fmaf(z, g0, -x * g2);
                suf[5] += fmaf(x, g1, -y * g0);
            }
        }
        // omega of the tile's last residue: from the later tile, or a structural 0
        if (tid == 0) s_go[3 * (n - 1) + 2] = (r0 + n == L) ? 0.f : omega_next;
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            span_store_bulk(so, s_go_base);
            bulk_commit();
        }
        span_store_edges_f32(so, s_go_base);
        omega_next = s_misc[0];
#pragma unroll
        for (int k = 0; k < 6; ++k) carry6[k] = tot6[k];
        __syncthreads();
    }
    if (tid == 0) bulk_wait_all();
}

// ---------------------------------------------------------------------------
// Host-side launch helpers (called from capi.cu).

int bb_rpt_for(int Lmax) {
    int r = (Lmax + kBBThreads - 1) / kBBThreads;
    return r < 1 ? 1 : (r > 4 ? 4 : r);
}
int bb_tile_for(int Lmax) { return kBBThreads * bb_rpt_for(Lmax); }

size_t bb_forward_smem(int rpt) {
    const int tile = kBBThreads * rpt;
    return BBSmem<kBBThreads>::kData + round16(16 + 12 * (tile + 1)) + round16(16 + 36 * tile);
}
size_t bb_backward_smem(int rpt) {
    const int tile = kBBThreads * rpt;
    return BBSmem<kBBThreads>::kData + round16(16 + 12 * (tile + 1)) + round16(16 + 36 * tile) +
           round16(16 + 12 * tile);
}

template <int RPT, bool O>
static cudaError_t launch_fwd(const BBArgs& a, cudaStream_t st) {
    auto k = bb_forward_kernel<kBBThreads, RPT, O>;
    const size_t sm = bb_forward_smem(RPT);
    static size_t configured = 0;  // set the smem opt-in once per instance (not inside graph capture)
    if (configured < sm) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        if (e != cudaSuccess) return e;
        configured = sm;
    }
    k<<<a.B, kBBThreads, sm, st>>>(a.angles, a.lengths, a.Lmax, a.coords, a.err, a.K);
    return cudaGetLastError();
}
template <int RPT, bool O>
static cudaError_t launch_bwd(const BBArgs& a, cudaStream_t st) {
    auto k = bb_backward_kernel<kBBThreads, RPT, O>;
    const size_t sm = bb_backward_smem(RPT);
    static size_t configured = 0;  // set the smem opt-in once per instance (not inside graph capture)
    if (configured < sm) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        if (e != cudaSuccess) return e;
        configured = sm;
    }
    k<<<a.B, kBBThreads, sm, st>>>(a.angles, a.lengths, a.Lmax, a.grad_coords, a.grad_angles, a.err, a.ws_prefix,
                                   a.max_tiles, a.K);
    return cudaGetLastError();
}

cudaError_t bb_forward_launch(const BBArgs& a, cudaStream_t st) {
    const int r = bb_rpt_for(a.Lmax);
    if (a.ortho) {
        switch (r) {
            case 1: return launch_fwd<1, true>(a, st);
            case 2: return launch_fwd<2, true>(a, st);
            case 3: return launch_fwd<3, true>(a, st);
            default: return launch_fwd<4, true>(a, st);
        }
    }
    switch (r) {
        case 1: return launch_fwd<1, false>(a, st);
        case 2: return launch_fwd<2, false>(a, st);
        case 3: return launch_fwd<3, false>(a, st);
        default: return launch_fwd<4, false>(a, st);
    }
}

cudaError_t bb_backward_launch(const BBArgs& a, cudaStream_t st) {
    const int r = bb_rpt_for(a.Lmax);
    if (a.ortho) {
        switch (r) {
            case 1: return launch_bwd<1, true>(a, st);
            case 2: return launch_bwd<2, true>(a, st);
            case 3: return launch_bwd<3, true>(a, st);
            default: return launch_bwd<4, true>(a, st);
        }
    }
    switch (r) {
        case 1: return launch_bwd<1, false>(a, st);
        case 2: return launch_bwd<2, false>(a, st);
        case 3: return launch_bwd<3, false>(a, st);
        default: return launch_bwd<4, false>(a, st);
    }
}

}  // namespace tpl
