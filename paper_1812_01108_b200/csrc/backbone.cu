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
// one reverse suffix sum per chain: O(L) instead of the paper's O(L^2).  Two
// entry points: from the angles (bb_backward_kernel: the frames are recomputed,
// each thread in the local frame of its chunk) and from the forward's
// coordinates (bb_backward_xyz_kernel: e_i is the unit bond vector, no trig and
// no transform scan -- the path the autograd layer and the bench take).
//
// Work decomposition: a CTA of NT threads owns one chain at a time; a tile is
// NT*RPT residues; each thread handles RPT consecutive residues, one block-wide
// scan combines the chunks.  CTAs are persistent over chains (grid <= resident
// CTAs) and run a two-deep TMA pipeline: the next work item's tile is bulk-copied
// into the other shared-memory buffer while the current one is computed.
//   forward : every tile of every chain, first to last (prefix carried);
//   backward: from angles, phase A = tile prefixes of all but the last tile (to
//             the workspace), then phase B = tiles last to first (suffix
//             carried); from coordinates, tiles last to first only.
// Few long chains (f4): the *_dl_kernel variants put the tiles of a chain on
// different CTAs that exchange their aggregates through workspace slots.
// Fewer chains than about 1.4 x SMs of 641-1024 residues: the *_cl_kernel
// variants split each chain over a 2-CTA thread-block cluster that exchanges the
// part aggregates through distributed shared memory.
// Variants of the chain-serial kernels: chain segments over ranks (f4,
// segment.cu) and the fused LRMSD loss (f1, kLoss).
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "lrmsd_math.cuh"

namespace tpl {

template <int NT>
struct BBSmem {
    static constexpr int NW = NT / 32;
    static constexpr int kBar = 0;                         // 2 uint64 mbarriers (one per buffer)
    static constexpr int kScratch = 16;                    // 2*NW*12 floats (affine scan)
    static constexpr int kSuf = kScratch + 2 * NW * 12 * 4;  // 2*NW*6 + 8 floats (suffix scan)
    static constexpr int kTotal = kSuf + (2 * NW * 6 + 8) * 4;  // 12 floats
    static constexpr int kMisc = kTotal + 48;              // 16 floats of misc
    static constexpr int kData = ((kMisc + 64 + 15) / 16) * 16;
};

__host__ __device__ constexpr int round16(int x) { return (x + 15) & ~15; }
// __launch_bounds__ min-blocks so that ptxas keeps <= 128 registers/thread
// (2 CTAs of 256, 4 of 128, 16 of 32 threads per SM).
__host__ __device__ constexpr int kMinBlocks128Regs(int nt) { return 65536 / (nt * 128); }

// The three transforms of residue j (local index rl in the staged tile):
// k = 0: C_{j-1} -> N_j by omega_{j-1} (identity for j = 0, reading Q1),
// k = 1: N_j -> CA_j by phi_j, k = 2: CA_j -> C_j by psi_j.
// kSlow = false: branch-free hot path, |angle| folded into *maxabs; the caller
// redoes the tile with kSlow = true if any |angle| > kSinCosFastMax.
template <bool kSlow>
__device__ __forceinline__ void bb_residue_trig(const float* s_ang, int rl, int j, float (&c)[3], float (&s)[3],
                                                float* maxabs, float om0 = 0.f) {
    // om0: omega_{-1} of a chain segment that continues an earlier one (f4)
    const float x[3] = {j > 0 ? s_ang[3 * rl - 1] : om0, s_ang[3 * rl + 0], s_ang[3 * rl + 1]};
    if (kSlow) tpl_sincos_n<3>(x, s, c);
    else tpl_sincos_hot<3>(x, s, c, maxabs);
}

// ---------------------------------------------------------------------------
// Work-item iterator of one CTA (every thread computes the same sequence).
// Chains b = blockIdx.x, blockIdx.x + gridDim.x, ...; the length of the next
// chain is loaded one chain ahead so the prefetch never waits for it.
struct BBIter {
    const int* lengths;
    int B, Lmax, tile, stride;
    bool fwd;
    unsigned* err;
    bool skipA;        // backward without phase A (the prefix is not needed)
    int b, L, bn, Ln;  // current chain and the next one
    int t, nt, phase;  // tile, tiles in chain, 0 = fwd/phase A, 1 = phase B
    bool valid;

    __device__ int load_len(int c) const { return c < B ? __ldg(lengths + c) : 0; }
    __device__ void next_chain() {
        b = bn;
        L = Ln;
        bn = b + stride;
        Ln = load_len(bn);
    }
    __device__ void start_chain() {  // skips invalid chains (flagged), sets the first tile
        while (b < B && (L < 1 || L > Lmax)) {
            if (threadIdx.x == 0) atomicOr(err, ERR_LENGTH);
            next_chain();
        }
        valid = b < B;
        if (!valid) return;
        nt = (L + tile - 1) / tile;
        phase = fwd ? 0 : ((nt == 1 || skipA) ? 1 : 0);
        t = (!fwd && phase == 1) ? nt - 1 : 0;
    }
    __device__ void init() {
        b = blockIdx.x;
        L = load_len(b);
        bn = b + stride;
        Ln = load_len(bn);
        start_chain();
    }
    __device__ void advance() {
        if (fwd) {
            if (t + 1 < nt) { ++t; return; }
        } else if (phase == 0) {
            if (t + 1 < nt - 1) ++t;
            else { phase = 1; t = nt - 1; }
            return;
        } else if (t > 0) {
            --t;
            return;
        }
        next_chain();
        start_chain();
    }
    __device__ int r0() const { return t * tile; }
    __device__ int n() const { return min(tile, L - t * tile); }
};

// ---------------------------------------------------------------------------
// Work items of the decoupled ("DL") kernels: every (chain, tile) pair is an
// item, i = b * max_tiles + (fwd ? t : max_tiles - 1 - t), dealt round-robin
// to a co-resident persistent grid.  An item only waits for items with a
// smaller index (earlier tiles in the forward, later tiles in the backward),
// so the smallest unfinished item can always proceed: tiles of one chain run
// on different SMs at the same time and exchange only their aggregates.
struct DLIter {
    const int* lengths;
    int B, Lmax, tile, max_tiles, stride;
    bool fwd;
    unsigned* err;
    int i, b, L, t, nt;
    bool valid;
    static constexpr int phase = 1;  // for bb_issue: a backward item always loads dL/dr

    __device__ void settle() {
        const int n_items = B * max_tiles;
        int cb = -1, cL = 0;
        for (; i < n_items; i += stride) {
            const int bb = i / max_tiles, tr = i - bb * max_tiles;
            if (bb != cb) {
                cb = bb;
                cL = __ldg(lengths + bb);
            }
            if (cL < 1 || cL > Lmax) {
                if (tr == 0 && threadIdx.x == 0) atomicOr(err, ERR_LENGTH);
                continue;
            }
            const int ntt = (cL + tile - 1) / tile;
            const int tt = fwd ? tr : max_tiles - 1 - tr;
            if (tt < ntt) {
                b = bb;
                L = cL;
                t = tt;
                nt = ntt;
                valid = true;
                return;
            }
        }
        valid = false;
    }
    __device__ void init() {
        i = blockIdx.x;
        settle();
    }
    __device__ void advance() {
        i += stride;
        settle();
    }
    __device__ int r0() const { return t * tile; }
    __device__ int n() const { return min(tile, L - t * tile); }
};

// Issue (thread 0) the bulk copies of one work item into buffer `buf`.
template <typename It>
__device__ __forceinline__ void bb_issue(const It& it, const float* angles, const float* grad_coords,
                                         char* s_ang, char* s_g, uint64_t* bar) {
    const int r0 = it.r0(), n = it.n(), pre = r0 > 0 ? 1 : 0;
    const Span sa = make_span(angles + ((size_t)it.b * it.Lmax + r0 - pre) * 3, (n + pre) * 12);
    unsigned bytes = unsigned(sa.mid);
    Span sg{};
    const bool with_g = grad_coords && it.phase == 1;
    if (with_g) {
        sg = make_span(grad_coords + ((size_t)it.b * 3 * it.Lmax + 3 * (size_t)r0) * 3, n * 36);
        bytes += unsigned(sg.mid);
    }
    mbar_arrive_expect_tx(bar, bytes);
    span_load_bulk(sa, s_ang, bar);
    if (with_g) span_load_bulk(sg, s_g, bar);
}

// Segment mode (f4, both pointers non-null): chain b continues an earlier
// segment, so its residue 0 carries the omega bond omega_prev[b] from an
// identity frame (the previous segment's last C), and the chain's aggregate
// transform is written to agg_out[b][12] for the exchange between ranks.
// kLoss (f1, fused LRMSD): the target tile is bulk-loaded beside the output, the
// chain's raw fp64 moments (sum x, sum y, sum x y^T, sum |x|^2, sum |y|^2; PAPER
// §4 step 1) are reduced over its tiles, and at the chain's end thread
// 0 solves steps 2-3 (lrmsd_math.cuh) into loss_out[b] and loss_state[b][16].
// The kLoss variant is compiled for 2 CTAs/SM (up to 255 registers): capped at
// 128 it spilled the 17 fp64 moment accumulators (fused step 25.0 -> 20.5 us).
// kMinB overrides the CTAs/SM the registers are sized for (the launcher picks 2
// for 128 x 7 when the chains fit two per SM: 256 x 700 fwd 6.80 -> 6.61 us).
template <int NT, int RPT, int kNS, bool kLoss = false, int kMinB = 0>
__global__ void __launch_bounds__(NT, kMinB > 0 ? kMinB : (kLoss ? 2 : kMinBlocks128Regs(NT))) bb_forward_kernel(const float* __restrict__ angles,
                                                        const int* __restrict__ lengths, int B, int Lmax,
                                                        float* __restrict__ coords, unsigned* __restrict__ err,
                                                        const float* __restrict__ omega_prev,
                                                        float* __restrict__ agg_out,
                                                        const float* __restrict__ target,
                                                        float* __restrict__ loss_out,
                                                        float* __restrict__ loss_state) {
    constexpr int TILE = NT * RPT;
    constexpr int ANG = round16(16 + 12 * (TILE + 1));
    constexpr int OUT = round16(16 + 36 * TILE);
    using S = BBSmem<NT>;
    extern __shared__ __align__(16) char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::kBar);
    float* scratch = reinterpret_cast<float*>(smem + S::kScratch);
    float* s_total = reinterpret_cast<float*>(smem + S::kTotal);
    char* s_ang_buf = smem + S::kData;  // 2 x ANG
    char* s_out_base = s_ang_buf + 2 * ANG;
    char* s_tgt_base = s_out_base + OUT;                                            // kLoss: target tile
    double* s_mred = reinterpret_cast<double*>(s_tgt_base + OUT);                   // kLoss: 17 x NT partials
    double* s_macc = s_mred + 17 * NT;                                              // kLoss: the chain's moments
    uint64_t* bar_t = reinterpret_cast<uint64_t*>(s_macc + 18);                     // kLoss

    const int tid = threadIdx.x;
    TPL_STAMP(0);
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        if (kLoss) mbar_init(bar_t, 1);
        fence_barrier_init();
    }
    unsigned tphase = 0;
    pdl_wait();
    // Speculative first load: when every chain fits one tile, the CTA's first
    // chain is bulk-loaded whole (Lmax residues) before its length arrives, so
    // the lengths load no longer precedes the TMA on the critical path.
    const bool spec = !kLoss && Lmax <= TILE && int(blockIdx.x) < B;
    if (tid == 0 && spec) {
        const Span s0 = make_span(angles + (size_t)blockIdx.x * Lmax * 3, Lmax * 12);
        mbar_arrive_expect_tx(bar, unsigned(s0.mid));
        span_load_bulk(s0, s_ang_buf, bar);
    }
    BBIter it{lengths, B, Lmax, TILE, int(gridDim.x), true, err, false};
    it.init();
    TPL_STAMP(1);
    __syncthreads();
    const bool spec_hit = spec && it.valid && it.b == int(blockIdx.x);
    unsigned phases = 0;  // bit k = parity of buffer k
    if (spec && !spec_hit) {  // first chain invalid: drain the speculative copy
        if (tid == 0) mbar_wait(bar, 0);
        phases ^= 1u;
    }
    if (tid == 0 && it.valid && !spec_hit) bb_issue(it, angles, nullptr, s_ang_buf, nullptr, bar);

    Aff carry = aff_identity();
    const int rl0 = tid * RPT;
    for (int k = 0; it.valid; ++k) {
        const int buf = k & 1;
        const int b = it.b, L = it.L, r0 = it.r0(), n = it.n(), pre = r0 > 0 ? 1 : 0;
        const int nl = (k == 0 && spec_hit) ? Lmax : n;  // residues the copy covers
        if (r0 == 0) carry = aff_identity();
        BBIter nx = it;
        nx.advance();
        if (tid == 0 && nx.valid) bb_issue(nx, angles, nullptr, s_ang_buf + (buf ^ 1) * ANG, nullptr, bar + (buf ^ 1));
        // ---- angles [r0-pre, r0+n): bulk part by TMA, <16-byte edges by threads
        char* s_ang_base = s_ang_buf + buf * ANG;
        const Span sa = make_span(angles + ((size_t)b * Lmax + r0 - pre) * 3, (nl + pre) * 12);
        span_load_edges_f32(sa, s_ang_base);
        const Span so = make_span(coords + ((size_t)b * 3 * Lmax + 3 * (size_t)r0) * 3, n * 36);
        float* s_out = reinterpret_cast<float*>(s_out_base + so.mis());
        Span stg{};
        if (kLoss) {  // the target tile (single buffer: the previous item's moments pass is done)
            stg = make_span(target + ((size_t)b * 3 * Lmax + 3 * (size_t)r0) * 3, n * 36);
            if (tid == 0) {
                mbar_arrive_expect_tx(bar_t, unsigned(stg.mid));
                span_load_bulk(stg, s_tgt_base, bar_t);
            }
            span_load_edges_f32(stg, s_tgt_base);
            if (r0 == 0 && tid < 17) s_macc[tid] = 0.0;  // read after the moments pass's barrier
        }
        TPL_STAMP(2);
        mbar_wait(bar + buf, (phases >> buf) & 1u);
        phases ^= 1u << buf;
        __syncthreads();
        TPL_STAMP(3);
        const float* s_ang = reinterpret_cast<const float*>(s_ang_base + sa.mis()) + 3 * pre;
        const bool seg0 = omega_prev != nullptr && r0 == 0;  // residue 0 continues a segment
        const float om0 = seg0 ? __ldg(omega_prev + b) : 0.f;

        // ---- pass 1: the thread's chunk composed from the identity; local
        //      atom positions stay in registers (RPT is small and odd, so the
        //      strided shared-memory accesses below are bank-conflict free)
        Aff M;
        const int nq = max(0, min(RPT, n - rl0));
        float px[3 * RPT], py[3 * RPT], pz[3 * RPT];
        float maxabs = 0.f;
        auto pass1 = [&](auto slow) {
            constexpr bool kSlow = decltype(slow)::value;
            M = aff_identity();
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                if (q < nq) {
                    const int rl = rl0 + q;
                    float c[3], s[3];
                    bb_residue_trig<kSlow>(s_ang, rl, r0 + rl, c, s, &maxabs, om0);
                    if (r0 + rl > 0 || seg0) aff_bond_bb_x2<0>(M, c[0], s[0]);
                    px[3 * q] = M.t0; py[3 * q] = M.t1; pz[3 * q] = M.t2;
                    aff_bond_bb_x2<1>(M, c[1], s[1]);
                    px[3 * q + 1] = M.t0; py[3 * q + 1] = M.t1; pz[3 * q + 1] = M.t2;
                    aff_bond_bb_x2<2>(M, c[2], s[2]);
                    px[3 * q + 2] = M.t0; py[3 * q + 2] = M.t1; pz[3 * q + 2] = M.t2;
                }
            }
        };
        pass1(std::false_type{});
        // rare: huge angles.  pass 1 is thread-local, so the redo is decided per warp (a
        // warp-uniform branch, no block barrier: the block scan below synchronises)
        if (__any_sync(0xffffffffu, maxabs > kSinCosFastMax)) pass1(std::true_type{});
        if (kNS >= 1) aff_orthonormalize(M);
        if ((tid & 31) == 0) bulk_wait_read_all();  // the output staging is free again (per-warp groups)
        TPL_STAMP(4);
        const Aff P = block_exclusive_scan<NT, kNS>(M, carry, scratch, s_total);
        carry = load_aff(s_total);
        if (agg_out != nullptr && r0 + n == L && tid < 12) agg_out[(size_t)b * 12 + tid] = s_total[tid];
        // Let the next kernel launch only now: dependents launched earlier sit on
        // SM resources while waiting and slowed alternating fwd/bwd by ~3 us.
        if (!nx.valid) pdl_trigger();
        TPL_STAMP(5);

        // ---- pass 2: chunk prefix applied, positions to the output staging buffer
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            if (q < nq) {
                float* o = s_out + 9 * (rl0 + q);
#pragma unroll
                for (int kk = 0; kk < 3; ++kk) {
                    const int a = 3 * q + kk;
                    apply(P, px[a], py[a], pz[a], o[3 * kk], o[3 * kk + 1], o[3 * kk + 2]);
                }
            }
        }
        TPL_STAMP(6);
        fence_proxy_async_smem();
        if (kLoss) {
            __syncthreads();
            if (tid == 0) {
                span_store_bulk(so, s_out_base);
                bulk_commit();
            }
            span_store_edges_f32(so, s_out_base);
        } else {
            // per-warp stores: a warp's residues are contiguous, so each warp sends its
            // own chunk as soon as its lanes are done (no block barrier); the chunk
            // starts 36 * 32 * RPT bytes apart, so shared and global keep the same
            // 16-byte phase
            __syncwarp();
            const int lane = tid & 31, w0 = (tid >> 5) * 32 * RPT, wn = min(32 * RPT, n - w0);
            if (wn > 0) {
                const Span sw = make_span(coords + ((size_t)b * 3 * Lmax + 3 * (size_t)(r0 + w0)) * 3, wn * 36);
                const float* src = s_out + 9 * w0;
                if (lane == 0 && sw.mid > 0) {
                    bulk_s2g(const_cast<char*>(sw.g) + sw.head, reinterpret_cast<const char*>(src) + sw.head,
                             unsigned(sw.mid));
                    bulk_commit();
                }
                float* g = reinterpret_cast<float*>(const_cast<char*>(sw.g));
                const int nh = sw.head >> 2, ntl = sw.tail() >> 2, off_t = (sw.head + sw.mid) >> 2;
                for (int e = lane; e < nh + ntl; e += 32) {
                    const int idx = e < nh ? e : off_t + (e - nh);
                    g[idx] = src[idx];
                }
            }
        }
        TPL_STAMP(7);
        if (kLoss) {  // moments of (x, y) over the tile's atoms, fp64
            mbar_wait(bar_t, tphase);
            tphase ^= 1u;
            __syncthreads();  // the target edges are in place
            const float* xo = s_out;
            const float* yo = reinterpret_cast<const float*>(s_tgt_base + stg.mis());
            double m[17];
#pragma unroll
            for (int q = 0; q < 17; ++q) m[q] = 0.0;
            for (int a = tid; a < 3 * n; a += NT) {
                const double x0 = xo[3 * a], x1 = xo[3 * a + 1], x2 = xo[3 * a + 2];
                const double y0 = yo[3 * a], y1 = yo[3 * a + 1], y2 = yo[3 * a + 2];
                m[0] += x0; m[1] += x1; m[2] += x2;
                m[3] += y0; m[4] += y1; m[5] += y2;
                m[6] += x0 * y0; m[7] += x0 * y1; m[8] += x0 * y2;
                m[9] += x1 * y0; m[10] += x1 * y1; m[11] += x1 * y2;
                m[12] += x2 * y0; m[13] += x2 * y1; m[14] += x2 * y2;
                m[15] += x0 * x0 + x1 * x1 + x2 * x2;
                m[16] += y0 * y0 + y1 * y1 + y2 * y2;
            }
            // transposed reduction (fixed order): every thread parks its 17 partials, then
            // warp w folds moments w, w + NW, ... (NT/32 values per lane, then a shuffle tree)
            const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
            for (int q = 0; q < 17; ++q) s_mred[q * NT + tid] = m[q];
            __syncthreads();
            for (int q = warp; q < 17; q += NT / 32) {
                double v = 0.0;
#pragma unroll
                for (int k = 0; k < NT / 32; ++k) v += s_mred[q * NT + lane + 32 * k];
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
                if (lane == 0) s_macc[q] += v;
            }
            __syncthreads();
            if (tid == 0 && r0 + n == L) lrmsd_solve(s_macc, 3.0 * L, loss_out + b, loss_state + (size_t)b * 16);
        }
        (void)L;
        it = nx;
    }
    TPL_STAMP(8);
    // Only the shared-memory source must outlive the CTA; grid completion (and the
    // dependent's griddepcontrol.wait) covers visibility of the global writes.
    if ((tid & 31) == 0) bulk_wait_read_all();
    TPL_STAMP(9);
}

// Cluster-split forward: one cluster of CL CTAs per chain, CTA rank c takes
// the residues [c h, (c + 1) h) with h = ceil(L / CL).  Every CTA scans its
// part from the identity; its aggregate A_c goes to the shared memory of each
// later CTA of the cluster (st.shared::cluster + a remote mbarrier arrival),
// and CTA r places its part with C_r = N(..N(A_0 A_1)..A_{r-1}) composed in
// rank order (deterministic).  Halves (CL = 2) the serial pass-1 chain of a
// chain-per-CTA launch when chains are about as many as SMs.  Chains up to
// CL * NT * RPT residues.
template <int NT, int RPT, int CL, int kNS>
__global__ void __launch_bounds__(NT, kMinBlocks128Regs(NT)) bb_forward_cl_kernel(const float* __restrict__ angles,
                                                           const int* __restrict__ lengths, int B, int Lmax,
                                                           float* __restrict__ coords, unsigned* __restrict__ err) {
    constexpr int TILE = NT * RPT;
    constexpr int ANG = round16(16 + 12 * (TILE + 1));
    constexpr int SLOTS = round16(48 * CL);
    using S = BBSmem<NT>;
    extern __shared__ __align__(16) char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::kBar);  // [0] angles TMA, [1] carries
    float* scratch = reinterpret_cast<float*>(smem + S::kScratch);
    float* s_total = reinterpret_cast<float*>(smem + S::kTotal);
    float* s_slots = reinterpret_cast<float*>(smem + S::kData);  // A_c of earlier ranks c
    char* s_ang_base = smem + S::kData + SLOTS;
    char* s_out_base = s_ang_base + ANG;

    const int tid = threadIdx.x;
    const unsigned rank = cluster_ctarank();
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, rank > 0 ? rank : 1);
        fence_mbarrier_init_cluster();
    }
    __syncthreads();
    cluster_arrive_relaxed();  // the carry barriers are initialised
    pdl_wait();
    const int b = blockIdx.x / CL;
    // speculative part load assuming L = Lmax (uniform batches), issued before the
    // length arrives; it is used whenever it covers the actual part
    const int hs = (Lmax + CL - 1) / CL, r0s = int(rank) * hs, ns = min(hs, Lmax - r0s), pres = r0s > 0 ? 1 : 0;
    const bool spec = ns > 0 && b < B;
    const Span ss = make_span(angles + ((size_t)b * Lmax + r0s - pres) * 3, (ns + pres) * 12);
    if (tid == 0 && spec) {
        mbar_arrive_expect_tx(bar, unsigned(ss.mid));
        span_load_bulk(ss, s_ang_base, bar);
    }
    const int L = b < B ? __ldg(lengths + b) : 0;
    if (L < 1 || L > Lmax) {
        if (tid == 0 && rank == 0 && b < B) atomicOr(err, ERR_LENGTH);
        if (tid == 0 && spec) mbar_wait(bar, 0);  // no bulk copy may outlive the CTA
        return;
    }
    const int h = (L + CL - 1) / CL, r0 = int(rank) * h, n = min(h, L - r0);
    if (n <= 0) {  // no earlier CTA sends to an empty part
        if (tid == 0 && spec) mbar_wait(bar, 0);
        return;
    }
    const int pre = r0 > 0 ? 1 : 0;
    const bool hit = spec && r0 == r0s && n <= ns;
    unsigned ph = 0;
    const Span sa = hit ? ss : make_span(angles + ((size_t)b * Lmax + r0 - pre) * 3, (n + pre) * 12);
    if (!hit) {
        if (tid == 0) {
            if (spec) mbar_wait(bar, 0);  // drain the speculative copy before refilling the buffer
            mbar_arrive_expect_tx(bar, unsigned(sa.mid));
            span_load_bulk(sa, s_ang_base, bar);
        }
        if (spec) ph = 1;
    }
    span_load_edges_f32(sa, s_ang_base);
    const Span so = make_span(coords + ((size_t)b * 3 * Lmax + 3 * (size_t)r0) * 3, n * 36);
    float* s_out = reinterpret_cast<float*>(s_out_base + so.mis());
    mbar_wait(bar, ph);
    __syncthreads();
    // every CTA of the cluster has initialised its carry barrier (they arrived
    // right after the init, so this wait is short).  All threads, warp-aligned:
    // a lone thread's non-aligned barrier.cluster.wait in a divergent branch hung.
    cluster_wait_aligned();
    const float* s_ang = reinterpret_cast<const float*>(s_ang_base + sa.mis()) + 3 * pre;

    // ---- pass 1 (as bb_forward_kernel)
    const int rl0 = tid * RPT;
    Aff M;
    const int nq = max(0, min(RPT, n - rl0));
    float px[3 * RPT], py[3 * RPT], pz[3 * RPT];
    float maxabs = 0.f;
    auto pass1 = [&](auto slow) {
        constexpr bool kSlow = decltype(slow)::value;
        M = aff_identity();
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            if (q < nq) {
                const int rl = rl0 + q;
                float c[3], s[3];
                bb_residue_trig<kSlow>(s_ang, rl, r0 + rl, c, s, &maxabs);
                if (r0 + rl > 0) aff_bond_bb<0>(M, c[0], s[0]);
                px[3 * q] = M.t0; py[3 * q] = M.t1; pz[3 * q] = M.t2;
                aff_bond_bb<1>(M, c[1], s[1]);
                px[3 * q + 1] = M.t0; py[3 * q + 1] = M.t1; pz[3 * q + 1] = M.t2;
                aff_bond_bb<2>(M, c[2], s[2]);
                px[3 * q + 2] = M.t0; py[3 * q + 2] = M.t1; pz[3 * q + 2] = M.t2;
            }
        }
    };
    pass1(std::false_type{});
    if (__any_sync(0xffffffffu, maxabs > kSinCosFastMax)) pass1(std::true_type{});  // rare: huge angles (per warp)
    if (kNS >= 1) aff_orthonormalize(M);
    Aff P = block_exclusive_scan<NT, kNS>(M, aff_identity(), scratch, s_total);  // part-local prefix
    // ---- exchange: A_rank to every later non-empty part of the chain
    if (tid == 0 && r0 + n < L) {
        const float* A = s_total;
        for (int r = int(rank) + 1; r < CL && r * h < L; ++r) {
            const uint32_t dst = mapa_shared(smem_u32(s_slots + 12 * rank), unsigned(r));
            st_cluster_v4(dst, A[0], A[1], A[2], A[3]);
            st_cluster_v4(dst + 16, A[4], A[5], A[6], A[7]);
            st_cluster_v4(dst + 32, A[8], A[9], A[10], A[11]);
            mbar_arrive_remote(mapa_shared(smem_u32(bar + 1), unsigned(r)));
        }
    }
    if (rank > 0) {
        mbar_wait_cluster(bar + 1, 0);
        Aff C = load_aff(s_slots);
        for (int c = 1; c < int(rank); ++c) {
            C = aff_compose(C, load_aff(s_slots + 12 * c));
            if (kNS >= 1) aff_orthonormalize(C);
        }
        P = aff_compose(C, P);
        if (kNS >= 1) aff_orthonormalize(P);
    }
    pdl_trigger();
    // ---- pass 2
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        if (q < nq) {
            float* o = s_out + 9 * (rl0 + q);
#pragma unroll
            for (int kk = 0; kk < 3; ++kk) {
                const int a = 3 * q + kk;
                apply(P, px[a], py[a], pz[a], o[3 * kk], o[3 * kk + 1], o[3 * kk + 2]);
            }
        }
    }
    fence_proxy_async_smem();
    __syncwarp();
    {  // per-warp stores (as bb_forward_kernel)
        const int lane = tid & 31, w0 = (tid >> 5) * 32 * RPT, wn = min(32 * RPT, n - w0);
        if (wn > 0) {
            const Span sw = make_span(coords + ((size_t)b * 3 * Lmax + 3 * (size_t)(r0 + w0)) * 3, wn * 36);
            const float* src = s_out + 9 * w0;
            if (lane == 0 && sw.mid > 0) {
                bulk_s2g(const_cast<char*>(sw.g) + sw.head, reinterpret_cast<const char*>(src) + sw.head,
                         unsigned(sw.mid));
                bulk_commit();
            }
            float* g = reinterpret_cast<float*>(const_cast<char*>(sw.g));
            const int nh = sw.head >> 2, ntl = sw.tail() >> 2, off_t = (sw.head + sw.mid) >> 2;
            for (int e = lane; e < nh + ntl; e += 32) {
                const int idx = e < nh ? e : off_t + (e - nh);
                g[idx] = src[idx];
            }
        }
        if (lane == 0) bulk_wait_read_all();
    }
}

// Decoupled forward: each (chain, tile) item scans its tile from the identity,
// publishes the tile aggregate A_t (unless it is the chain's last tile) and
// takes its prefix C_t = N(...N(N(A_0) A_1)... A_{t-1}) from the published
// aggregates in a fixed order (bitwise deterministic; N = Newton-Schulz).
// Slots: [B][max_tiles] x 16 floats (12 payload + flag) after the header.
template <int NT, int RPT, int kNS>
__global__ void __launch_bounds__(NT, kMinBlocks128Regs(NT)) bb_forward_dl_kernel(const float* __restrict__ angles,
                                                           const int* __restrict__ lengths, int B, int Lmax,
                                                           float* __restrict__ coords, unsigned* __restrict__ hdr,
                                                           float* __restrict__ slots, int max_tiles) {
    constexpr int TILE = NT * RPT;
    constexpr int ANG = round16(16 + 12 * (TILE + 1));
    using S = BBSmem<NT>;
    extern __shared__ __align__(16) char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::kBar);
    float* scratch = reinterpret_cast<float*>(smem + S::kScratch);
    float* s_total = reinterpret_cast<float*>(smem + S::kTotal);
    float* s_pre = reinterpret_cast<float*>(smem + S::kMisc);  // the tile's prefix C_t
    char* s_ang_buf = smem + S::kData;  // 2 x ANG
    char* s_out_base = s_ang_buf + 2 * ANG;

    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        fence_barrier_init();
    }
    pdl_wait();
    const unsigned fv = launch_epoch(hdr) + 1u;
    DLIter it{lengths, B, Lmax, TILE, max_tiles, int(gridDim.x), true, hdr};
    it.init();
    __syncthreads();
    if (tid == 0 && it.valid) bb_issue(it, angles, nullptr, s_ang_buf, nullptr, bar);

    unsigned phases = 0;
    const int rl0 = tid * RPT;
    for (int k = 0; it.valid; ++k) {
        const int buf = k & 1;
        const int b = it.b, r0 = it.r0(), n = it.n(), t = it.t, pre = r0 > 0 ? 1 : 0;
        DLIter nx = it;
        nx.advance();
        if (tid == 0 && nx.valid) bb_issue(nx, angles, nullptr, s_ang_buf + (buf ^ 1) * ANG, nullptr, bar + (buf ^ 1));
        char* s_ang_base = s_ang_buf + buf * ANG;
        const Span sa = make_span(angles + ((size_t)b * Lmax + r0 - pre) * 3, (n + pre) * 12);
        span_load_edges_f32(sa, s_ang_base);
        const Span so = make_span(coords + ((size_t)b * 3 * Lmax + 3 * (size_t)r0) * 3, n * 36);
        float* s_out = reinterpret_cast<float*>(s_out_base + so.mis());
        mbar_wait(bar + buf, (phases >> buf) & 1u);
        phases ^= 1u << buf;
        __syncthreads();
        const float* s_ang = reinterpret_cast<const float*>(s_ang_base + sa.mis()) + 3 * pre;

        Aff M;
        const int nq = max(0, min(RPT, n - rl0));
        float px[3 * RPT], py[3 * RPT], pz[3 * RPT];
        float maxabs = 0.f;
        auto pass1 = [&](auto slow) {
            constexpr bool kSlow = decltype(slow)::value;
            M = aff_identity();
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                if (q < nq) {
                    const int rl = rl0 + q;
                    float c[3], s[3];
                    bb_residue_trig<kSlow>(s_ang, rl, r0 + rl, c, s, &maxabs);
                    if (r0 + rl > 0) aff_bond_bb<0>(M, c[0], s[0]);
                    px[3 * q] = M.t0; py[3 * q] = M.t1; pz[3 * q] = M.t2;
                    aff_bond_bb<1>(M, c[1], s[1]);
                    px[3 * q + 1] = M.t0; py[3 * q + 1] = M.t1; pz[3 * q + 1] = M.t2;
                    aff_bond_bb<2>(M, c[2], s[2]);
                    px[3 * q + 2] = M.t0; py[3 * q + 2] = M.t1; pz[3 * q + 2] = M.t2;
                }
            }
        };
        pass1(std::false_type{});
        if (__any_sync(0xffffffffu, maxabs > kSinCosFastMax)) pass1(std::true_type{});  // rare: huge angles (per warp)
        if (kNS >= 1) aff_orthonormalize(M);
        if (tid == 0) bulk_wait_read_all();  // the output staging is free again
        Aff P = block_exclusive_scan<NT, kNS>(M, aff_identity(), scratch, s_total);  // tile-local prefix
        if (t > 0 || it.nt > 1) {
            if (tid == 0) {
                float* slot = slots + ((size_t)b * max_tiles + t) * 16;
                if (t + 1 < it.nt) {  // publish A_t for the later tiles
#pragma unroll
                    for (int q = 0; q < 12; ++q) slot[q] = s_total[q];
                    __threadfence();
                    st_release_gpu(reinterpret_cast<unsigned*>(slot + 12), fv);
                }
                Aff C = aff_identity();
                for (int u = 0; u < t; ++u) {  // fixed order: deterministic rounding
                    const float* su = slots + ((size_t)b * max_tiles + u) * 16;
                    wait_flag(reinterpret_cast<const unsigned*>(su + 12), fv);
                    Aff A;
                    A.r00 = __ldcg(su + 0); A.r01 = __ldcg(su + 1); A.r02 = __ldcg(su + 2); A.t0 = __ldcg(su + 3);
                    A.r10 = __ldcg(su + 4); A.r11 = __ldcg(su + 5); A.r12 = __ldcg(su + 6); A.t1 = __ldcg(su + 7);
                    A.r20 = __ldcg(su + 8); A.r21 = __ldcg(su + 9); A.r22 = __ldcg(su + 10); A.t2 = __ldcg(su + 11);
                    C = aff_compose(C, A);
                    if (kNS >= 1) aff_orthonormalize(C);
                }
                store_aff(s_pre, C);
            }
            __syncthreads();
            if (t > 0) {
                P = aff_compose(load_aff(s_pre), P);
                if (kNS >= 1) aff_orthonormalize(P);
            }
        }
        if (!nx.valid) pdl_trigger();

        // pass 2: prefix applied, positions to the output staging buffer
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            if (q < nq) {
                float* o = s_out + 9 * (rl0 + q);
#pragma unroll
                for (int kk = 0; kk < 3; ++kk) {
                    const int a = 3 * q + kk;
                    apply(P, px[a], py[a], pz[a], o[3 * kk], o[3 * kk + 1], o[3 * kk + 2]);
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
        it = nx;
    }
    __syncthreads();
    if (tid == 0) {
        bulk_wait_read_all();
        finish_epoch(hdr);
    }
}

template <int NT, int RPT, int kNS>
__global__ void __launch_bounds__(NT, kMinBlocks128Regs(NT)) bb_backward_kernel(const float* __restrict__ angles,
                                                         const int* __restrict__ lengths, int B, int Lmax,
                                                         const float* __restrict__ grad_coords,
                                                         float* __restrict__ grad_angles, unsigned* __restrict__ err,
                                                         float* __restrict__ ws_prefix, int max_tiles) {
    constexpr int TILE = NT * RPT;
    constexpr int ANG = round16(16 + 12 * (TILE + 1));
    constexpr int GB = round16(16 + 36 * TILE);
    using S = BBSmem<NT>;
    extern __shared__ __align__(16) char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::kBar);
    float* scratch = reinterpret_cast<float*>(smem + S::kScratch);
    float* s_suf = reinterpret_cast<float*>(smem + S::kSuf);
    float* s_total = reinterpret_cast<float*>(smem + S::kTotal);
    float* s_misc = reinterpret_cast<float*>(smem + S::kMisc);
    char* s_ang_buf = smem + S::kData;    // 2 x ANG
    char* s_g_buf = s_ang_buf + 2 * ANG;  // 2 x GB
    char* s_go_base = s_g_buf + 2 * GB;

    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        fence_barrier_init();
    }
    pdl_wait();
    BBIter it{lengths, B, Lmax, TILE, int(gridDim.x), false, err, false};
    it.init();
    __syncthreads();
    if (tid == 0 && it.valid) bb_issue(it, angles, grad_coords, s_ang_buf, s_g_buf, bar);

    unsigned phases = 0;
    const int rl0 = tid * RPT;
    Aff carryA = aff_identity();                        // phase A prefix carry
    float carry6[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // phase B suffix carry
    float omega_next = 0.f;  // dL/d omega of the tile's last residue (from the later tile)
    for (int k = 0; it.valid; ++k) {
        const int buf = k & 1;
        const int b = it.b, L = it.L, t = it.t, r0 = it.r0(), pre = r0 > 0 ? 1 : 0;
        const int n = it.n();
        const bool phaseB = it.phase == 1;
        if (!phaseB && t == 0) carryA = aff_identity();
        if (phaseB && t == it.nt - 1) {
#pragma unroll
            for (int q = 0; q < 6; ++q) carry6[q] = 0.f;
            omega_next = 0.f;
        }
        float* pref = ws_prefix + (size_t)b * max_tiles * 12;
        BBIter nx = it;
        nx.advance();
        if (tid == 0 && nx.valid)
            bb_issue(nx, angles, grad_coords, s_ang_buf + (buf ^ 1) * ANG, s_g_buf + (buf ^ 1) * GB, bar + (buf ^ 1));
        char* s_ang_base = s_ang_buf + buf * ANG;
        char* s_g_base = s_g_buf + buf * GB;
        const Span sa = make_span(angles + ((size_t)b * Lmax + r0 - pre) * 3, (n + pre) * 12);
        span_load_edges_f32(sa, s_ang_base);
        Span sg{};
        if (phaseB) {
            sg = make_span(grad_coords + ((size_t)b * 3 * Lmax + 3 * (size_t)r0) * 3, n * 36);
            span_load_edges_f32(sg, s_g_base);
        }
        mbar_wait(bar + buf, (phases >> buf) & 1u);
        phases ^= 1u << buf;
        __syncthreads();
        const float* s_ang = reinterpret_cast<const float*>(s_ang_base + sa.mis()) + 3 * pre;
        const int nq = max(0, min(RPT, n - rl0));

        if (!phaseB) {
            // ---- phase A: chunk aggregates only; the tile total becomes the prefix of tile t+1
            Aff M;
            float maxabs = 0.f;
            auto chunk = [&](auto slow) {
                constexpr bool kSlow = decltype(slow)::value;
                M = aff_identity();
#pragma unroll 2
                for (int q = 0; q < RPT; ++q) {
                    const int rl = rl0 + q;
                    float c[3], s[3];
                    bb_residue_trig<kSlow>(s_ang, rl, r0 + rl, c, s, &maxabs);
                    if (r0 + rl > 0) aff_bond_bb<0>(M, c[0], s[0]);
                    aff_bond_bb<1>(M, c[1], s[1]);
                    aff_bond_bb<2>(M, c[2], s[2]);
                }
            };
            chunk(std::false_type{});
            if (__syncthreads_or(maxabs > kSinCosFastMax)) chunk(std::true_type{});
            if (kNS >= 1) aff_orthonormalize(M);
            block_exclusive_scan<NT, kNS>(M, carryA, scratch, s_total);
            carryA = load_aff(s_total);
            if (tid < 12) pref[(t + 1) * 12 + tid] = s_total[tid];
            __syncthreads();  // the prefix is read by the tile's phase-B item
            it = nx;
            continue;
        }

        // ---- phase B
        const Aff carry = (t == 0) ? aff_identity() : load_aff(pref + t * 12);
        float* s_g = reinterpret_cast<float*>(s_g_base + sg.mis());

        // pass 1: local chunk; positions and rotation axes stay in registers
        constexpr int APT = 3 * RPT;
        Aff M;
        float maxabs = 0.f;
        float px[APT], py[APT], pz[APT], ex[APT], ey[APT], ez[APT];
        auto pass1 = [&](auto slow) {
            constexpr bool kSlow = decltype(slow)::value;
            M = aff_identity();
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                if (q < nq) {
                    const int rl = rl0 + q;
                    float c[3], s[3];
                    bb_residue_trig<kSlow>(s_ang, rl, r0 + rl, c, s, &maxabs);
                    auto save = [&](int a) {
                        px[a] = M.t0; py[a] = M.t1; pz[a] = M.t2;
                        ex[a] = M.r00; ey[a] = M.r10; ez[a] = M.r20;
                    };
                    if (r0 + rl > 0) aff_bond_bb<0>(M, c[0], s[0]);
                    save(3 * q);
                    aff_bond_bb<1>(M, c[1], s[1]);
                    save(3 * q + 1);
                    aff_bond_bb<2>(M, c[2], s[2]);
                    save(3 * q + 2);
                }
            }
        };
        pass1(std::false_type{});
        if (__any_sync(0xffffffffu, maxabs > kSinCosFastMax)) pass1(std::true_type{});  // rare: huge angles (per warp)
        if (kNS >= 1) aff_orthonormalize(M);
        if (tid == 0) bulk_wait_read_all();  // the gradient staging is free again
        const Aff P = block_exclusive_scan<NT, kNS>(M, carry, scratch, s_total);

        // pass 2: gradients rotated into the chunk frame (g_loc = R^T g)
        float sl[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        float gx[APT], gy[APT], gz[APT];
#pragma unroll
        for (int a = 0; a < APT; ++a) {
            gx[a] = gy[a] = gz[a] = 0.f;
            if (a / 3 < nq) {
                const float* g = s_g + 9 * rl0 + 3 * a;
                const float g0 = g[0], g1 = g[1], g2 = g[2];
                gx[a] = fmaf(P.r00, g0, fmaf(P.r10, g1, P.r20 * g2));
                gy[a] = fmaf(P.r01, g0, fmaf(P.r11, g1, P.r21 * g2));
                gz[a] = fmaf(P.r02, g0, fmaf(P.r12, g1, P.r22 * g2));
                sl[0] += gx[a]; sl[1] += gy[a]; sl[2] += gz[a];
                sl[3] += fmaf(py[a], gz[a], -pz[a] * gy[a]);
                sl[4] += fmaf(pz[a], gx[a], -px[a] * gz[a]);
                sl[5] += fmaf(px[a], gy[a], -py[a] * gx[a]);
            }
        }
        // thread totals in the global frame: S = R S_l, T = R T_l + t x S
        float sum6[6];
        sum6[0] = fmaf(P.r00, sl[0], fmaf(P.r01, sl[1], P.r02 * sl[2]));
        sum6[1] = fmaf(P.r10, sl[0], fmaf(P.r11, sl[1], P.r12 * sl[2]));
        sum6[2] = fmaf(P.r20, sl[0], fmaf(P.r21, sl[1], P.r22 * sl[2]));
        sum6[3] = fmaf(P.r00, sl[3], fmaf(P.r01, sl[4], P.r02 * sl[5])) + fmaf(P.t1, sum6[2], -P.t2 * sum6[1]);
        sum6[4] = fmaf(P.r10, sl[3], fmaf(P.r11, sl[4], P.r12 * sl[5])) + fmaf(P.t2, sum6[0], -P.t0 * sum6[2]);
        sum6[5] = fmaf(P.r20, sl[3], fmaf(P.r21, sl[4], P.r22 * sl[5])) + fmaf(P.t0, sum6[1], -P.t1 * sum6[0]);
        float suf[6], tot6[6];
        block_exclusive_suffix6<NT>(sum6, carry6, s_suf, suf, tot6);
        if (!nx.valid) pdl_trigger();  // late trigger (see the forward kernel)
        // later atoms into the chunk frame: S_l = R^T S, T_l = R^T (T - t x S)
        float su[6];
        {
            const float w0 = suf[3] - fmaf(P.t1, suf[2], -P.t2 * suf[1]);
            const float w1 = suf[4] - fmaf(P.t2, suf[0], -P.t0 * suf[2]);
            const float w2 = suf[5] - fmaf(P.t0, suf[1], -P.t1 * suf[0]);
            su[0] = fmaf(P.r00, suf[0], fmaf(P.r10, suf[1], P.r20 * suf[2]));
            su[1] = fmaf(P.r01, suf[0], fmaf(P.r11, suf[1], P.r21 * suf[2]));
            su[2] = fmaf(P.r02, suf[0], fmaf(P.r12, suf[1], P.r22 * suf[2]));
            su[3] = fmaf(P.r00, w0, fmaf(P.r10, w1, P.r20 * w2));
            su[4] = fmaf(P.r01, w0, fmaf(P.r11, w1, P.r21 * w2));
            su[5] = fmaf(P.r02, w0, fmaf(P.r12, w1, P.r22 * w2));
        }

        // pass 3: atoms last to first, grad alpha_i = e_i . (T - p_i x S)   (chunk frame)
        const Span so = make_span(grad_angles + ((size_t)b * Lmax + r0) * 3, n * 12);
        float* s_go = reinterpret_cast<float*>(s_go_base + so.mis());
#pragma unroll
        for (int q = RPT - 1; q >= 0; --q) {
            if (q < nq) {
                const int rl = rl0 + q;
                const int j = r0 + rl;
                float ga[3];
#pragma unroll
                for (int kk = 2; kk >= 0; --kk) {
                    const int a = 3 * q + kk;
                    const float x = px[a], y = py[a], z = pz[a];
                    const float c0 = su[3] - fmaf(y, su[2], -z * su[1]);
                    const float c1 = su[4] - fmaf(z, su[0], -x * su[2]);
                    const float c2 = su[5] - fmaf(x, su[1], -y * su[0]);
                    ga[kk] = fmaf(ex[a], c0, fmaf(ey[a], c1, ez[a] * c2));
                    su[0] += gx[a]; su[1] += gy[a]; su[2] += gz[a];
                    su[3] += fmaf(y, gz[a], -z * gy[a]);
                    su[4] += fmaf(z, gx[a], -x * gz[a]);
                    su[5] += fmaf(x, gy[a], -y * gx[a]);
                }
                s_go[3 * rl + 0] = ga[1];  // phi_j
                s_go[3 * rl + 1] = ga[2];  // psi_j
                if (j > 0) {               // omega_{j-1}
                    if (rl > 0) s_go[3 * (rl - 1) + 2] = ga[0];
                    else s_misc[0] = ga[0];  // belongs to the previous tile
                }
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
        for (int q = 0; q < 6; ++q) carry6[q] = tot6[q];
        __syncthreads();
        it = nx;
    }
    // Only the shared-memory source must outlive the CTA; grid completion (and the
    // dependent's griddepcontrol.wait) covers visibility of the global writes.
    if (tid == 0) bulk_wait_read_all();
}

// ---------------------------------------------------------------------------
// Backward from the forward's coordinates (no angles, no trig, no affine scan).
// The rotation axis of alpha_a is the unit bond vector e_a = (r_a - r_{a-1}) /
// |r_a - r_{a-1}| through r_a (M_a = M_{a-1} R_y(theta) T_x(d) R_x(alpha): the
// x-axis of frame a is the bond direction and its origin is r_a), so with
// S_a = sum_{b>a} g_b and T_a = sum_{b>a} (r_b - c) x g_b,
//   dL/dalpha_a = e_a . (T_a - (r_a - c) x S_a)
// for any reference point c (c = the tile's first atom, to keep moments small).
// One reverse suffix sum of (S, T) per chain; tiles last to first.
__device__ __forceinline__ void bbx_issue(const BBIter& it, const float* coords, const float* grad_coords,
                                          char* s_x, char* s_g, uint64_t* bar) {
    const int r0 = it.r0(), n = it.n(), pre = r0 > 0 ? 1 : 0;
    const size_t base = ((size_t)it.b * 3 * it.Lmax + 3 * (size_t)r0) * 3;
    const Span sx = make_span(coords + base - 3 * pre, (3 * n + pre) * 12);
    const Span sg = make_span(grad_coords + base, n * 36);
    mbar_arrive_expect_tx(bar, unsigned(sx.mid + sg.mid));
    span_load_bulk(sx, s_x, bar);
    span_load_bulk(sg, s_g, bar);
}

// kLoss (f1, fused LRMSD): grad_coords is the LRMSD target y, and dL/dr_i =
// dL/dLRMSD (x~_i - U^T y~_i) / (N LRMSD) (reading Q19) is formed
// on the fly from the forward's state -- no dL/dr array is written or read.
// kDB: two staging buffers (the next item's tiles load during this one); without
// it one buffer, refilled after the walk -- for grids where every CTA owns one
// item, so that twice the threads fit per SM.
// kPW: every thread closes omega of its own last residue from its exclusive suffix
// (the lever arm of N_{j+1} about itself is zero) and each warp bulk-stores its own
// residues as soon as its lanes are done (no block barrier before the store).
template <int NT, int RPT, bool kLoss = false, bool kDB = true, bool kPW = false>
__global__ void __launch_bounds__(NT, kMinBlocks128Regs(NT)) bb_backward_xyz_kernel(const float* __restrict__ coords,
                                                             const int* __restrict__ lengths, int B, int Lmax,
                                                             const float* __restrict__ grad_coords,
                                                             float* __restrict__ grad_angles,
                                                             unsigned* __restrict__ err,
                                                             const float* __restrict__ seg_totals, int n_seg,
                                                             int seg, const float* __restrict__ loss_state,
                                                             const float* __restrict__ loss_grad) {
    constexpr int TILE = NT * RPT;
    constexpr int XB = round16(16 + 36 * TILE + 12);  // tile atoms + the previous atom
    constexpr int GB = round16(16 + 36 * TILE);
    using S = BBSmem<NT>;
    extern __shared__ __align__(16) char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::kBar);
    float* s_suf = reinterpret_cast<float*>(smem + S::kSuf);
    float* s_misc = reinterpret_cast<float*>(smem + S::kMisc);
    constexpr int NB = kDB ? 2 : 1;
    char* s_x_buf = smem + S::kData;    // NB x XB
    char* s_g_buf = s_x_buf + NB * XB;  // NB x GB
    char* s_go_base = s_g_buf + NB * GB;

    const int tid = threadIdx.x;
    TPL_STAMP(0);
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        fence_barrier_init();
    }
    pdl_wait();
    BBIter it{lengths, B, Lmax, TILE, int(gridDim.x), false, err, true};
    it.init();
    __syncthreads();
    if (tid == 0 && it.valid) bbx_issue(it, coords, grad_coords, s_x_buf, s_g_buf, bar);

    unsigned phases = 0;

    const int rl0 = tid * RPT;
    float carry6[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // (S, T) of the later tiles, about c_prev
    float cpx = 0.f, cpy = 0.f, cpz = 0.f;              // reference point of the later tile
    float omega_next = 0.f;
    float lU[9], lcx[3], lcy[3], lsc = 0.f;                     // kLoss: the chain's LRMSD state
    bool has_ext = false;                                      // f4: later segments exist
    float ext[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, cnx = 0.f, cny = 0.f, cnz = 0.f;
    for (int k = 0; it.valid; ++k) {
        const int buf = kDB ? (k & 1) : 0;
        const int b = it.b, L = it.L, r0 = it.r0(), n = it.n(), pre = r0 > 0 ? 1 : 0;
        const bool last_tile = r0 + n == L;
        BBIter nx = it;
        nx.advance();
        if (kDB && tid == 0 && nx.valid)
            bbx_issue(nx, coords, grad_coords, s_x_buf + (buf ^ 1) * XB, s_g_buf + (buf ^ 1) * GB, bar + (buf ^ 1));
        char* s_x_base = s_x_buf + buf * XB;
        char* s_g_base = s_g_buf + buf * GB;
        const size_t base = ((size_t)b * 3 * Lmax + 3 * (size_t)r0) * 3;
        const Span sx = make_span(coords + base - 3 * pre, (3 * n + pre) * 12);
        const Span sg = make_span(grad_coords + base, n * 36);
        span_load_edges_f32(sx, s_x_base);
        span_load_edges_f32(sg, s_g_base);
        mbar_wait(bar + buf, (phases >> buf) & 1u);
        phases ^= 1u << buf;
        __syncthreads();
        if (k < 2) TPL_STAMP(2 + 4 * k);
        const float* s_x = reinterpret_cast<const float*>(s_x_base + sx.mis()) + 3 * pre;  // atom 0 of the tile
        const float* s_g = reinterpret_cast<const float*>(s_g_base + sg.mis());
        // dL/dr of one atom: the staged array, or (kLoss) the LRMSD gradient from x and y
        auto grad_of = [&](const float* xa, const float* ga, float& gx, float& gy, float& gz) {
            if (kLoss) {
                const float yx = ga[0] - lcy[0], yy = ga[1] - lcy[1], yz = ga[2] - lcy[2];
                gx = lsc * (xa[0] - lcx[0] - fmaf(lU[0], yx, fmaf(lU[3], yy, lU[6] * yz)));
                gy = lsc * (xa[1] - lcx[1] - fmaf(lU[1], yx, fmaf(lU[4], yy, lU[7] * yz)));
                gz = lsc * (xa[2] - lcx[2] - fmaf(lU[2], yx, fmaf(lU[5], yy, lU[8] * yz)));
            } else {
                gx = ga[0]; gy = ga[1]; gz = ga[2];
            }
        };
        const int nq = max(0, min(RPT, n - rl0));
        const float cx = s_x[0], cy = s_x[1], cz = s_x[2];
        if (last_tile) {
#pragma unroll
            for (int q = 0; q < 6; ++q) carry6[q] = 0.f;
            omega_next = 0.f;
            if (kLoss) {
                const float* st = loss_state + (size_t)b * 16;
#pragma unroll
                for (int q = 0; q < 9; ++q) lU[q] = __ldg(st + q);
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    lcx[q] = __ldg(st + 9 + q);
                    lcy[q] = __ldg(st + 12 + q);
                }
                lsc = __ldg(st + 15) * __ldg(loss_grad + b);
            }
            // f4 segments: the later segments' totals (fixed order) about the next
            // segment's first atom N, which also closes omega of the last residue
            has_ext = seg_totals != nullptr && seg + 1 < n_seg;
            if (has_ext) {
                const float* nt0 = seg_totals + ((size_t)(seg + 1) * B + b) * 12;
                cnx = __ldg(nt0 + 6); cny = __ldg(nt0 + 7); cnz = __ldg(nt0 + 8);
#pragma unroll
                for (int q = 0; q < 6; ++q) ext[q] = 0.f;
                for (int r = n_seg - 1; r > seg; --r) {
                    const float* tr = seg_totals + ((size_t)r * B + b) * 12;
                    const float S0 = __ldg(tr), S1 = __ldg(tr + 1), S2 = __ldg(tr + 2);
                    const float dx = __ldg(tr + 6) - cnx, dy = __ldg(tr + 7) - cny, dz = __ldg(tr + 8) - cnz;
                    ext[0] += S0; ext[1] += S1; ext[2] += S2;
                    ext[3] += __ldg(tr + 3) + fmaf(dy, S2, -dz * S1);
                    ext[4] += __ldg(tr + 4) + fmaf(dz, S0, -dx * S2);
                    ext[5] += __ldg(tr + 5) + fmaf(dx, S1, -dy * S0);
                }
            }
        } else {  // move the later tiles' moment to this tile's reference: T_c = T_c' + (c' - c) x S
            const float dx = cpx - cx, dy = cpy - cy, dz = cpz - cz;
            carry6[3] += fmaf(dy, carry6[2], -dz * carry6[1]);
            carry6[4] += fmaf(dz, carry6[0], -dx * carry6[2]);
            carry6[5] += fmaf(dx, carry6[1], -dy * carry6[0]);
        }
        cpx = cx; cpy = cy; cpz = cz;

        // pass 1: this thread's atoms into registers (positions about c, dL/dr, unit
        // bond vectors -- all independent of the suffix sums), and its (S, T) about c
        constexpr int APT = 3 * RPT;
        float Px[APT], Py[APT], Pz[APT], Gx[APT], Gy[APT], Gz[APT], Ex[APT], Ey[APT], Ez[APT];
        float sum6[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int a = 0; a < APT; ++a) {
            Px[a] = Py[a] = Pz[a] = Gx[a] = Gy[a] = Gz[a] = Ex[a] = Ey[a] = Ez[a] = 0.f;
            if (a / 3 < nq) {
                const float* x = s_x + 9 * rl0 + 3 * a;
                const float* g = s_g + 9 * rl0 + 3 * a;
                const float x0 = x[0], x1 = x[1], x2 = x[2];
                Px[a] = x0 - cx; Py[a] = x1 - cy; Pz[a] = x2 - cz;
                grad_of(x, g, Gx[a], Gy[a], Gz[a]);
                if (r0 + rl0 + a / 3 > 0 || a % 3 > 0) {  // atom 0 of the chain carries no angle
                    const float ux = x0 - x[-3], uy = x1 - x[-2], uz = x2 - x[-1];
                    const float inv = bb_invd(a % 3);  // the model bond length ending at atom a
                    Ex[a] = ux * inv; Ey[a] = uy * inv; Ez[a] = uz * inv;
                }
                sum6[0] += Gx[a]; sum6[1] += Gy[a]; sum6[2] += Gz[a];
                sum6[3] += fmaf(Py[a], Gz[a], -Pz[a] * Gy[a]);
                sum6[4] += fmaf(Pz[a], Gx[a], -Px[a] * Gz[a]);
                sum6[5] += fmaf(Px[a], Gy[a], -Py[a] * Gx[a]);
            }
        }
        if (kPW ? (tid & 31) == 0 : tid == 0) bulk_wait_read_all();  // the output staging is free again
        if (k < 2) TPL_STAMP(3 + 4 * k);
        float su[6], tot6[6];
        block_exclusive_suffix6<NT>(sum6, carry6, s_suf, su, tot6);
        if (k < 2) TPL_STAMP(4 + 4 * k);
        if (!nx.valid) pdl_trigger();
        if (has_ext) {  // later segments, about this tile's reference: T_c = T_n + (n - c) x S
            const float dx = cnx - cx, dy = cny - cy, dz = cnz - cz;
            su[0] += ext[0]; su[1] += ext[1]; su[2] += ext[2];
            su[3] += ext[3] + fmaf(dy, ext[2], -dz * ext[1]);
            su[4] += ext[4] + fmaf(dz, ext[0], -dx * ext[2]);
            su[5] += ext[5] + fmaf(dx, ext[1], -dy * ext[0]);
        }

        // pass 2: atoms last to first
        const Span so = make_span(grad_angles + ((size_t)b * Lmax + r0) * 3, n * 12);
        float* s_go = reinterpret_cast<float*>(s_go_base + so.mis());
        float w_last = 0.f;  // kPW: omega of this thread's last residue, e . (T - p_N x S) about N_{j+1}
        if (kPW && nq > 0) {
            const int an = 3 * (rl0 + nq);  // atom index of N_{j+1} in the tile
            float nx_ = 0.f, ny_ = 0.f, nz_ = 0.f;
            bool has_n = true;
            if (rl0 + nq < n) {
                nx_ = s_x[3 * an]; ny_ = s_x[3 * an + 1]; nz_ = s_x[3 * an + 2];
            } else if (!last_tile) {
                const float* gn = coords + ((size_t)b * 3 * Lmax + 3 * (size_t)(r0 + n)) * 3;
                nx_ = __ldg(gn); ny_ = __ldg(gn + 1); nz_ = __ldg(gn + 2);
            } else if (has_ext) {
                nx_ = cnx; ny_ = cny; nz_ = cnz;
            } else {
                has_n = false;  // omega_{L-1} is a structural zero
            }
            if (has_n) {
                const float* xc = s_x + 3 * (an - 1);
                const float ux = nx_ - xc[0], uy = ny_ - xc[1], uz = nz_ - xc[2];
                const float px = nx_ - cx, py = ny_ - cy, pz = nz_ - cz;
                const float c0 = su[3] - fmaf(py, su[2], -pz * su[1]);
                const float c1 = su[4] - fmaf(pz, su[0], -px * su[2]);
                const float c2 = su[5] - fmaf(px, su[1], -py * su[0]);
                w_last = bb_invd(0) * fmaf(ux, c0, fmaf(uy, c1, uz * c2));
            }
        }
#pragma unroll
        for (int q = RPT - 1; q >= 0; --q) {
            if (q < nq) {
                const int rl = rl0 + q;
                const int j = r0 + rl;
                float ga[3];
#pragma unroll
                for (int kk = 2; kk >= 0; --kk) {
                    const int a = 3 * q + kk;  // the thread's atom (registers)
                    const float px = Px[a], py = Py[a], pz = Pz[a], gx = Gx[a], gy = Gy[a], gz = Gz[a];
                    const float c0 = su[3] - fmaf(py, su[2], -pz * su[1]);
                    const float c1 = su[4] - fmaf(pz, su[0], -px * su[2]);
                    const float c2 = su[5] - fmaf(px, su[1], -py * su[0]);
                    ga[kk] = fmaf(Ex[a], c0, fmaf(Ey[a], c1, Ez[a] * c2));  // 0 for atom 0 of the chain
                    su[0] += gx; su[1] += gy; su[2] += gz;
                    su[3] += fmaf(py, gz, -pz * gy);
                    su[4] += fmaf(pz, gx, -px * gz);
                    su[5] += fmaf(px, gy, -py * gx);
                }
                s_go[3 * rl + 0] = ga[1];  // phi_j
                s_go[3 * rl + 1] = ga[2];  // psi_j
                if (kPW) {
                    if (q > 0) s_go[3 * (rl - 1) + 2] = ga[0];  // omega_{j-1}, this thread's residue
                    if (q == nq - 1) s_go[3 * rl + 2] = w_last;
                } else if (j > 0) {  // omega_{j-1}
                    if (rl > 0) s_go[3 * (rl - 1) + 2] = ga[0];
                    else s_misc[0] = ga[0];  // belongs to the previous tile
                }
            }
        }
        if (k < 2) TPL_STAMP(11 + k);
        if constexpr (kPW) {
            // per-warp stores (as bb_forward_kernel): a warp's residues are contiguous and
            // start 12 * 32 * RPT bytes apart, so shared and global keep the same 16-byte phase
            fence_proxy_async_smem();
            __syncwarp();
            const int lane = tid & 31, w0 = (tid >> 5) * 32 * RPT, wn = min(32 * RPT, n - w0);
            if (wn > 0) {
                const Span sw = make_span(grad_angles + ((size_t)b * Lmax + r0 + w0) * 3, wn * 12);
                const float* src = s_go + 3 * w0;
                if (lane == 0 && sw.mid > 0) {
                    bulk_s2g(const_cast<char*>(sw.g) + sw.head, reinterpret_cast<const char*>(src) + sw.head,
                             unsigned(sw.mid));
                    bulk_commit();
                }
                float* g = reinterpret_cast<float*>(const_cast<char*>(sw.g));
                const int nh = sw.head >> 2, ntl = sw.tail() >> 2, off_t = (sw.head + sw.mid) >> 2;
                for (int e = lane; e < nh + ntl; e += 32) {
                    const int idx = e < nh ? e : off_t + (e - nh);
                    g[idx] = src[idx];
                }
            }
#pragma unroll
            for (int q = 0; q < 6; ++q) carry6[q] = tot6[q];
            __syncthreads();  // s_x, s_g and the scan scratch are free again
            if (!kDB && tid == 0 && nx.valid) bbx_issue(nx, coords, grad_coords, s_x_buf, s_g_buf, bar);
            it = nx;
            continue;
        }
        if (tid == 0) {
            float w = last_tile ? 0.f : omega_next;
            if (last_tile && has_ext) {  // omega_{L-1} = e . T_n (the later segments about their N)
                const float* xc = s_x + 3 * (3 * n - 1);
                const float ux = cnx - xc[0], uy = cny - xc[1], uz = cnz - xc[2];
                w = bb_invd(0) * fmaf(ux, ext[3], fmaf(uy, ext[4], uz * ext[5]));
            }
            s_go[3 * (n - 1) + 2] = w;
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            span_store_bulk(so, s_go_base);
            bulk_commit();
            if (!kDB && nx.valid) bbx_issue(nx, coords, grad_coords, s_x_buf, s_g_buf, bar);  // buffer released
        }
        if (k < 2) TPL_STAMP(5 + 4 * k);
        span_store_edges_f32(so, s_go_base);
        omega_next = s_misc[0];
#pragma unroll
        for (int q = 0; q < 6; ++q) carry6[q] = tot6[q];
        __syncthreads();
        it = nx;
    }
    if (kPW ? (tid & 31) == 0 : tid == 0) bulk_wait_read_all();
    TPL_STAMP(10);
}

// Cluster-split coordinate backward: one cluster of CL CTAs per chain, parts as
// bb_forward_cl_kernel.  Each CTA reduces its part's (S, T) about its first atom
// c_r and sends (S, T, c_r) to the shared memory of every earlier CTA; CTA r adds
// the later parts' totals (fixed order, moved to the next part's first atom N)
// to its suffix sums, which also closes omega of its last residue (the same
// algebra as the f4 segment carry).  Chains up to CL * NT * RPT residues.
template <int NT, int RPT, int CL>
__global__ void __launch_bounds__(NT, kMinBlocks128Regs(NT)) bb_backward_xyz_cl_kernel(
    const float* __restrict__ coords, const int* __restrict__ lengths, int B, int Lmax,
    const float* __restrict__ grad_coords, float* __restrict__ grad_angles, unsigned* __restrict__ err) {
    constexpr int TILE = NT * RPT;
    constexpr int XB = round16(16 + 36 * TILE + 12);  // the previous atom and the part's atoms
    constexpr int GB = round16(16 + 36 * TILE);
    constexpr int SLOTS = round16(48 * CL);
    using S = BBSmem<NT>;
    extern __shared__ __align__(16) char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::kBar);  // [0] TMA, [1] later parts' totals
    float* s_suf = reinterpret_cast<float*>(smem + S::kSuf);
    float* s_slots = reinterpret_cast<float*>(smem + S::kData);  // (S, T, c) of later ranks
    char* s_x_base = smem + S::kData + SLOTS;
    char* s_g_base = s_x_base + XB;
    char* s_go_base = s_g_base + GB;

    const int tid = threadIdx.x;
    const unsigned rank = cluster_ctarank();
    pdl_wait();
    const int b = blockIdx.x / CL;
    const int L = b < B ? __ldg(lengths + b) : 0;
    const bool ok = L >= 1 && L <= Lmax;
    const int h = ok ? (L + CL - 1) / CL : 1, r0 = int(rank) * h, n = ok ? min(h, L - r0) : 0;
    int nlater = 0;  // later non-empty parts: the arrivals this CTA waits for
    for (int r = int(rank) + 1; r < CL; ++r) nlater += (ok && r * h < L) ? 1 : 0;
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, nlater > 0 ? nlater : 1);
        fence_mbarrier_init_cluster();
        fence_barrier_init();
    }
    __syncthreads();
    cluster_arrive_relaxed();
    if (!ok) {
        if (tid == 0 && rank == 0 && b < B) atomicOr(err, ERR_LENGTH);
        return;
    }
    if (n <= 0) return;  // no CTA sends to (or waits for) an empty part
    const int pre = r0 > 0 ? 1 : 0;
    const size_t base = ((size_t)b * 3 * Lmax + 3 * (size_t)r0) * 3;
    const Span sx = make_span(coords + base - 3 * pre, (3 * n + pre) * 12);
    const Span sg = make_span(grad_coords + base, n * 36);
    if (tid == 0) {
        mbar_arrive_expect_tx(bar, unsigned(sx.mid + sg.mid));
        span_load_bulk(sx, s_x_base, bar);
        span_load_bulk(sg, s_g_base, bar);
    }
    span_load_edges_f32(sx, s_x_base);
    span_load_edges_f32(sg, s_g_base);
    mbar_wait(bar, 0);
    __syncthreads();
    cluster_wait_aligned();  // every CTA's barriers are initialised (see bb_forward_cl_kernel)
    const float* s_x = reinterpret_cast<const float*>(s_x_base + sx.mis()) + 3 * pre;  // atom 0 of the part
    const float* s_g = reinterpret_cast<const float*>(s_g_base + sg.mis());
    const float cx = s_x[0], cy = s_x[1], cz = s_x[2];
    const int rl0 = tid * RPT;
    const int nq = max(0, min(RPT, n - rl0));

    // pass 1 (as bb_backward_xyz_kernel)
    constexpr int APT = 3 * RPT;
    float Px[APT], Py[APT], Pz[APT], Gx[APT], Gy[APT], Gz[APT], Ex[APT], Ey[APT], Ez[APT];
    float sum6[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int a = 0; a < APT; ++a) {
        Px[a] = Py[a] = Pz[a] = Gx[a] = Gy[a] = Gz[a] = Ex[a] = Ey[a] = Ez[a] = 0.f;
        if (a / 3 < nq) {
            const float* x = s_x + 9 * rl0 + 3 * a;
            const float* g = s_g + 9 * rl0 + 3 * a;
            const float x0 = x[0], x1 = x[1], x2 = x[2];
            Px[a] = x0 - cx; Py[a] = x1 - cy; Pz[a] = x2 - cz;
            Gx[a] = g[0]; Gy[a] = g[1]; Gz[a] = g[2];
            if (r0 + rl0 + a / 3 > 0 || a % 3 > 0) {  // atom 0 of the chain carries no angle
                const float ux = x0 - x[-3], uy = x1 - x[-2], uz = x2 - x[-1];
                const float inv = bb_invd(a % 3);  // the model bond length ending at atom a
                Ex[a] = ux * inv; Ey[a] = uy * inv; Ez[a] = uz * inv;
            }
            sum6[0] += Gx[a]; sum6[1] += Gy[a]; sum6[2] += Gz[a];
            sum6[3] += fmaf(Py[a], Gz[a], -Pz[a] * Gy[a]);
            sum6[4] += fmaf(Pz[a], Gx[a], -Px[a] * Gz[a]);
            sum6[5] += fmaf(Px[a], Gy[a], -Py[a] * Gx[a]);
        }
    }
    const float zero6[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float su[6], tot6[6];
    block_exclusive_suffix6<NT>(sum6, zero6, s_suf, su, tot6);
    // ---- exchange: this part's (S, T about c_r, c_r) to every earlier CTA
    if (tid == 0) {
        for (int r = 0; r < int(rank); ++r) {
            const uint32_t dst = mapa_shared(smem_u32(s_slots + 12 * rank), unsigned(r));
            st_cluster_v4(dst, tot6[0], tot6[1], tot6[2], tot6[3]);
            st_cluster_v4(dst + 16, tot6[4], tot6[5], cx, cy);
            st_cluster_v2(dst + 32, cz, 0.f);
            mbar_arrive_remote(mapa_shared(smem_u32(bar + 1), unsigned(r)));
        }
    }
    float ext[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, cnx = 0.f, cny = 0.f, cnz = 0.f;
    if (nlater > 0) {  // later parts, last to first, about the next part's first atom N
        mbar_wait_cluster(bar + 1, 0);
        const float* n0 = s_slots + 12 * (rank + 1);
        cnx = n0[6]; cny = n0[7]; cnz = n0[8];
        for (int r = int(rank) + nlater; r > int(rank); --r) {
            const float* tr = s_slots + 12 * r;
            const float S0 = tr[0], S1 = tr[1], S2 = tr[2];
            const float dx = tr[6] - cnx, dy = tr[7] - cny, dz = tr[8] - cnz;
            ext[0] += S0; ext[1] += S1; ext[2] += S2;
            ext[3] += tr[3] + fmaf(dy, S2, -dz * S1);
            ext[4] += tr[4] + fmaf(dz, S0, -dx * S2);
            ext[5] += tr[5] + fmaf(dx, S1, -dy * S0);
        }
        const float dx = cnx - cx, dy = cny - cy, dz = cnz - cz;  // to this part's reference
        su[0] += ext[0]; su[1] += ext[1]; su[2] += ext[2];
        su[3] += ext[3] + fmaf(dy, ext[2], -dz * ext[1]);
        su[4] += ext[4] + fmaf(dz, ext[0], -dx * ext[2]);
        su[5] += ext[5] + fmaf(dx, ext[1], -dy * ext[0]);
    }
    pdl_trigger();

    // pass 2: atoms last to first
    const Span so = make_span(grad_angles + ((size_t)b * Lmax + r0) * 3, n * 12);
    float* s_go = reinterpret_cast<float*>(s_go_base + so.mis());
#pragma unroll
    for (int q = RPT - 1; q >= 0; --q) {
        if (q < nq) {
            const int rl = rl0 + q;
            float ga[3];
#pragma unroll
            for (int kk = 2; kk >= 0; --kk) {
                const int a = 3 * q + kk;
                const float px = Px[a], py = Py[a], pz = Pz[a], gx = Gx[a], gy = Gy[a], gz = Gz[a];
                const float c0 = su[3] - fmaf(py, su[2], -pz * su[1]);
                const float c1 = su[4] - fmaf(pz, su[0], -px * su[2]);
                const float c2 = su[5] - fmaf(px, su[1], -py * su[0]);
                ga[kk] = fmaf(Ex[a], c0, fmaf(Ey[a], c1, Ez[a] * c2));
                su[0] += gx; su[1] += gy; su[2] += gz;
                su[3] += fmaf(py, gz, -pz * gy);
                su[4] += fmaf(pz, gx, -px * gz);
                su[5] += fmaf(px, gy, -py * gx);
            }
            s_go[3 * rl + 0] = ga[1];                      // phi_j
            s_go[3 * rl + 1] = ga[2];                      // psi_j
            if (rl > 0) s_go[3 * (rl - 1) + 2] = ga[0];  // omega_{j-1} (the previous part computes its own)
        }
    }
    if (tid == 0) {  // omega of the part's last residue: e . T_N of the later parts (0 at the chain end)
        float w = 0.f;
        if (nlater > 0) {
            const float* xc = s_x + 3 * (3 * n - 1);
            const float ux = cnx - xc[0], uy = cny - xc[1], uz = cnz - xc[2];
            w = bb_invd(0) * fmaf(ux, ext[3], fmaf(uy, ext[4], uz * ext[5]));
        }
        s_go[3 * (n - 1) + 2] = w;
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
        span_store_bulk(so, s_go_base);
        bulk_commit();
    }
    span_store_edges_f32(so, s_go_base);
    if (tid == 0) bulk_wait_read_all();
}

// Decoupled coordinate backward: every (chain, tile) item sums its tile, publishes
// (S_t, T_t about c_t, c_t) unless it is the chain's first tile, and adds the
// later tiles' totals (fixed order, moved to its own reference) as its carry.
// omega of the tile's last residue is computed here from the next tile's first
// atom N: its own term drops out of e . (T - (r_N - c) x S) (zero lever arm).
template <int NT, int RPT>
__global__ void __launch_bounds__(NT, kMinBlocks128Regs(NT)) bb_backward_xyz_dl_kernel(
    const float* __restrict__ coords, const int* __restrict__ lengths, int B, int Lmax,
    const float* __restrict__ grad_coords, float* __restrict__ grad_angles, unsigned* __restrict__ hdr,
    float* __restrict__ slots, int max_tiles) {
    constexpr int TILE = NT * RPT;
    constexpr int XB = round16(16 + 36 * TILE + 24);  // the previous atom, the tile, the next atom
    constexpr int GB = round16(16 + 36 * TILE);
    using S = BBSmem<NT>;
    extern __shared__ __align__(16) char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::kBar);
    float* s_suf = reinterpret_cast<float*>(smem + S::kSuf);
    float* s_misc = reinterpret_cast<float*>(smem + S::kMisc);  // carry (6)
    char* s_x_buf = smem + S::kData;   // 2 x XB
    char* s_g_buf = s_x_buf + 2 * XB;  // 2 x GB
    char* s_go_base = s_g_buf + 2 * GB;

    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        fence_barrier_init();
    }
    pdl_wait();
    const unsigned fv = launch_epoch(hdr) + 1u;
    DLIter it{lengths, B, Lmax, TILE, max_tiles, int(gridDim.x), false, hdr};
    it.init();
    auto spans = [&](const DLIter& w, Span& sx, Span& sg) {
        const int r0 = w.r0(), n = w.n(), pre = r0 > 0 ? 1 : 0, post = r0 + n < w.L ? 1 : 0;
        const size_t base = ((size_t)w.b * 3 * w.Lmax + 3 * (size_t)r0) * 3;
        sx = make_span(coords + base - 3 * pre, (3 * n + pre + post) * 12);
        sg = make_span(grad_coords + base, n * 36);
    };
    auto issue = [&](const DLIter& w, int buf) {
        Span sx, sg;
        spans(w, sx, sg);
        mbar_arrive_expect_tx(bar + buf, unsigned(sx.mid + sg.mid));
        span_load_bulk(sx, s_x_buf + buf * XB, bar + buf);
        span_load_bulk(sg, s_g_buf + buf * GB, bar + buf);
    };
    __syncthreads();
    if (tid == 0 && it.valid) issue(it, 0);

    unsigned phases = 0;
    const int rl0 = tid * RPT;
    for (int k = 0; it.valid; ++k) {
        const int buf = k & 1;
        const int b = it.b, L = it.L, r0 = it.r0(), n = it.n(), t = it.t, pre = r0 > 0 ? 1 : 0;
        const bool last_tile = r0 + n == L;
        DLIter nx = it;
        nx.advance();
        if (tid == 0 && nx.valid) issue(nx, buf ^ 1);
        char* s_x_base = s_x_buf + buf * XB;
        char* s_g_base = s_g_buf + buf * GB;
        Span sx, sg;
        spans(it, sx, sg);
        span_load_edges_f32(sx, s_x_base);
        span_load_edges_f32(sg, s_g_base);
        mbar_wait(bar + buf, (phases >> buf) & 1u);
        phases ^= 1u << buf;
        __syncthreads();
        const float* s_x = reinterpret_cast<const float*>(s_x_base + sx.mis()) + 3 * pre;  // atom 0 of the tile
        const float* s_g = reinterpret_cast<const float*>(s_g_base + sg.mis());
        const int nq = max(0, min(RPT, n - rl0));
        const float cx = s_x[0], cy = s_x[1], cz = s_x[2];

        // pass 1: this thread's (S, T) about c
        float sum6[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int a = 0; a < 3 * RPT; ++a) {
            if (a / 3 < nq) {
                const float* x = s_x + 9 * rl0 + 3 * a;
                const float* g = s_g + 9 * rl0 + 3 * a;
                const float px = x[0] - cx, py = x[1] - cy, pz = x[2] - cz, gx = g[0], gy = g[1], gz = g[2];
                sum6[0] += gx; sum6[1] += gy; sum6[2] += gz;
                sum6[3] += fmaf(py, gz, -pz * gy);
                sum6[4] += fmaf(pz, gx, -px * gz);
                sum6[5] += fmaf(px, gy, -py * gx);
            }
        }
        if (tid == 0) bulk_wait_read_all();  // the output staging is free again
        const float zero6[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        float su[6], tot6[6];
        block_exclusive_suffix6<NT>(sum6, zero6, s_suf, su, tot6);  // tile-local
        if (tid == 0) {
            float* slot = slots + ((size_t)b * max_tiles + t) * 16;
            if (t > 0) {  // publish for the earlier tiles
#pragma unroll
                for (int q = 0; q < 6; ++q) slot[q] = tot6[q];
                slot[6] = cx; slot[7] = cy; slot[8] = cz;
                __threadfence();
                st_release_gpu(reinterpret_cast<unsigned*>(slot + 12), fv);
            }
            float cr[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            for (int u = it.nt - 1; u > t; --u) {  // fixed order: deterministic rounding
                const float* sl = slots + ((size_t)b * max_tiles + u) * 16;
                wait_flag(reinterpret_cast<const unsigned*>(sl + 12), fv);
                const float S0 = __ldcg(sl + 0), S1 = __ldcg(sl + 1), S2 = __ldcg(sl + 2);
                const float dx = __ldcg(sl + 6) - cx, dy = __ldcg(sl + 7) - cy, dz = __ldcg(sl + 8) - cz;
                cr[0] += S0; cr[1] += S1; cr[2] += S2;
                cr[3] += __ldcg(sl + 3) + fmaf(dy, S2, -dz * S1);
                cr[4] += __ldcg(sl + 4) + fmaf(dz, S0, -dx * S2);
                cr[5] += __ldcg(sl + 5) + fmaf(dx, S1, -dy * S0);
            }
#pragma unroll
            for (int q = 0; q < 6; ++q) s_misc[q] = cr[q];
        }
        __syncthreads();
        float carry[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            carry[q] = s_misc[q];
            su[q] += carry[q];
        }
        if (!nx.valid) pdl_trigger();

        // pass 2: atoms last to first
        const Span so = make_span(grad_angles + ((size_t)b * Lmax + r0) * 3, n * 12);
        float* s_go = reinterpret_cast<float*>(s_go_base + so.mis());
        if (nq > 0 && rl0 + nq == n) {  // omega of the tile's last residue (0 at the chain end)
            float gw = 0.f;
            if (!last_tile) {
                const float* xn = s_x + 9 * n;  // N of the next tile's first residue
                const float* xc = xn - 3;       // C of this tile's last residue
                const float ux = xn[0] - xc[0], uy = xn[1] - xc[1], uz = xn[2] - xc[2];
                const float px = xn[0] - cx, py = xn[1] - cy, pz = xn[2] - cz;
                const float c0 = carry[3] - fmaf(py, carry[2], -pz * carry[1]);
                const float c1 = carry[4] - fmaf(pz, carry[0], -px * carry[2]);
                const float c2 = carry[5] - fmaf(px, carry[1], -py * carry[0]);
                gw = bb_invd(0) * fmaf(ux, c0, fmaf(uy, c1, uz * c2));
            }
            s_go[3 * (n - 1) + 2] = gw;
        }
#pragma unroll
        for (int q = RPT - 1; q >= 0; --q) {
            if (q < nq) {
                const int rl = rl0 + q;
                const int j = r0 + rl;
                float ga[3];
#pragma unroll
                for (int kk = 2; kk >= 0; --kk) {
                    const int a = 3 * rl + kk;
                    const float* x = s_x + 3 * a;
                    const float* g = s_g + 3 * a;
                    const float x0 = x[0], x1 = x[1], x2 = x[2];
                    const float px = x0 - cx, py = x1 - cy, pz = x2 - cz;
                    const float gx = g[0], gy = g[1], gz = g[2];
                    if (j > 0 || kk > 0) {
                        const float ux = x0 - x[-3], uy = x1 - x[-2], uz = x2 - x[-1];
                        const float inv = bb_invd(kk);  // the model bond length ending at this atom
                        const float c0 = su[3] - fmaf(py, su[2], -pz * su[1]);
                        const float c1 = su[4] - fmaf(pz, su[0], -px * su[2]);
                        const float c2 = su[5] - fmaf(px, su[1], -py * su[0]);
                        ga[kk] = inv * fmaf(ux, c0, fmaf(uy, c1, uz * c2));
                    } else {
                        ga[kk] = 0.f;
                    }
                    su[0] += gx; su[1] += gy; su[2] += gz;
                    su[3] += fmaf(py, gz, -pz * gy);
                    su[4] += fmaf(pz, gx, -px * gz);
                    su[5] += fmaf(px, gy, -py * gx);
                }
                s_go[3 * rl + 0] = ga[1];                   // phi_j
                s_go[3 * rl + 1] = ga[2];                   // psi_j
                if (rl > 0) s_go[3 * (rl - 1) + 2] = ga[0];  // omega_{j-1} (the previous tile owns rl = 0's)
            }
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            span_store_bulk(so, s_go_base);
            bulk_commit();
        }
        span_store_edges_f32(so, s_go_base);
        __syncthreads();
        it = nx;
    }
    __syncthreads();
    if (tid == 0) {
        bulk_wait_read_all();
        finish_epoch(hdr);
    }
}

// ---------------------------------------------------------------------------
// Host-side launch helpers (called from capi.cu).

// Launch shape: NT threads per chain, RPT residues per thread (tile NT*RPT).
// Chains longer than the largest tile loop over tiles.
struct BBShape {
    int nt, rpt;
};
struct BBClShape {
    int nt, rpt, cl;
};
static int bb_nt_env() {  // TPL_BB_NT=32|128|256 forces the block size (tuning); 0 = default
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("TPL_BB_NT");
        const int x = e ? std::atoi(e) : 0;
        v = (x == 32 || x == 128 || x == 256) ? x : 0;
    }
    return v;
}
// Odd residues-per-thread only: the per-thread strides 3*RPT (angles) and
// 9*RPT (coordinates) in shared memory are then bank-conflict free.
// Forward: 128 threads, RPT in {1,3,5,7} (tile <= 896).  Backward keeps 9
// floats per atom in registers: 256 threads, RPT in {1,3} (tile <= 768).
static BBShape env_shape(const char* name);
static BBShape bb_shape(bool fwd, int Lmax) {
    if (fwd) {  // TPL_BBFS=NTxRPT forces the chain-serial forward shape (tuning)
        static const BBShape e = env_shape("TPL_BBFS");
        if (e.nt) return e;
    }
    int nt = bb_nt_env();
    if (!nt) nt = (fwd || Lmax > 128) ? (fwd ? 128 : 256) : 128;
    static const int f128[4] = {1, 3, 5, 7}, f256[3] = {1, 3, 5}, b128[2] = {1, 3}, b256[2] = {1, 3},
                     w32[4] = {1, 3, 5, 7};
    const int* opts = nt == 32 ? w32 : fwd ? (nt == 256 ? f256 : f128) : (nt == 256 ? b256 : b128);
    const int n = nt == 32 ? (fwd ? 4 : 3) : fwd ? (nt == 256 ? 3 : 4) : 2;
    for (int i = 0; i < n; ++i)
        if (nt * opts[i] >= Lmax) return {nt, opts[i]};
    return {nt, opts[n - 1]};
}
int bb_rpt_for(int Lmax) { return bb_shape(false, Lmax).rpt; }
int bb_tile_for(int Lmax) {  // backward tile: sizes the workspace's per-tile prefixes
    const BBShape s = bb_shape(false, Lmax);
    return s.nt * s.rpt;
}

template <int NT>
static size_t fwd_smem(int rpt, bool loss = false) {
    const int tile = NT * rpt;
    const size_t out = round16(16 + 36 * tile);
    return BBSmem<NT>::kData + 2 * round16(16 + 12 * (tile + 1)) + out +
           (loss ? out + 17 * NT * 8 + 18 * 8 + 16 : 0);
}
template <int NT>
static size_t bwd_smem(int rpt) {
    const int tile = NT * rpt;
    return BBSmem<NT>::kData + 2 * round16(16 + 12 * (tile + 1)) + 2 * round16(16 + 36 * tile) +
           round16(16 + 12 * tile);
}

static int sm_count() { return device_sm_count(); }


// Grid of the chain-serial kernels: the co-resident CTAs, each walking chains
// b, b + grid, ...; for rows longer than 1024 residues one CTA per chain, which
// lets the block scheduler balance ragged batches (config 4, 4096 x U[50, 2000]:
// 212 -> 185 us; uniform 1024-4096 x 1000-2000 within +-1.6%), while shorter
// rows keep the persistent grid (one CTA per chain costs 4096 x 700 8%; dynamic
// chain claiming through a workspace counter cost more in atomics than it saved).
// TPL_GRID=<m> forces m x the co-resident grid (0: one CTA per chain).
static int chain_grid(int B, int cap, int Lmax) {
    static const int mult = [] {
        const char* e = std::getenv("TPL_GRID");
        return e ? std::atoi(e) : -1;
    }();
    if (mult == 0 || (mult < 0 && Lmax > 1024)) return B;
    const long g = long(mult > 0 ? mult : 1) * cap;
    return B < g ? B : int(g);
}

template <int NT, int RPT, int NS, bool LOSS = false, int MINB = 0>
static cudaError_t launch_fwd(const BBArgs& a, cudaStream_t st) {
    auto k = bb_forward_kernel<NT, RPT, NS, LOSS, MINB>;
    const size_t sm = fwd_smem<NT>(RPT, LOSS);
    static LaunchCfg cfg;
    cudaError_t e = ensure_launch_cfg(cfg, k, NT, sm);
    if (e != cudaSuccess) return e;
    const int grid_cap = cfg.cap_now();
    const int grid = chain_grid(a.B, grid_cap, a.Lmax);
    return launch_pdl(k, grid, NT, sm, st, a.angles, a.lengths, a.B, a.Lmax, a.coords, a.err,
                      static_cast<const float*>(a.seg_omega_prev), a.seg_agg_out, a.loss_target, a.loss_out,
                      a.loss_state_out);
}
template <int NT, int RPT, int NS>
static cudaError_t launch_bwd(const BBArgs& a, cudaStream_t st) {
    auto k = bb_backward_kernel<NT, RPT, NS>;
    const size_t sm = bwd_smem<NT>(RPT);
    static LaunchCfg cfg;
    cudaError_t e = ensure_launch_cfg(cfg, k, NT, sm);
    if (e != cudaSuccess) return e;
    const int grid_cap = cfg.cap_now();
    const int grid = chain_grid(a.B, grid_cap, a.Lmax);
    return launch_pdl(k, grid, NT, sm, st, a.angles, a.lengths, a.B, a.Lmax, a.grad_coords, a.grad_angles, a.err,
                      a.ws_prefix, a.max_tiles);
}

template <bool kFwd, int NS>
static cudaError_t dispatch(const BBArgs& a, cudaStream_t st) {
    const BBShape s = bb_shape(kFwd, a.Lmax);
    if (kFwd) {
        // 128 x 7 with at most two chains per SM: registers for 2 CTAs/SM (no spills)
        if (s.nt == 128 && s.rpt == 7 && a.B <= 2 * sm_count()) return launch_fwd<128, 7, NS, false, 2>(a, st);
#define TPL_BB_FWD(NT_, R_) \
    if (s.nt == NT_ && s.rpt == R_) return launch_fwd<NT_, R_, NS>(a, st);
        TPL_BB_FWD(32, 1) TPL_BB_FWD(32, 3) TPL_BB_FWD(32, 5) TPL_BB_FWD(32, 7)
        TPL_BB_FWD(128, 1) TPL_BB_FWD(128, 3) TPL_BB_FWD(128, 5) TPL_BB_FWD(128, 7)
        TPL_BB_FWD(256, 1) TPL_BB_FWD(256, 3) TPL_BB_FWD(256, 5)
#undef TPL_BB_FWD
    } else {
#define TPL_BB_BWD(NT_, R_) \
    if (s.nt == NT_ && s.rpt == R_) return launch_bwd<NT_, R_, NS>(a, st);
        TPL_BB_BWD(32, 1) TPL_BB_BWD(32, 3) TPL_BB_BWD(32, 5)
        TPL_BB_BWD(128, 1) TPL_BB_BWD(128, 3) TPL_BB_BWD(256, 1) TPL_BB_BWD(256, 3)
#undef TPL_BB_BWD
    }
    return cudaErrorInvalidConfiguration;
}

template <int NT, int RPT, bool LOSS = false, bool DB = true, bool PW = false>
static cudaError_t launch_bwd_xyz(const BBArgs& a, cudaStream_t st) {
    auto k = bb_backward_xyz_kernel<NT, RPT, LOSS, DB, PW>;
    const int tile = NT * RPT;
    const int nb = DB ? 2 : 1;
    const size_t sm = BBSmem<NT>::kData + nb * round16(16 + 36 * tile + 12) + nb * round16(16 + 36 * tile) +
                      round16(16 + 12 * tile);
    static LaunchCfg cfg;
    cudaError_t e = ensure_launch_cfg(cfg, k, NT, sm);
    if (e != cudaSuccess) return e;
    const int grid_cap = cfg.cap_now();
    const int grid = chain_grid(a.B, grid_cap, a.Lmax);
    return launch_pdl(k, grid, NT, sm, st, static_cast<const float*>(a.coords), a.lengths, a.B, a.Lmax,
                      LOSS ? a.loss_target : a.grad_coords, a.grad_angles, a.err, a.seg_totals, a.n_seg, a.seg,
                      a.loss_state, a.loss_grad);
}

// Shape of the coordinate backward: TPL_BBX=NTxRPT (tuning) or the default.
// Measured (tools/gpu_bbx.sh): with at most one chain per SM the serial tile
// chain dominates -> the largest tile (256 threads, RPT up to 5); with more
// chains than SMs the kernel streams HBM and small tiles win (more resident
// CTAs: 128 x 3 takes 60 KB of shared memory, 3 CTAs per SM).
static BBShape bbx_shape(int B, int Lmax) {
    static int env_nt = -1, env_rpt = 0;
    if (env_nt < 0) {
        env_nt = 0;
        if (const char* e = std::getenv("TPL_BBX")) {
            int nt = 0, r = 0;
            if (std::sscanf(e, "%dx%d", &nt, &r) == 2) { env_nt = nt; env_rpt = r; }
        }
    }
    if (env_nt) return {env_nt, env_rpt};
    if (B > sm_count()) return {128, Lmax > 128 ? 3 : 1};
    static const int opts[3] = {1, 3, 5};  // 256 x 7 would not fit in shared memory
    const int nt = Lmax > 128 ? 256 : 128;
    for (int i = 0; i < 3; ++i)
        if (nt * opts[i] >= Lmax) return {nt, opts[i]};
    return {nt, 5};
}

static bool dl_enabled(int B, int Lmax);
static BBShape bbx_dl_shape(int B, int Lmax);
template <int NT, int RPT>
static cudaError_t launch_bwd_xyz_dl(const BBArgs& a, cudaStream_t st);

// Cluster-split coordinate backward (TPL_BBXC=NTxRPTxCL forces a shape; "0" disables).
template <int NT, int RPT, int CL>
static cudaError_t launch_bwd_xyz_cl(const BBArgs& a, cudaStream_t st) {
    auto k = bb_backward_xyz_cl_kernel<NT, RPT, CL>;
    const int tile = NT * RPT;
    const size_t sm = BBSmem<NT>::kData + round16(48 * CL) + round16(16 + 36 * tile + 12) + round16(16 + 36 * tile) +
                      round16(16 + 12 * tile);
    static LaunchCfg cfg;
    cudaError_t e = ensure_launch_cfg(cfg, k, NT, sm);
    if (e != cudaSuccess) return e;
    return launch_cluster(k, a.B * CL, CL, NT, sm, st, static_cast<const float*>(a.coords), a.lengths, a.B, a.Lmax,
                          a.grad_coords, a.grad_angles, a.err);
}
static BBClShape bbxc_shape(int B, int Lmax) {
    static const BBClShape env = [] {
        BBClShape s{0, 0, 0};
        const char* e = std::getenv("TPL_BBXC");
        if (e && std::sscanf(e, "%dx%dx%d", &s.nt, &s.rpt, &s.cl) != 3) s = {-1, 0, 0};
        return s;
    }();
    if (env.nt < 0) return {0, 0, 0};
    if (env.nt > 0) return env.cl * env.nt * env.rpt >= Lmax ? env : BBClShape{0, 0, 0};
    // measured (tools/gpu_clx_probe.sh): the backward has no trig in pass 1, so the
    // split only pays where the chain-per-CTA kernel needs a second tile and the
    // chains leave SMs idle -- 128 x 1000 8.1 -> 7.2 us; 64 x 700 (4.9 vs 5.5 us),
    // 256 x 700 and 256 x 1000 stay chain-per-CTA
    if (Lmax > 768 && Lmax <= 1536 && B <= sm_count()) return {256, 3, 2};
    return {0, 0, 0};
}

cudaError_t bb_backward_xyz_launch(const BBArgs& a, cudaStream_t st) {
    if (!a.loss_state && !a.seg_totals && bbp_enabled() && bbp_backward_xyz_ok(a)) return bbp_backward_xyz_launch(a, st);
    // longer chains, more of them than the decoupled / cluster regimes: tiles walked per CTA,
    // opt-in (TPL_BBPXT=NTxRxNB): measured 89.7-91.0 us for config 4 against 86.1 us for the
    // chain-serial 128 x 3 kernel below (tools/gpu.sh ab), so the default stays there
    static const bool tiles_bwd = std::getenv("TPL_BBPXT") != nullptr;
    if (tiles_bwd && !a.loss_state && !a.seg_totals && bbp_enabled() && !dl_enabled(a.B, a.Lmax) &&
        a.B > sm_count())
        return bbp_backward_xyz_tiles_launch(a, st);
    if (a.loss_state) {  // f1 fused LRMSD: chain-serial shapes
        const BBShape l = bbx_shape(a.B, a.Lmax);
#define TPL_BBXL(NT_, R_) \
    if (l.nt == NT_ && l.rpt == R_) return launch_bwd_xyz<NT_, R_, true>(a, st);
        TPL_BBXL(128, 1) TPL_BBXL(128, 3) TPL_BBXL(128, 5) TPL_BBXL(256, 1) TPL_BBXL(256, 3) TPL_BBXL(256, 5)
#undef TPL_BBXL
        return cudaErrorInvalidConfiguration;
    }
    if (!a.seg_totals && dl_enabled(a.B, a.Lmax)) {
        const BBShape d = bbx_dl_shape(a.B, a.Lmax);
        if (d.nt == 128 && d.rpt == 1) return launch_bwd_xyz_dl<128, 1>(a, st);
        if (d.nt == 128 && d.rpt == 3) return launch_bwd_xyz_dl<128, 3>(a, st);
        if (d.nt == 128 && d.rpt == 5) return launch_bwd_xyz_dl<128, 5>(a, st);
        if (d.nt == 256 && d.rpt == 3) return launch_bwd_xyz_dl<256, 3>(a, st);
        return cudaErrorInvalidConfiguration;
    }
    if (!a.seg_totals) {
        const BBClShape c = bbxc_shape(a.B, a.Lmax);
        if (c.nt == 128 && c.rpt == 3 && c.cl == 2) return launch_bwd_xyz_cl<128, 3, 2>(a, st);
        if (c.nt == 128 && c.rpt == 5 && c.cl == 2) return launch_bwd_xyz_cl<128, 5, 2>(a, st);
        if (c.nt == 256 && c.rpt == 3 && c.cl == 2) return launch_bwd_xyz_cl<256, 3, 2>(a, st);
        if (c.nt > 0) return cudaErrorInvalidConfiguration;
    }
    // one 768-residue tile per chain and at most ~3 chains per SM (two resident): single-buffered
    // 256 x 3 (65 KB; 2 CTAs/SM at 128 registers) keeps every chain resident with 8 warps each
    const bool env_shape = std::getenv("TPL_BBX") != nullptr;
    static const bool pw = [] {
        const char* e = std::getenv("TPL_BBX_PW");
        return e != nullptr && e[0] == '1';
    }();
    if (!env_shape && a.Lmax <= 768 && a.B <= 3 * sm_count())
        return pw ? launch_bwd_xyz<256, 3, false, false, true>(a, st) : launch_bwd_xyz<256, 3, false, false>(a, st);
    // more chains than SMs: single-buffered 128 x 3 (twice the resident CTAs of the
    // double-buffered shape; measured, tools/gpu_bbxs.sh: 4096 x 700 56.0 -> 50.9 us,
    // 512 x 1000 18.2 -> 13.5 us, config 4 96.6 -> 86.2 us)
    if (!env_shape && a.B > sm_count() && a.Lmax > 128)
        return pw ? launch_bwd_xyz<128, 3, false, false, true>(a, st) : launch_bwd_xyz<128, 3, false, false>(a, st);
    const BBShape s = bbx_shape(a.B, a.Lmax);
#define TPL_BBX(NT_, R_) \
    if (s.nt == NT_ && s.rpt == R_) return launch_bwd_xyz<NT_, R_>(a, st);
    TPL_BBX(128, 1) TPL_BBX(128, 3) TPL_BBX(128, 5) TPL_BBX(128, 7)
    TPL_BBX(256, 1) TPL_BBX(256, 3) TPL_BBX(256, 5)
#undef TPL_BBX
    return cudaErrorInvalidConfiguration;
}

#ifdef TPL_PROFILE_PHASES
extern "C" __attribute__((visibility("default"))) int tpl_debug_stamps(unsigned long long* host, int n) {
    return int(cudaMemcpyFromSymbol(host, g_tpl_stamps, sizeof(unsigned long long) * n));
}
extern "C" __attribute__((visibility("default"))) int tpl_debug_stamps_clear(void) {
    static unsigned long long zeros[1 << 16];
    return int(cudaMemcpyToSymbol(g_tpl_stamps, zeros, sizeof(zeros)));
}
#endif

// ---- decoupled (DL) kernels: tiles of a chain on different CTAs
// When to split chains over CTAs.  Measured (tools/gpu_bbx.sh): splitting adds
// a carry exchange per tile and does not reduce the work of the busiest SM, so
// it only pays when few long chains would leave SMs idle (f4: 1 x 20000 fwd+bwd
// 154 -> 42 us, 64 x 2000 23 -> 20 us; 256 x 700 and 4096 x 700 stay
// chain-serial).  TPL_DL=0/1 forces it.
static bool dl_enabled(int B, int Lmax) {
    static int v = -2;
    if (v == -2) {
        const char* e = std::getenv("TPL_DL");
        v = e ? (e[0] == '0' ? 0 : 1) : -1;
    }
    if (v >= 0) return v == 1;
    return B <= 2 * sm_count() && Lmax > 1024;
}
static BBShape env_shape(const char* name) {
    const char* e = std::getenv(name);
    int nt = 0, r = 0;
    if (e && std::sscanf(e, "%dx%d", &nt, &r) == 2) return {nt, r};
    return {0, 0};
}
// Forward: 128 threads; residues per thread chosen so that the batch's tiles
// fill the GPU about twice (small tiles shorten each CTA's serial chain; too
// small tiles pay the scan once more per residue).  TPL_BBF=NTxRPT overrides.
static BBShape bbf_dl_shape(int, int) {
    static const BBShape env = env_shape("TPL_BBF");
    if (env.nt) return env;
    return {128, 5};  // measured best of 1/3/5 for 64 x 2000 and 1 x 20000
}
int bb_dl_max_tiles(int Lmax) { return (Lmax + 127) / 128; }  // slots: every DL tile has >= 128 residues

template <int NT, int RPT, int NS>
static cudaError_t launch_fwd_dl(const BBArgs& a, cudaStream_t st) {
    auto k = bb_forward_dl_kernel<NT, RPT, NS>;
    const size_t sm = fwd_smem<NT>(RPT);
    static LaunchCfg cfg;
    cudaError_t e = ensure_launch_cfg(cfg, k, NT, sm);
    if (e != cudaSuccess) return e;
    const int grid_cap = cfg.cap_now();
    const int max_tiles = (a.Lmax + NT * RPT - 1) / (NT * RPT);
    const long items = long(a.B) * max_tiles;
    const int grid = int(items < grid_cap ? items : grid_cap);  // co-resident: waits only on smaller items
    return launch_pdl(k, grid, NT, sm, st, a.angles, a.lengths, a.B, a.Lmax, a.coords, a.err, a.ws_prefix,
                      max_tiles);
}
template <int NT, int RPT>
static cudaError_t launch_bwd_xyz_dl(const BBArgs& a, cudaStream_t st) {
    auto k = bb_backward_xyz_dl_kernel<NT, RPT>;
    const int tile = NT * RPT;
    const size_t sm = BBSmem<NT>::kData + 2 * round16(16 + 36 * tile + 24) + 2 * round16(16 + 36 * tile) +
                      round16(16 + 12 * tile);
    static LaunchCfg cfg;
    cudaError_t e = ensure_launch_cfg(cfg, k, NT, sm);
    if (e != cudaSuccess) return e;
    const int grid_cap = cfg.cap_now();
    const int max_tiles = (a.Lmax + tile - 1) / tile;
    const long items = long(a.B) * max_tiles;
    const int grid = int(items < grid_cap ? items : grid_cap);
    return launch_pdl(k, grid, NT, sm, st, static_cast<const float*>(a.coords), a.lengths, a.B, a.Lmax,
                      a.grad_coords, a.grad_angles, a.err, a.ws_prefix, max_tiles);
}
// Backward: the same rule with 3 resident CTAs per SM (60 KB of staging each at 128 x 3).
static BBShape bbx_dl_shape(int, int) {
    static const BBShape env = env_shape("TPL_BBXD");
    if (env.nt) return env;
    return {128, 5};
}

template <int NS>
static cudaError_t dispatch_fwd_dl(const BBArgs& a, cudaStream_t st) {
    const BBShape s = bbf_dl_shape(a.B, a.Lmax);
    if (s.nt == 128 && s.rpt == 1) return launch_fwd_dl<128, 1, NS>(a, st);
    if (s.nt == 128 && s.rpt == 3) return launch_fwd_dl<128, 3, NS>(a, st);
    if (s.nt == 128 && s.rpt == 5) return launch_fwd_dl<128, 5, NS>(a, st);
    if (s.nt == 128 && s.rpt == 7) return launch_fwd_dl<128, 7, NS>(a, st);
    if (s.nt == 256 && s.rpt == 3) return launch_fwd_dl<256, 3, NS>(a, st);
    return cudaErrorInvalidConfiguration;
}

template <int NS>
static cudaError_t dispatch_fwd_loss(const BBArgs& a, cudaStream_t st) {  // f1: 128-thread chain-serial shapes
    static const int opts[4] = {1, 3, 5, 7};
    int r = 7;
    for (int i = 0; i < 4; ++i)
        if (128 * opts[i] >= a.Lmax) { r = opts[i]; break; }
    if (r == 1) return launch_fwd<128, 1, NS, true>(a, st);
    if (r == 3) return launch_fwd<128, 3, NS, true>(a, st);
    if (r == 5) return launch_fwd<128, 5, NS, true>(a, st);
    return launch_fwd<128, 7, NS, true>(a, st);
}

// Cluster-split forward shapes (TPL_BBFC=NTxRPTxCL forces one; "0" disables).
template <int NT, int RPT, int CL, int NS>
static cudaError_t launch_fwd_cl(const BBArgs& a, cudaStream_t st) {
    auto k = bb_forward_cl_kernel<NT, RPT, CL, NS>;
    const size_t sm = BBSmem<NT>::kData + round16(48 * CL) + round16(16 + 12 * (NT * RPT + 1)) +
                      round16(16 + 36 * NT * RPT);
    static LaunchCfg cfg;
    cudaError_t e = ensure_launch_cfg(cfg, k, NT, sm);
    if (e != cudaSuccess) return e;
    return launch_cluster(k, a.B * CL, CL, NT, sm, st, a.angles, a.lengths, a.B, a.Lmax, a.coords, a.err);
}
static BBClShape bbfc_shape(int B, int Lmax) {
    static const BBClShape env = [] {
        BBClShape s{0, 0, 0};
        const char* e = std::getenv("TPL_BBFC");
        if (e && std::sscanf(e, "%dx%dx%d", &s.nt, &s.rpt, &s.cl) != 3) s = {-1, 0, 0};
        return s;
    }();
    if (env.nt < 0) return {0, 0, 0};
    if (env.nt > 0) return env.cl * env.nt * env.rpt >= Lmax ? env : BBClShape{0, 0, 0};
    // measured (tools/gpu_cl_sweep.sh, fwd at 1 B200): the split pays where the
    // chain-per-CTA forward needs 7 residues per thread or a second tile and the
    // chains do not already fill the SMs twice -- 64 x 700 5.9 -> 5.0 us,
    // 128 x 1000 10.4 -> 6.8 us, 256 x 900 10.0 -> 8.4 us; 256 x 700 (7.2 vs
    // 7.4 us), 148 x 600 and 512 x 1000 stay chain-per-CTA
    const int sms = sm_count();
    if (Lmax > 640 && Lmax <= 768 && 10 * B <= 14 * sms) return {128, 3, 2};
    if (Lmax > 768 && Lmax <= 1024 && (10 * B <= 14 * sms || (Lmax > 896 && B <= 2 * sms))) return {128, 5, 2};
    return {0, 0, 0};
}
template <int NS>
static cudaError_t dispatch_fwd_cl(const BBArgs& a, BBClShape s, cudaStream_t st) {
#define TPL_BB_CL(NT_, R_, C_) \
    if (s.nt == NT_ && s.rpt == R_ && s.cl == C_) return launch_fwd_cl<NT_, R_, C_, NS>(a, st);
    TPL_BB_CL(128, 3, 2) TPL_BB_CL(128, 5, 2) TPL_BB_CL(128, 7, 2)
#undef TPL_BB_CL
    return cudaErrorInvalidConfiguration;
}

cudaError_t bb_forward_launch(const BBArgs& a, cudaStream_t st) {
    if (!a.loss_out && !a.seg_agg_out && !a.seg_omega_prev && bbp_enabled() && a.Lmax <= bbp_forward_max_L())
        return bbp_forward_launch(a, st);
    // longer chains, more of them than the decoupled kernels' regime: tiles walked per CTA
    if (!a.loss_out && !a.seg_agg_out && !a.seg_omega_prev && bbp_enabled() && a.ns == 1 && !dl_enabled(a.B, a.Lmax))
        return bbp_forward_tiles_launch(a, st);
    if (a.loss_out) return a.ns == 0 ? dispatch_fwd_loss<0>(a, st) : dispatch_fwd_loss<1>(a, st);
    if (a.ns == 2) return dispatch<true, 2>(a, st);  // TPL_ORTHO=2/3: chain-per-CTA shapes only
    if (a.ns == 3) return dispatch<true, 3>(a, st);
    if (!a.seg_agg_out && dl_enabled(a.B, a.Lmax))
        return a.ns == 0 ? dispatch_fwd_dl<0>(a, st) : dispatch_fwd_dl<1>(a, st);
    if (!a.seg_agg_out) {
        const BBClShape cs = bbfc_shape(a.B, a.Lmax);
        if (cs.nt > 0) return a.ns == 0 ? dispatch_fwd_cl<0>(a, cs, st) : dispatch_fwd_cl<1>(a, cs, st);
    }
    return a.ns == 0 ? dispatch<true, 0>(a, st) : dispatch<true, 1>(a, st);
}
cudaError_t bb_backward_launch(const BBArgs& a, cudaStream_t st) {
    return a.ns == 0 ? dispatch<false, 0>(a, st) : dispatch<false, 1>(a, st);
}

}  // namespace tpl
