// fullatom.cu -- batched full-atom model (§2) on sm_100a.
//
// Forward: the backbone chain N_j -> CA_j -> C_j -> N_{j+1} is the same
// associative transform product as the backbone model (same §3 constants,
// reading Q12), computed with the block-wide affine prefix scan.  After the
// scan every residue owns its global N, CA and C frames, and places its
// side-chain rigid groups locally:
//     M_g = M_parent R_x(pre) R(alpha_g, theta_g, d_g),  r = M_owner r°
// from the residue-type table staged in shared memory.  Atoms of a chain are
// packed residue after residue; per-residue output offsets come from a
// block-wide integer scan of the per-type atom counts, fused into the pass.
//
// Backward (Eq. 1): dL/dalpha_n = e_n . sum_{k in subtree(n)} (r_k - o_n) x g_k
// (e_n = rotation axis = x-axis of frame n, o_n its origin).  With atoms
// ordered N, CA, side chain, C, O the subtrees of the backbone nodes are
// suffixes of the chain: phi_j -> {residue j minus N} + later residues,
// psi_j -> {C-owned atoms of j} + later, omega_{j-1} -> residue j + later.
// Chi subtrees are residue-local: a side-chain branch is walked from its tip
// back to the CA frame (frames undone with the rigid inverse of each bond)
// accumulating the local sums.  One reverse suffix scan per chain: O(L).
// fa_backward_xyz_kernel computes the same from the forward's coordinates:
// every axis is the vector between two frame-origin atoms, so no angle, trig
// or transform is needed (the path the autograd layer takes).
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "packed.cuh"

namespace tpl {
// added to a thread's atom count when its residue type is out of range: far above any
// tile's atom count (< 2^16), and 512 threads x 2^21 stay below 2^31, so the tile's
// total (block total minus the carry) flags it without overflow
constexpr int kBadRestype = 1 << 21;

__host__ __device__ constexpr int r16(int x) { return (x + 15) & ~15; }

template <int NT>
struct FASmem {
    static constexpr int NW = NT / 32;
    static constexpr int kBar = 0;
    static constexpr int kScan = 16;                         // 2*NW*12 floats
    static constexpr int kSuf = kScan + 2 * NW * 12 * 4;     // 2*NW*6 + 8 floats
    static constexpr int kInt = kSuf + (2 * NW * 6 + 8) * 4;  // NW ints
    static constexpr int kTotal = r16(kInt + NW * 4);        // 12 floats
    static constexpr int kMisc = kTotal + 48;                // 16 floats / ints
    static constexpr int kTable = r16(kMisc + 64);           // n_types * sizeof(FAType)
};

template <int NT, int RPT>
struct FALayout {
    static constexpr int TILE = NT * RPT;
    static constexpr int ang_bytes = r16(16 + 32 * (TILE + 1));
    static constexpr int rt_bytes = r16(16 + TILE + 1);
    // atom staging (coords out, or grad_coords in) sized at launch: 16 + 12*maxatoms*TILE
    // grad-angle staging (backward): 16 + 32*TILE
    static constexpr int go_bytes = r16(16 + 32 * TILE);
};

__device__ __forceinline__ void cross_acc(float s[6], float qx, float qy, float qz, float g0, float g1, float g2) {
    s[0] += g0;
    s[1] += g1;
    s[2] += g2;
    s[3] += fmaf(qy, g2, -qz * g1);
    s[4] += fmaf(qz, g0, -qx * g2);
    s[5] += fmaf(qx, g1, -qy * g0);
}

// e . (T - o x S) for a 6-vector (S, T)
__device__ __forceinline__ float axis_moment(float ex, float ey, float ez, float ox, float oy, float oz,
                                             const float s[6]) {
    const float c0 = s[3] - fmaf(oy, s[2], -oz * s[1]);
    const float c1 = s[4] - fmaf(oz, s[0], -ox * s[2]);
    const float c2 = s[5] - fmaf(ox, s[1], -oy * s[0]);
    return fmaf(ex, c0, fmaf(ey, c1, ez * c2));
}

// a residue type's header (counts and origin atoms) as two 16-byte loads
struct FAHead {
    int n_groups, n_atoms, n_N, n_CA, first_C, iN, iCA, iC;
};
__device__ __forceinline__ FAHead load_head(const FAType& T) {
    FAHead h;
    const int4* s = reinterpret_cast<const int4*>(&T);
    int4* d = reinterpret_cast<int4*>(&h);
    d[0] = s[0];
    d[1] = s[1];
    return h;
}

// a side-chain group's constants as four independent 16-byte loads (the fields' latency
// chain -- parent, slot, angle, bond constants, atom range -- is one round trip)
__device__ __forceinline__ FAGroup load_group(const FAGroup& g) {
    FAGroup r;
    const int4* s = reinterpret_cast<const int4*>(&g);
    int4* d = reinterpret_cast<int4*>(&r);
    d[0] = s[0]; d[1] = s[1]; d[2] = s[2]; d[3] = s[3];
    return r;
}

// r° of atom k as one 16-byte load (the table row is float[4], 16-byte aligned)
__device__ __forceinline__ float4 r0_of(const FAType& T, int k) { return *reinterpret_cast<const float4*>(T.r[k]); }
__device__ __forceinline__ void apply4(const Aff& M, float4 r, float& ox, float& oy, float& oz) {
    apply(M, r.x, r.y, r.z, ox, oy, oz);
}

// Backbone chunk of one thread: residues [rl0, rl0+RPT) of the tile.  Returns the
// chunk aggregate (product of all its transforms) in M and keeps the bonds' (sin,
// cos); after the scan the thread walks its residues again from its prefix, so the
// per-residue N, CA and C frames are never held across the scan.
template <int RPT>
__device__ __forceinline__ void fa_chunk(const float* s_ang, int rl0, int r0, int n, Aff& M, float (&bs)[RPT][3],
                                         float (&bc)[RPT][3]) {
    M = aff_identity();
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int rl = rl0 + q;
        const int j = r0 + rl;
        if (rl < n) {
            // omega_{j-1} (C_{j-1} -> N_j; R_0 = I for j = 0), phi_j (-> CA_j), psi_j (-> C_j)
            const float x[3] = {j > 0 ? s_ang[8 * rl - 6] : 0.f, s_ang[8 * rl + 0], s_ang[8 * rl + 1]};
            tpl_sincos_n<3>(x, bs[q], bc[q]);
            if (j > 0) aff_bond_bb<0>(M, bc[q][0], bs[q][0]);
            aff_bond_bb<1>(M, bc[q][1], bs[q][1]);
            aff_bond_bb<2>(M, bc[q][2], bs[q][2]);
        }
    }
}

// kTS: residue table staged in shared memory (else read through L1);
// kMinB: __launch_bounds__ min blocks (register budget).  TPL_FAF tunes them.
template <int NT, int RPT, int kNS, bool kTS = true, int kMinB = 2, bool kDBI = true>
__global__ void __launch_bounds__(NT, kMinB) fa_forward_kernel(FAArgs a, int stage_atoms_per_res) {
    constexpr int TILE = NT * RPT;
    using S = FASmem<NT>;
    using Lay = FALayout<NT, RPT>;
    extern __shared__ __align__(16) char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::kBar);
    float* s_scan = reinterpret_cast<float*>(smem + S::kScan);
    int* s_int = reinterpret_cast<int*>(smem + S::kInt);
    float* s_total = reinterpret_cast<float*>(smem + S::kTotal);
    int* s_misc = reinterpret_cast<int*>(smem + S::kMisc);
    const FAType* __restrict__ s_types = kTS ? reinterpret_cast<const FAType*>(smem + S::kTable) : a.types;
    // kDBI: tile inputs double-buffered (angles + residue types; bar[0] / bar[1]): tile
    // t + 1's loads fly while tile t computes
    char* s_in_base = smem + S::kTable + (kTS ? r16(a.n_types * int(sizeof(FAType))) : 0);
    char* s_out_base = s_in_base + 2 * (Lay::ang_bytes + Lay::rt_bytes);

    const int b = blockIdx.x;
    const int tid = threadIdx.x;
    unsigned phase = 0;  // bit i: the parity bar[i] waits for next
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        fence_barrier_init();
        // the residue table is immutable after tpl_tables_create: it may be
        // fetched before pdl_wait, overlapping the previous kernel's tail
        if (kTS) {
            const unsigned tb = unsigned(a.n_types * sizeof(FAType));
            mbar_arrive_expect_tx(bar, tb);
            bulk_g2s(smem + S::kTable, a.types, tb, bar);
        }
    }
    if (tid == 0 && prefetch_regime(a.B)) {  // cold inputs into L2 under the previous kernel's tail (safe before the wait)
        const Span pa = make_span(a.angles + (size_t)b * a.Lmax * kFASlots, a.Lmax * 32);
        if (pa.mid > 0) prefetch_l2(pa.g + pa.head, unsigned(pa.mid));
    }
    pdl_wait();
    pdl_trigger();  // launched with PDL only for <= 2 chains per SM, where every CTA is resident
    const int L = a.lengths[b];
    __syncthreads();
    if (kTS) {
        mbar_wait(bar, phase);  // also before any early exit: no bulk copy may outlive the CTA
        phase ^= 1u;
    }
    if (L < 1 || L > a.Lmax) {
        if (tid == 0) atomicOr(a.err, ERR_LENGTH);
        return;
    }

    Aff carry = aff_identity();
    QT carryq = qt_identity();  // policies 1 and 3: the chain prefix in (quaternion, translation) form
    int carry_atoms = 0;
    const int rl0 = tid * RPT;
    float* coords = a.coords + (size_t)b * a.atom_stride * 3;
    auto in_spans = [&](int r0, Span& sa, Span& sr) {
        const int n = min(TILE, L - r0), pre = r0 > 0 ? 1 : 0;
        sa = make_span(a.angles + ((size_t)b * a.Lmax + r0 - pre) * kFASlots, (n + pre) * 32);
        sr = make_span(a.restype + (size_t)b * a.Lmax + r0, n);
    };
    auto issue_in = [&](int r0, int buf) {  // thread 0
        Span sa, sr;
        in_spans(r0, sa, sr);
        char* base = s_in_base + buf * (Lay::ang_bytes + Lay::rt_bytes);
        mbar_arrive_expect_tx(bar + buf, unsigned(sa.mid + sr.mid));
        span_load_bulk(sa, base, bar + buf);
        span_load_bulk(sr, base + Lay::ang_bytes, bar + buf);
    };
    // before an early return: the prefetch in flight must land first (no bulk copy may
    // outlive the CTA), and the stores drain
    auto drain = [&](int r0, int buf) {
        if (kDBI && r0 + TILE < L) mbar_wait(bar + (buf ^ 1), (phase >> (buf ^ 1)) & 1u);
        bulk_wait_all();
    };
    if (tid == 0) issue_in(0, 0);
    for (int r0 = 0, buf = 0; r0 < L; r0 += TILE, buf ^= kDBI ? 1 : 0) {
        const int n = min(TILE, L - r0);
        const int pre = r0 > 0 ? 1 : 0;
        Span sa, sr;
        in_spans(r0, sa, sr);
        char* s_ang_base = s_in_base + buf * (Lay::ang_bytes + Lay::rt_bytes);
        char* s_rt_base = s_ang_base + Lay::ang_bytes;
        // the other buffer (single-buffered: this one) was last read by tile t - 1,
        // before its closing barrier
        if (kDBI && tid == 0 && r0 + TILE < L) issue_in(r0 + TILE, buf ^ 1);
        if (!kDBI && tid == 0 && r0 > 0) issue_in(r0, 0);
        if (tid == 0) bulk_wait_read_all();  // the output staging is free again
        span_load_edges_f32(sa, s_ang_base);
        span_load_edges_u8(sr, s_rt_base);
        mbar_wait(bar + buf, (phase >> buf) & 1u);
        phase ^= 1u << buf;
        __syncthreads();
        const float* s_ang = reinterpret_cast<const float*>(s_ang_base + sa.mis()) + 8 * pre;
        const unsigned char* s_rt = reinterpret_cast<const unsigned char*>(s_rt_base + sr.mis());

        // residue types, atom counts, validity
        int cnt = 0;
        bool bad = false;
        int typ[RPT];
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int rl = rl0 + q;
            typ[q] = 0;
            if (rl < n) {
                const int t = s_rt[rl];
                if (t >= a.n_types) bad = true;
                else {
                    typ[q] = t;
                    cnt += s_types[t].n_atoms;
                }
            }
        }
        // a bad restype rides in the atom-count scan (kBadRestype >> any tile's atom count), so
        // the block-uniform early return needs no barrier of its own
        int tile_end_atoms;
        const int off0 = block_exclusive_sum_int<NT>(cnt + (bad ? kBadRestype : 0), carry_atoms, s_int, &tile_end_atoms);
        if (tile_end_atoms - carry_atoms >= kBadRestype) {
            if (tid == 0) {
                atomicOr(a.err, ERR_RESTYPE);
                drain(r0, buf);
            }
            return;
        }
        if (tile_end_atoms > a.atom_stride) {  // the chain's atoms do not fit its row: flag, skip
            if (tid == 0) {
                atomicOr(a.err, ERR_STRIDE);
                drain(r0, buf);
            }
            return;
        }

        Aff M;
        float bs[RPT][3], bc[RPT][3];
        fa_chunk<RPT>(s_ang, rl0, r0, n, M, bs, bc);
        if (kNS == 2) aff_orthonormalize(M);  // the quaternion scans (1, 3) renormalise at the extraction
        // policies 1 / 3: the (quaternion, translation) scan of packed.cuh (renormalised every
        // combine, 7 floats per shuffle level; reading Q25); 0 / 2: the 3x4 affine scan
        Aff P;
        if (kNS == 1 || kNS == 3) {
            P = block_exclusive_scan_qt_carry<NT>(M, s_scan, carryq);
        } else {
            P = block_exclusive_scan<NT, kNS>(M, carry, s_scan, s_total);
            carry = load_aff(s_total);
        }

        const int n_tile_atoms = tile_end_atoms - carry_atoms;
        const Span so = make_span(coords + (size_t)carry_atoms * 3, n_tile_atoms * 12);
        float* s_out = reinterpret_cast<float*>(s_out_base + so.mis());
        int off = off0 - carry_atoms;  // tile-local atom index of the thread's first atom
        Aff Gb = P;                     // the chain walked again from the thread's prefix
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int rl = rl0 + q;
            if (rl < n) {
                const FAType& T = s_types[typ[q]];
                const FAHead h = load_head(T);
                if (r0 + rl > 0) aff_bond_bb<0>(Gb, bc[q][0], bs[q][0]);
                const Aff gN = Gb;
                aff_bond_bb<1>(Gb, bc[q][1], bs[q][1]);
                const Aff gCA = Gb;
                aff_bond_bb<2>(Gb, bc[q][2], bs[q][2]);
                const Aff gC = Gb;
                const float* ang = s_ang + 8 * rl;
                float* o = s_out + 3 * off;
                int k = 0;
                for (; k < h.n_N; ++k) apply4(gN, r0_of(T, k), o[3 * k], o[3 * k + 1], o[3 * k + 2]);
                for (; k < h.n_N + h.n_CA; ++k)
                    apply4(gCA, r0_of(T, k), o[3 * k], o[3 * k + 1], o[3 * k + 2]);
                Aff G = gCA;
                for (int g = 0; g < h.n_groups; ++g) {
                    const FAGroup gr = load_group(T.g[g]);
                    if (gr.parent < 0) {
                        G = gCA;
                        if (gr.has_pre) aff_rot_x(G, gr.cb, gr.sb);
                    }
                    float s, c;
                    if (gr.slot >= 0) tpl_sincos(ang[gr.slot], &s, &c);
                    else { s = gr.sa; c = gr.ca; }
                    const BondC bc{gr.ct, gr.st, gr.d};
                    aff_bond(G, c, s, bc);
#pragma unroll 2
                    for (k = gr.first_atom; k < gr.end_atom; ++k)
                        apply4(G, r0_of(T, k), o[3 * k], o[3 * k + 1], o[3 * k + 2]);
                }
                for (k = h.first_C; k < h.n_atoms; ++k)
                    apply4(gC, r0_of(T, k), o[3 * k], o[3 * k + 1], o[3 * k + 2]);
                off += h.n_atoms;
            }
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            span_store_bulk(so, s_out_base);
            bulk_commit();
        }
        span_store_edges_f32(so, s_out_base);
        carry_atoms = tile_end_atoms;
    }
    (void)s_misc;
    (void)stage_atoms_per_res;
    if (tid == 0) bulk_wait_all();
}

// Residue-local backward: positions of every atom of one residue, the
// chi gradients (written to go[slot]) and the residue's sums needed by the
// backbone gradients.  CA-relative moments keep the local sums accurate.
struct ResSums {
    float all[6];  // S, T^CA over all atoms of the residue
    float nN[6];   // over N-owned atoms
    float cC[6];   // over C-owned atoms
};

__device__ __forceinline__ void fa_residue_backward(const FAType& T, const float* ang, const Aff& gN, const Aff& gCA,
                                                    const Aff& gC, const float* gk, float* go, ResSums& R) {
#pragma unroll
    for (int k = 0; k < 6; ++k) R.all[k] = R.nN[k] = R.cC[k] = 0.f;
    const float cx = gCA.t0, cy = gCA.t1, cz = gCA.t2;
    const FAHead h = load_head(T);
    int k = 0;
    for (; k < h.n_N; ++k) {
        float x, y, z;
        apply4(gN, r0_of(T, k), x, y, z);
        cross_acc(R.nN, x - cx, y - cy, z - cz, gk[3 * k], gk[3 * k + 1], gk[3 * k + 2]);
    }
    for (; k < h.n_N + h.n_CA; ++k) {
        float x, y, z;
        apply4(gCA, r0_of(T, k), x, y, z);
        cross_acc(R.all, x - cx, y - cy, z - cz, gk[3 * k], gk[3 * k + 1], gk[3 * k + 2]);
    }
    for (k = h.first_C; k < h.n_atoms; ++k) {
        float x, y, z;
        apply4(gC, r0_of(T, k), x, y, z);
        cross_acc(R.cC, x - cx, y - cy, z - cz, gk[3 * k], gk[3 * k + 1], gk[3 * k + 2]);
    }
    // side-chain branches: forward to the branch tip, then walk back
    int g0 = 0;
    while (g0 < h.n_groups) {
        int g1 = g0;
        while (g1 + 1 < h.n_groups && T.g[g1 + 1].parent == g1) ++g1;
        Aff G = gCA;
        if (T.g[g0].has_pre) aff_rot_x(G, T.g[g0].cb, T.g[g0].sb);
        for (int g = g0; g <= g1; ++g) {
            const FAGroup gr = load_group(T.g[g]);
            float s, c;
            if (gr.slot >= 0) tpl_sincos(ang[gr.slot], &s, &c);
            else { s = gr.sa; c = gr.ca; }
            aff_bond(G, c, s, BondC{gr.ct, gr.st, gr.d});
        }
        float br[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int g = g1; g >= g0; --g) {
            const FAGroup gr = load_group(T.g[g]);
            for (k = gr.first_atom; k < gr.end_atom; ++k) {
                float x, y, z;
                apply4(G, r0_of(T, k), x, y, z);
                cross_acc(br, x - cx, y - cy, z - cz, gk[3 * k], gk[3 * k + 1], gk[3 * k + 2]);
            }
            if (gr.slot >= 0) go[gr.slot] = axis_moment(G.r00, G.r10, G.r20, G.t0 - cx, G.t1 - cy, G.t2 - cz, br);
            if (g > g0) {
                float s, c;
                if (gr.slot >= 0) tpl_sincos(ang[gr.slot], &s, &c);
                else { s = gr.sa; c = gr.ca; }
                aff_unbond(G, c, s, BondC{gr.ct, gr.st, gr.d});
            }
        }
#pragma unroll
        for (int q = 0; q < 6; ++q) R.all[q] += br[q];
        g0 = g1 + 1;
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) R.all[q] += R.nN[q] + R.cC[q];
}

template <int NT, int RPT, int kNS>
__global__ void __launch_bounds__(NT, 3) fa_backward_kernel(FAArgs a, int stage_atoms_per_res) {
    constexpr int TILE = NT * RPT;
    using S = FASmem<NT>;
    using Lay = FALayout<NT, RPT>;
    extern __shared__ __align__(16) char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::kBar);
    float* s_scan = reinterpret_cast<float*>(smem + S::kScan);
    float* s_suf = reinterpret_cast<float*>(smem + S::kSuf);
    int* s_int = reinterpret_cast<int*>(smem + S::kInt);
    float* s_total = reinterpret_cast<float*>(smem + S::kTotal);
    float* s_misc = reinterpret_cast<float*>(smem + S::kMisc);
    const FAType* s_types = reinterpret_cast<const FAType*>(smem + S::kTable);
    char* s_ang_base = smem + S::kTable + r16(a.n_types * int(sizeof(FAType)));
    char* s_rt_base = s_ang_base + Lay::ang_bytes;
    char* s_go_base = s_rt_base + Lay::rt_bytes;
    char* s_g_base = s_go_base + Lay::go_bytes;

    const int b = blockIdx.x;
    const int tid = threadIdx.x;
    unsigned phase = 0;  // bit i: the parity bar[i] waits for next
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        fence_barrier_init();
        // the residue table is immutable after tpl_tables_create: it may be
        // fetched before pdl_wait, overlapping the previous kernel's tail
        const unsigned tb = unsigned(a.n_types * sizeof(FAType));
        mbar_arrive_expect_tx(bar, tb);
        bulk_g2s(smem + S::kTable, a.types, tb, bar);
    }
    pdl_wait();  // the dependent launches when this grid exits (early triggers cost SM slots)
    const int L = a.lengths[b];
    __syncthreads();
    mbar_wait(bar, phase);  // also before any early exit: no bulk copy may outlive the CTA
    phase ^= 1u;
    if (L < 1 || L > a.Lmax) {
        if (tid == 0) atomicOr(a.err, ERR_LENGTH);
        return;
    }

    const int n_tiles = (L + TILE - 1) / TILE;
    const int rl0 = tid * RPT;
    float* pref = a.ws_prefix + (size_t)b * a.max_tiles * 16;

    // ---- phase A: prefix transform and atom offset at every tile start
    if (n_tiles > 1) {
        Aff carry = aff_identity();
        int carry_atoms = 0;
        for (int t = 0; t + 1 < n_tiles; ++t) {
            const int r0 = t * TILE;
            const int pre = r0 > 0 ? 1 : 0;
            const Span sa = make_span(a.angles + ((size_t)b * a.Lmax + r0 - pre) * kFASlots, (TILE + pre) * 32);
            const Span sr = make_span(a.restype + (size_t)b * a.Lmax + r0, TILE);
            if (tid == 0) {
                mbar_arrive_expect_tx(bar, unsigned(sa.mid + sr.mid));
                span_load_bulk(sa, s_ang_base, bar);
                span_load_bulk(sr, s_rt_base, bar);
            }
            span_load_edges_f32(sa, s_ang_base);
            span_load_edges_u8(sr, s_rt_base);
            mbar_wait(bar, phase);
            phase ^= 1u;
            __syncthreads();
            const float* s_ang = reinterpret_cast<const float*>(s_ang_base + sa.mis()) + 8 * pre;
            const unsigned char* s_rt = reinterpret_cast<const unsigned char*>(s_rt_base + sr.mis());
            int cnt = 0;
            bool bad = false;
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const int t2 = s_rt[rl0 + q];
                if (t2 >= a.n_types) bad = true;
                else cnt += s_types[t2].n_atoms;
            }
            if (__syncthreads_or(bad)) {
                if (tid == 0) atomicOr(a.err, ERR_RESTYPE);
                return;
            }
            int tile_end;
            block_exclusive_sum_int<NT>(cnt, carry_atoms, s_int, &tile_end);
            if (tile_end > a.atom_stride) {
                if (tid == 0) atomicOr(a.err, ERR_STRIDE);
                return;
            }
            Aff M;
            float bs[RPT][3], bc[RPT][3];
            fa_chunk<RPT>(s_ang, rl0, r0, TILE, M, bs, bc);
            if (kNS >= 1) aff_orthonormalize(M);
            block_exclusive_scan<NT, kNS>(M, carry, s_scan, s_total);
            carry = load_aff(s_total);
            carry_atoms = tile_end;
            if (tid < 12) pref[(t + 1) * 16 + tid] = s_total[tid];
            if (tid == 12) pref[(t + 1) * 16 + 12] = __int_as_float(tile_end);
        }
        __syncthreads();
    }

    // ---- phase B: tiles last to first
    float carry6[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float omega_next = 0.f;
    const float* gcb = a.grad_coords + (size_t)b * a.atom_stride * 3;
    for (int t = n_tiles - 1; t >= 0; --t) {
        const int r0 = t * TILE;
        const int n = min(TILE, L - r0);
        const int pre = r0 > 0 ? 1 : 0;
        const Aff carry = (t == 0) ? aff_identity() : load_aff(pref + t * 16);
        const int carry_atoms = (t == 0) ? 0 : __float_as_int(pref[t * 16 + 12]);
        const Span sa = make_span(a.angles + ((size_t)b * a.Lmax + r0 - pre) * kFASlots, (n + pre) * 32);
        const Span sr = make_span(a.restype + (size_t)b * a.Lmax + r0, n);
        if (tid == 0) {
            bulk_wait_read_all();
            mbar_arrive_expect_tx(bar, unsigned(sa.mid + sr.mid));
            span_load_bulk(sa, s_ang_base, bar);
            span_load_bulk(sr, s_rt_base, bar);
        }
        span_load_edges_f32(sa, s_ang_base);
        span_load_edges_u8(sr, s_rt_base);
        mbar_wait(bar, phase);
        phase ^= 1u;
        __syncthreads();
        const float* s_ang = reinterpret_cast<const float*>(s_ang_base + sa.mis()) + 8 * pre;
        const unsigned char* s_rt = reinterpret_cast<const unsigned char*>(s_rt_base + sr.mis());

        int cnt = 0;
        bool bad = false;
        int typ[RPT];
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int rl = rl0 + q;
            typ[q] = 0;
            if (rl < n) {
                const int t2 = s_rt[rl];
                if (t2 >= a.n_types) bad = true;
                else {
                    typ[q] = t2;
                    cnt += s_types[t2].n_atoms;
                }
            }
        }
        int tile_end;  // a bad restype rides in the scan (as the forward)
        const int off0 = block_exclusive_sum_int<NT>(cnt + (bad ? kBadRestype : 0), carry_atoms, s_int, &tile_end);
        if (tile_end - carry_atoms >= kBadRestype) {
            if (tid == 0) {
                atomicOr(a.err, ERR_RESTYPE);
                bulk_wait_all();
            }
            return;
        }
        if (tile_end > a.atom_stride) {
            if (tid == 0) {
                atomicOr(a.err, ERR_STRIDE);
                bulk_wait_all();
            }
            return;
        }
        // stage grad_coords of the tile's atoms (second round on the barrier)
        const Span sg = make_span(gcb + (size_t)carry_atoms * 3, (tile_end - carry_atoms) * 12);
        if (tid == 0) {
            mbar_arrive_expect_tx(bar, unsigned(sg.mid));
            span_load_bulk(sg, s_g_base, bar);
        }
        span_load_edges_f32(sg, s_g_base);

        Aff M;
        float bs[RPT][3], bc[RPT][3];
        fa_chunk<RPT>(s_ang, rl0, r0, n, M, bs, bc);
        if (kNS >= 1) aff_orthonormalize(M);
        const Aff P = block_exclusive_scan<NT, kNS>(M, carry, s_scan, s_total);  // contains __syncthreads
        mbar_wait(bar, phase);
        phase ^= 1u;
        __syncthreads();
        const float* s_g = reinterpret_cast<const float*>(s_g_base + sg.mis());
        float* s_go = reinterpret_cast<float*>(s_go_base + 16);  // 16-aligned; stored with plain edges below

        // residue pass: positions, chi gradients, residue sums
        float axN[RPT][6], axCA[RPT][6], axC[RPT][6];  // e (3) and o - CA (3) of the three backbone nodes
        float cax[RPT][3];
        ResSums RS[RPT];
        float thr[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        int off = off0 - carry_atoms;
        Aff Gb = P;  // the chain walked again from the thread's prefix
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int rl = rl0 + q;
            if (rl < n) {
                const FAType& T = s_types[typ[q]];
                const FAHead h = load_head(T);
                if (r0 + rl > 0) aff_bond_bb<0>(Gb, bc[q][0], bs[q][0]);
                const Aff gN = Gb;
                aff_bond_bb<1>(Gb, bc[q][1], bs[q][1]);
                const Aff gCA = Gb;
                aff_bond_bb<2>(Gb, bc[q][2], bs[q][2]);
                const Aff gC = Gb;
                float* go = s_go + 8 * rl;
                go[0] = go[1] = 0.f;
#pragma unroll
                for (int s = 3; s < 8; ++s) go[s] = 0.f;
                fa_residue_backward(T, s_ang + 8 * rl, gN, gCA, gC, s_g + 3 * off, go, RS[q]);
                cax[q][0] = gCA.t0; cax[q][1] = gCA.t1; cax[q][2] = gCA.t2;
                axN[q][0] = gN.r00; axN[q][1] = gN.r10; axN[q][2] = gN.r20;
                axN[q][3] = gN.t0 - gCA.t0; axN[q][4] = gN.t1 - gCA.t1; axN[q][5] = gN.t2 - gCA.t2;
                axCA[q][0] = gCA.r00; axCA[q][1] = gCA.r10; axCA[q][2] = gCA.r20;
                axCA[q][3] = 0.f; axCA[q][4] = 0.f; axCA[q][5] = 0.f;
                axC[q][0] = gC.r00; axC[q][1] = gC.r10; axC[q][2] = gC.r20;
                axC[q][3] = gC.t0 - gCA.t0; axC[q][4] = gC.t1 - gCA.t1; axC[q][5] = gC.t2 - gCA.t2;
                // absolute moment of the residue: T = T^CA + CA x S
                const float* s6 = RS[q].all;
                thr[0] += s6[0]; thr[1] += s6[1]; thr[2] += s6[2];
                thr[3] += s6[3] + fmaf(gCA.t1, s6[2], -gCA.t2 * s6[1]);
                thr[4] += s6[4] + fmaf(gCA.t2, s6[0], -gCA.t0 * s6[2]);
                thr[5] += s6[5] + fmaf(gCA.t0, s6[1], -gCA.t1 * s6[0]);
                off += h.n_atoms;
            }
        }
        float suf[6], tot6[6];
        block_exclusive_suffix6<NT>(thr, carry6, s_suf, suf, tot6);

        // backbone gradients, residues last to first; suf = sums (absolute) over later residues
#pragma unroll
        for (int q = RPT - 1; q >= 0; --q) {
            const int rl = rl0 + q;
            const int j = r0 + rl;
            if (rl < n) {
                float* go = s_go + 8 * rl;
                const float cx = cax[q][0], cy = cax[q][1], cz = cax[q][2];
                // later residues as CA-relative moments: T^CA = T - CA x S
                float aft[6];
                aft[0] = suf[0]; aft[1] = suf[1]; aft[2] = suf[2];
                aft[3] = suf[3] - fmaf(cy, suf[2], -cz * suf[1]);
                aft[4] = suf[4] - fmaf(cz, suf[0], -cx * suf[2]);
                aft[5] = suf[5] - fmaf(cx, suf[1], -cy * suf[0]);
                float s6[6];
                // psi_j: C-owned atoms + later residues, axis through C
#pragma unroll
                for (int k = 0; k < 6; ++k) s6[k] = RS[q].cC[k] + aft[k];
                go[1] = axis_moment(axC[q][0], axC[q][1], axC[q][2], axC[q][3], axC[q][4], axC[q][5], s6);
                // phi_j: residue minus N-owned + later, axis through CA
#pragma unroll
                for (int k = 0; k < 6; ++k) s6[k] = RS[q].all[k] - RS[q].nN[k] + aft[k];
                go[0] = axis_moment(axCA[q][0], axCA[q][1], axCA[q][2], 0.f, 0.f, 0.f, s6);
                // omega_{j-1}: residue + later, axis through N
                if (j > 0) {
#pragma unroll
                    for (int k = 0; k < 6; ++k) s6[k] = RS[q].all[k] + aft[k];
                    const float gw = axis_moment(axN[q][0], axN[q][1], axN[q][2], axN[q][3], axN[q][4], axN[q][5], s6);
                    if (rl > 0) s_go[8 * (rl - 1) + 2] = gw;
                    else s_misc[0] = gw;
                }
                // fold this residue into the suffix
                const float* r6 = RS[q].all;
                suf[0] += r6[0]; suf[1] += r6[1]; suf[2] += r6[2];
                suf[3] += r6[3] + fmaf(cy, r6[2], -cz * r6[1]);
                suf[4] += r6[4] + fmaf(cz, r6[0], -cx * r6[2]);
                suf[5] += r6[5] + fmaf(cx, r6[1], -cy * r6[0]);
            }
        }
        if (tid == 0) s_go[8 * (n - 1) + 2] = (r0 + n == L) ? 0.f : omega_next;
        __syncthreads();
        // store the tile's grad record [n][8] (32 B per residue: 16-B aligned when the row base is)
        {
            float* dst = a.grad_angles + ((size_t)b * a.Lmax + r0) * kFASlots;
            if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
                fence_proxy_async_smem();
                __syncthreads();
                if (tid == 0) {
                    bulk_s2g(dst, s_go, unsigned(n * 32));
                    bulk_commit();
                }
            } else {
                for (int i = tid; i < n * 8; i += NT) dst[i] = s_go[i];
            }
        }
        omega_next = s_misc[0];
#pragma unroll
        for (int k = 0; k < 6; ++k) carry6[k] = tot6[k];
        __syncthreads();
    }
    (void)stage_atoms_per_res;
    if (tid == 0) bulk_wait_all();
}

// ---------------------------------------------------------------------------
// Backward from the forward's coordinates.  Every angle rotates a frame whose
// origin is an atom (table check xyz_ok), about the bond from the parent
// frame's origin atom: e = unit(r_origin - r_parent_origin), o = r_origin.
//   phi_j: N_j -> CA_j through CA_j, subtree {residue j minus N-owned} + later
//   psi_j: CA_j -> C_j through C_j, subtree {C-owned atoms of j} + later
//   omega_j: C_j -> N_{j+1} through N_{j+1}, subtree {residues > j}
//   chi_g: parent origin -> group origin, subtree = groups g..(branch end)
// No angles and no transforms are read.  Residue-local sums are taken about
// CA_j, the chain suffix about the tile's first atom (moments stay small).
// Tile atom offsets come from a pre-pass over the chain's residue types.
template <int NT>
struct FAXSmem {
    static constexpr int NW = NT / 32;
    static constexpr int kBar = 0;                   // 4 mbarriers: 2 tile buffers, table, chain restype
    static constexpr int kSuf = 32;                         // 2*NW*6 + 8 floats
    static constexpr int kInt = kSuf + (2 * NW * 6 + 8) * 4;  // NW ints
    static constexpr int kTable = r16(kInt + NW * 4);
};

struct FAXTile {  // byte layout of one tile buffer
    int x, g, total;
};
__host__ __device__ inline FAXTile fax_tile_layout(int tile, int max_atoms) {
    FAXTile l;
    l.x = 0;
    l.g = l.x + r16(16 + 12 * max_atoms * tile);
    l.total = l.g + r16(16 + 12 * max_atoms * tile);
    return l;
}

// kDB: double-buffered tiles (prefetch tile t-1 during t); kTabSmem: the
// residue table staged in shared memory (else read through L1).  Both cost
// shared memory, i.e. resident CTAs; tools/gpu_fax.sh measures the variants.
__host__ __device__ constexpr int fax_table_bytes(bool tab_smem, int n_types) {
    return tab_smem ? r16(n_types * int(sizeof(FAType))) : 0;
}

template <int NT, int RPT, bool kDB, bool kTabSmem>
__global__ void __launch_bounds__(NT) fa_backward_xyz_kernel(FAArgs a, int max_tiles) {
    constexpr int TILE = NT * RPT;
    static_assert(TILE * kMaxAtomsPerRes < 65536, "tile-relative atom offsets are 16-bit");
    using S = FAXSmem<NT>;
    extern __shared__ __align__(16) char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::kBar);
    float* s_suf = reinterpret_cast<float*>(smem + S::kSuf);
    int* s_int = reinterpret_cast<int*>(smem + S::kInt);
    const FAType* __restrict__ s_types =
        kTabSmem ? reinterpret_cast<const FAType*>(smem + S::kTable) : a.types;
    int* s_off = reinterpret_cast<int*>(smem + S::kTable + fax_table_bytes(kTabSmem, a.n_types));
    // tile-relative atom offsets fit 16 bits (< TILE * kMaxAtomsPerRes <= 8192)
    unsigned short* s_roff = reinterpret_cast<unsigned short*>(reinterpret_cast<char*>(s_off) + r16(4 * (max_tiles + 1)));
    char* s_rt_base = reinterpret_cast<char*>(s_roff) + r16(2 * max_tiles * NT);  // the chain's restype
    char* s_buf = s_rt_base + r16(16 + a.Lmax);
    const FAXTile lay = fax_tile_layout(TILE, a.max_atoms);
    char* s_go_base = s_buf + (kDB ? 2 : 1) * lay.total;

    const int b = blockIdx.x;
    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        mbar_init(bar + 2, 1);
        mbar_init(bar + 3, 1);
        fence_barrier_init();
        if (kTabSmem) {
            const unsigned tb = unsigned(a.n_types * sizeof(FAType));
            mbar_arrive_expect_tx(bar + 2, tb);
            bulk_g2s(smem + S::kTable, a.types, tb, bar + 2);
        }
    }
    if (tid == 0 && prefetch_regime(a.B)) {  // dL/dr is cold: into L2 under the previous kernel's tail
        const Span pg = make_span(a.grad_coords + (size_t)b * a.atom_stride * 3, a.atom_stride * 12);
        if (pg.mid > 0) prefetch_l2(pg.g + pg.head, unsigned(pg.mid));
    }
    pdl_wait();
    pdl_trigger();
    const int L = a.lengths[b];
    __syncthreads();
    if (kTabSmem) mbar_wait(bar + 2, 0);
    if (L < 1 || L > a.Lmax) {
        if (tid == 0) atomicOr(a.err, ERR_LENGTH);
        return;
    }
    const unsigned char* rtb = a.restype + (size_t)b * a.Lmax;
    const int n_tiles = (L + TILE - 1) / TILE;
    const int rl0 = tid * RPT;
    // the chain's residue types, once (bar 3)
    const unsigned char* s_rtc;
    {
        const Span sr = make_span(rtb, L);
        if (tid == 0) {
            mbar_arrive_expect_tx(bar + 3, unsigned(sr.mid));
            span_load_bulk(sr, s_rt_base, bar + 3);
        }
        span_load_edges_u8(sr, s_rt_base);
        mbar_wait(bar + 3, 0);
        __syncthreads();
        s_rtc = reinterpret_cast<const unsigned char*>(s_rt_base + sr.mis());
    }

    // pre-pass: atom offset of every tile start and of every thread's first atom within
    // its tile (s_roff: the tile loop needs no scan of its own), validity of the types
    {
        int carry = 0;
        bool bad = false;
        for (int t = 0; t < n_tiles; ++t) {
            int cnt = 0;
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const int j = t * TILE + rl0 + q;
                if (j < L) {
                    const int ty = s_rtc[j];
                    if (ty >= a.n_types) bad = true;
                    else cnt += s_types[ty].n_atoms;
                }
            }
            int end;
            s_roff[t * NT + tid] = (unsigned short)(block_exclusive_sum_int<NT>(cnt, carry, s_int, &end) - carry);
            if (tid == 0) s_off[t] = carry;
            carry = end;
        }
        if (tid == 0) s_off[n_tiles] = carry;
        if (__syncthreads_or(bad)) {
            if (tid == 0) atomicOr(a.err, ERR_RESTYPE);
            return;
        }
        if (carry > a.atom_stride) {  // uniform: carry is the block total
            if (tid == 0) atomicOr(a.err, ERR_STRIDE);
            return;
        }
    }

    const float* xb = a.coords + (size_t)b * a.atom_stride * 3;
    const float* gb = a.grad_coords + (size_t)b * a.atom_stride * 3;
    auto spans = [&](int t, Span& sx, Span& sg) {
        const int a0 = s_off[t], a1 = s_off[t + 1];
        sx = make_span(xb + (size_t)a0 * 3, (a1 - a0) * 12);
        sg = make_span(gb + (size_t)a0 * 3, (a1 - a0) * 12);
    };
    auto issue = [&](int t, int buf) {
        Span sx, sg;
        spans(t, sx, sg);
        char* base = s_buf + buf * lay.total;
        mbar_arrive_expect_tx(bar + buf, unsigned(sx.mid + sg.mid));
        span_load_bulk(sx, base + lay.x, bar + buf);
        span_load_bulk(sg, base + lay.g, bar + buf);
    };
    if (tid == 0) issue(n_tiles - 1, 0);

    float carry6[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float cpx = 0.f, cpy = 0.f, cpz = 0.f;
    unsigned phases = 0;
    for (int k = 0; k < n_tiles; ++k) {
        const int t = n_tiles - 1 - k, buf = kDB ? (k & 1) : 0;
        const int r0 = t * TILE, n = min(TILE, L - r0);
        if (kDB && tid == 0 && t > 0) issue(t - 1, buf ^ 1);
        Span sx, sg;
        spans(t, sx, sg);
        char* base = s_buf + buf * lay.total;
        span_load_edges_f32(sx, base + lay.x);
        span_load_edges_f32(sg, base + lay.g);
        mbar_wait(bar + buf, (phases >> buf) & 1u);
        phases ^= 1u << buf;
        __syncthreads();
        const unsigned char* s_rt = s_rtc + r0;
        const float* X = reinterpret_cast<const float*>(base + lay.x + sx.mis());
        const float* G = reinterpret_cast<const float*>(base + lay.g + sg.mis());

        if (tid == 0) bulk_wait_read_all();  // grad staging free (read by the previous store)
        int typ[RPT];
#pragma unroll
        for (int q = 0; q < RPT; ++q) typ[q] = rl0 + q < n ? s_rt[rl0 + q] : 0;
        const int off0 = s_roff[t * NT + tid];
        const float rx = X[0], ry = X[1], rz = X[2];  // tile reference point
        if (k > 0) {  // later tiles' moment about this tile's reference
            const float dx = cpx - rx, dy = cpy - ry, dz = cpz - rz;
            carry6[3] += fmaf(dy, carry6[2], -dz * carry6[1]);
            carry6[4] += fmaf(dz, carry6[0], -dx * carry6[2]);
            carry6[5] += fmaf(dx, carry6[1], -dy * carry6[0]);
        }
        cpx = rx; cpy = ry; cpz = rz;
        float* s_go = reinterpret_cast<float*>(s_go_base);  // [n][8], 16-B aligned rows when dst is

        // residue pass: chi gradients, residue sums about CA, and the backbone
        // positions the gradient pass needs (the staging is released after it)
        float RA[RPT][6], RN[RPT][6], RC[RPT][6];
        float PN[RPT][3], PCA[RPT][3], PC[RPT][3], PNX[RPT][3];  // N, CA, C, next residue's N
        float thr[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        int off = off0;
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
#pragma unroll
            for (int c = 0; c < 6; ++c) RA[q][c] = RN[q][c] = RC[q][c] = 0.f;
#pragma unroll
            for (int c = 0; c < 3; ++c) PN[q][c] = PCA[q][c] = PC[q][c] = PNX[q][c] = 0.f;
            const int rl = rl0 + q;
            if (rl < n) {
                const FAType& T = s_types[typ[q]];
                const FAHead h = load_head(T);
                const float* x = X + 3 * off;
                const float* g = G + 3 * off;
                float* go = s_go + 8 * rl;
#pragma unroll
                for (int c = 3; c < 8; ++c) go[c] = 0.f;
                const float cx = x[3 * h.iCA], cy = x[3 * h.iCA + 1], cz = x[3 * h.iCA + 2];
                PCA[q][0] = cx; PCA[q][1] = cy; PCA[q][2] = cz;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    PN[q][c] = x[3 * h.iN + c];
                    PC[q][c] = x[3 * h.iC + c];
                }
                const int j = r0 + rl;
                if (j + 1 < L) {  // N of the next residue: in this tile, or the first of the later tile
                    const int iN = s_types[s_rtc[j + 1]].iN;
                    const float* xn = rl + 1 < n ? x + 3 * h.n_atoms : xb + (size_t)s_off[t + 1] * 3;
#pragma unroll
                    for (int c = 0; c < 3; ++c) PNX[q][c] = xn[3 * iN + c];
                }
                auto acc = [&](float* s6, int i) {
                    cross_acc(s6, x[3 * i] - cx, x[3 * i + 1] - cy, x[3 * i + 2] - cz, g[3 * i], g[3 * i + 1],
                              g[3 * i + 2]);
                };
                for (int i = 0; i < h.n_N; ++i) acc(RN[q], i);
                for (int i = h.n_N; i < h.n_N + h.n_CA; ++i) acc(RA[q], i);
                for (int i = h.first_C; i < h.n_atoms; ++i) acc(RC[q], i);
                float br[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                for (int gi = h.n_groups - 1; gi >= 0; --gi) {
                    const FAGroup gr = load_group(T.g[gi]);
#pragma unroll 2
                    for (int i = gr.first_atom; i < gr.end_atom; ++i) acc(br, i);
                    if (gr.slot >= 0) {
                        const int o = gr.origin, p = gr.porigin;
                        const float ox = x[3 * o] - cx, oy = x[3 * o + 1] - cy, oz = x[3 * o + 2] - cz;
                        const float ux = x[3 * o] - x[3 * p], uy = x[3 * o + 1] - x[3 * p + 1],
                                    uz = x[3 * o + 2] - x[3 * p + 2];
                        const float inv = rsqrtf(fmaf(ux, ux, fmaf(uy, uy, uz * uz)));
                        go[gr.slot] = inv * axis_moment(ux, uy, uz, ox, oy, oz, br);
                    }
                    if (gr.parent < 0) {
#pragma unroll
                        for (int c = 0; c < 6; ++c) { RA[q][c] += br[c]; br[c] = 0.f; }
                    }
                }
#pragma unroll
                for (int c = 0; c < 6; ++c) RA[q][c] += RN[q][c] + RC[q][c];
                // residue moment about the tile reference: T_r = T_CA + (CA - r) x S
                const float dx = cx - rx, dy = cy - ry, dz = cz - rz;
                const float* s6 = RA[q];
                thr[0] += s6[0]; thr[1] += s6[1]; thr[2] += s6[2];
                thr[3] += s6[3] + fmaf(dy, s6[2], -dz * s6[1]);
                thr[4] += s6[4] + fmaf(dz, s6[0], -dx * s6[2]);
                thr[5] += s6[5] + fmaf(dx, s6[1], -dy * s6[0]);
                off += h.n_atoms;
            }
        }
        float suf[6], tot6[6];
        block_exclusive_suffix6<NT>(thr, carry6, s_suf, suf, tot6);
        // every thread is past the residue pass: the single buffer may refill
        if (!kDB && tid == 0 && t > 0) issue(t - 1, 0);

        // backbone gradients, residues last to first (registers only)
#pragma unroll
        for (int q = RPT - 1; q >= 0; --q) {
            const int rl = rl0 + q;
            const int j = r0 + rl;
            if (rl < n) {
                float* go = s_go + 8 * rl;
                const float cx = PCA[q][0], cy = PCA[q][1], cz = PCA[q][2];
                const float dx = cx - rx, dy = cy - ry, dz = cz - rz;
                float aft[6];  // later residues, moment about CA_j
                aft[0] = suf[0]; aft[1] = suf[1]; aft[2] = suf[2];
                aft[3] = suf[3] - fmaf(dy, suf[2], -dz * suf[1]);
                aft[4] = suf[4] - fmaf(dz, suf[0], -dx * suf[2]);
                aft[5] = suf[5] - fmaf(dx, suf[1], -dy * suf[0]);
                const float nx = PN[q][0], ny = PN[q][1], nz = PN[q][2];
                const float kx = PC[q][0], ky = PC[q][1], kz = PC[q][2];
                float s6[6];
                // psi_j
#pragma unroll
                for (int c = 0; c < 6; ++c) s6[c] = RC[q][c] + aft[c];
                {
                    const float ux = kx - cx, uy = ky - cy, uz = kz - cz;
                    go[1] = bb_invd(2) * axis_moment(ux, uy, uz, ux, uy, uz, s6);
                }
                // phi_j
#pragma unroll
                for (int c = 0; c < 6; ++c) s6[c] = RA[q][c] - RN[q][c] + aft[c];
                {
                    const float ux = cx - nx, uy = cy - ny, uz = cz - nz;
                    go[0] = bb_invd(1) * axis_moment(ux, uy, uz, 0.f, 0.f, 0.f, s6);
                }
                // omega_j: C_j -> N_{j+1}, later residues
                float gw = 0.f;
                if (j + 1 < L) {
                    const float px = PNX[q][0], py = PNX[q][1], pz = PNX[q][2];
                    const float ux = px - kx, uy = py - ky, uz = pz - kz;
                    gw = bb_invd(0) *
                         axis_moment(ux, uy, uz, px - cx, py - cy, pz - cz, aft);
                }
                go[2] = gw;
                // fold this residue into the suffix (about the tile reference)
                const float* r6 = RA[q];
                suf[0] += r6[0]; suf[1] += r6[1]; suf[2] += r6[2];
                suf[3] += r6[3] + fmaf(dy, r6[2], -dz * r6[1]);
                suf[4] += r6[4] + fmaf(dz, r6[0], -dx * r6[2]);
                suf[5] += r6[5] + fmaf(dx, r6[1], -dy * r6[0]);
            }
        }
        __syncthreads();
        {
            float* dst = a.grad_angles + ((size_t)b * a.Lmax + r0) * kFASlots;
            if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
                fence_proxy_async_smem();
                __syncthreads();
                if (tid == 0) {
                    bulk_s2g(dst, s_go, unsigned(n * 32));
                    bulk_commit();
                }
            } else {
                for (int i = tid; i < n * 8; i += NT) dst[i] = s_go[i];
            }
        }
#pragma unroll
        for (int c = 0; c < 6; ++c) carry6[c] = tot6[c];
        __syncthreads();
    }
    if (tid == 0) bulk_wait_all();
}

// ---------------------------------------------------------------------------
// One residue per thread; 256-thread forward CTAs, 128-thread backward CTAs
// (the backward keeps more per-residue state: <= 170 registers, 3 CTAs/SM).
// Chains longer than a tile loop over tiles.  The atom staging buffer is sized
// by the table's largest residue type (FAArgs.max_atoms).
constexpr int kFAFwdThreads = 256, kFAFwdRPT = 1;
constexpr int kFABwdThreads = 128, kFABwdRPT = 1;
int fa_rpt_for(int) { return kFABwdRPT; }
int fa_tile_for(int) { return kFABwdThreads * kFABwdRPT; }  // backward tile: sizes the workspace prefixes

template <int NT, int RPT>
static size_t fa_fwd_smem(int n_types, int max_atoms, bool ts = true, int in_bufs = 1) {
    using S = FASmem<NT>;
    using Lay = FALayout<NT, RPT>;
    return S::kTable + (ts ? r16(n_types * int(sizeof(FAType))) : 0) + in_bufs * (Lay::ang_bytes + Lay::rt_bytes) +
           r16(16 + 12 * max_atoms * Lay::TILE);
}
template <int NT, int RPT>
static size_t fa_bwd_smem(int n_types, int max_atoms) {
    using Lay = FALayout<NT, RPT>;
    return fa_fwd_smem<NT, RPT>(n_types, max_atoms) + Lay::go_bytes;
}

template <int NT, int NS, bool TS, int MINB, int RPT = 1, bool DBI = true>
static cudaError_t fa_fwd_v(const FAArgs& a, cudaStream_t st) {
    auto k = fa_forward_kernel<NT, RPT, NS, TS, MINB, DBI>;
    const size_t sm = fa_fwd_smem<NT, RPT>(a.n_types, a.max_atoms, TS, DBI ? 2 : 1);
    static LaunchCfg cfg;  // one grid CTA per chain: only the shared-memory opt-in is used
    cudaError_t e = ensure_launch_cfg(cfg, k, NT, sm);
    if (e != cudaSuccess) return e;
    return launch_bbp(k, a.B, NT, BBPLaunch{sm, a.B <= 2 * device_sm_count()}, st, a, a.max_atoms);
}
// TPL_FAF=NTxTSxMINB (tuning) or the default.
struct FAFShape {
    int nt, ts, minb, rpt;
};
static FAFShape faf_shape(int B, int Lmax) {
    static FAFShape env{-1, 0, 0, 1};
    if (env.nt < 0) {
        env = {0, 0, 0, 1};
        if (const char* e = std::getenv("TPL_FAF")) {
            FAFShape s{0, 1, 2, 1};
            if (std::sscanf(e, "%dx%dx%dx%d", &s.nt, &s.ts, &s.minb, &s.rpt) >= 3) env = s;
        }
    }
    if (env.nt) return env;
    // measured (TPL_FAF sweeps, same box): few chains -> 256 threads, table in shared
    // memory; at most one chain per SM and chains longer than 256 residues: one
    // 512-thread tile per chain instead of two serial 256-residue tiles (config 3:
    // 13.7 -> 10.6 us); many chains -> table through L1 and either 128 threads x 1
    // residue at 6 CTAs/SM or 64 threads x 2 residues at 8 CTAs/SM (the block scan,
    // a third of the kernel's instructions at one residue per thread, amortised over
    // two).  64 x 2 wins for long chains in large batches (x 500: 1024 chains 66.0 ->
    // 52.6 us, 2048 104.9 -> 100.8, 8192 360.5 -> 331.7) and loses for shorter ones
    // (x 300: 512 chains 25.9 -> 30.2 us, 4096 134.4 -> 138.8).
    if (B <= 148 && Lmax > 256) return FAFShape{512, 1, 1, 1};
    if (B <= 2 * 148) return FAFShape{256, 1, 2, 1};
    return B >= 1024 && Lmax > 384 ? FAFShape{64, 0, 8, 2} : FAFShape{128, 0, 6, 1};
}
template <int NS>
static cudaError_t fa_fwd(const FAArgs& a, cudaStream_t st) {
    const FAFShape s = faf_shape(a.B, a.Lmax);
#define TPL_FAF(NT_, TS_, MB_) \
    if (s.nt == NT_ && s.ts == TS_ && s.minb == MB_ && s.rpt == 1) return fa_fwd_v<NT_, NS, TS_, MB_>(a, st);
    TPL_FAF(256, 1, 2) TPL_FAF(256, 0, 2) TPL_FAF(256, 0, 3) TPL_FAF(256, 1, 3) TPL_FAF(512, 1, 1)
    TPL_FAF(128, 1, 4) TPL_FAF(128, 0, 4) TPL_FAF(128, 0, 6) TPL_FAF(128, 1, 6)
#undef TPL_FAF
#define TPL_FAF2(NT_, TS_, MB_) \
    if (s.nt == NT_ && s.ts == TS_ && s.minb == MB_ && s.rpt == 2) return fa_fwd_v<NT_, NS, TS_, MB_, 2, false>(a, st);
    TPL_FAF2(64, 0, 8) TPL_FAF2(64, 0, 6) TPL_FAF2(128, 0, 4) TPL_FAF2(256, 1, 2)
#undef TPL_FAF2
    return cudaErrorInvalidConfiguration;
}
template <int NS>
static cudaError_t fa_bwd(const FAArgs& a, cudaStream_t st) {
    auto k = fa_backward_kernel<kFABwdThreads, kFABwdRPT, NS>;
    const size_t sm = fa_bwd_smem<kFABwdThreads, kFABwdRPT>(a.n_types, a.max_atoms);
    static LaunchCfg cfg;  // one grid CTA per chain: only the shared-memory opt-in is used
    cudaError_t e = ensure_launch_cfg(cfg, k, kFABwdThreads, sm);
    if (e != cudaSuccess) return e;
    return launch_pdl(k, a.B, kFABwdThreads, sm, st, a, a.max_atoms);
}

// TPL_FAX=NTxRPTxDBxTS (tuning) or the default.
struct FAXShape {
    int nt, rpt, db, ts;
};
static FAXShape fax_shape(int B, int Lmax) {
    static FAXShape env{-1, 0, 0, 0};
    if (env.nt < 0) {
        env = {0, 0, 0, 0};
        if (const char* e = std::getenv("TPL_FAX")) {
            FAXShape s{0, 1, 0, 0};
            if (std::sscanf(e, "%dx%dx%dx%d", &s.nt, &s.rpt, &s.db, &s.ts) >= 2) env = s;
        }
    }
    if (env.nt) return env;
    // measured (tools/gpu_fax.sh): single buffer + table through L1 (more resident
    // CTAs) wins; few chains -> long tiles (latency), many chains -> 64 threads
    if (B <= 148 && Lmax > 256) return FAXShape{512, 1, 0, 0};  // config 3: 15.3 -> 11.2 us
    return B <= 2 * 148 ? FAXShape{256, 1, 0, 0} : FAXShape{64, 1, 0, 0};
}

template <int NT, int RPT, bool DB, bool TS>
static cudaError_t fa_bwd_xyz(const FAArgs& a, cudaStream_t st) {
    auto k = fa_backward_xyz_kernel<NT, RPT, DB, TS>;
    constexpr int TILE = NT * RPT;
    const int max_tiles = (a.Lmax + TILE - 1) / TILE;
    const size_t sm = FAXSmem<NT>::kTable + fax_table_bytes(TS, a.n_types) + r16(4 * (max_tiles + 1)) +
                      r16(2 * max_tiles * NT) + r16(16 + a.Lmax) + (DB ? 2 : 1) * fax_tile_layout(TILE, a.max_atoms).total + r16(32 * TILE);
    static LaunchCfg cfg;  // one grid CTA per chain: only the shared-memory opt-in is used
    cudaError_t e = ensure_launch_cfg(cfg, k, NT, sm);
    if (e != cudaSuccess) return e;
    return launch_bbp(k, a.B, NT, BBPLaunch{sm, a.B <= 2 * device_sm_count()}, st, a, max_tiles);
}

cudaError_t fa_backward_xyz_launch(const FAArgs& a, cudaStream_t st) {
    const FAXShape s = fax_shape(a.B, a.Lmax);
#define TPL_FAX(NT_, R_, DB_, TS_) \
    if (s.nt == NT_ && s.rpt == R_ && s.db == DB_ && s.ts == TS_) return fa_bwd_xyz<NT_, R_, DB_, TS_>(a, st);
    TPL_FAX(64, 1, 0, 0) TPL_FAX(128, 1, 0, 0) TPL_FAX(256, 1, 0, 0) TPL_FAX(512, 1, 0, 0)
    TPL_FAX(64, 1, 1, 1) TPL_FAX(128, 1, 1, 1) TPL_FAX(256, 1, 1, 1)
#undef TPL_FAX
    return cudaErrorInvalidConfiguration;
}

cudaError_t fa_forward_launch(const FAArgs& a, cudaStream_t st) {
    // FA scans combine one residue per thread over up to 16 warps: re-orthonormalise
    // each cross-warp combine too (policy 3; FA at L = 700: 1.03e-3 -> see DESIGN)
    return a.ns == 0 ? fa_fwd<0>(a, st) : a.ns == 1 && std::getenv("TPL_FA_NS1") ? fa_fwd<1>(a, st) : fa_fwd<3>(a, st);
}
cudaError_t fa_backward_launch(const FAArgs& a, cudaStream_t st) {
    return a.ns == 0 ? fa_bwd<0>(a, st) : a.ns == 1 && std::getenv("TPL_FA_NS1") ? fa_bwd<1>(a, st) : fa_bwd<3>(a, st);
}

}  // namespace tpl
