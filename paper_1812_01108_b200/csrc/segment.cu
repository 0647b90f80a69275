// segment.cu -- SURVEY §8(f) row f4, across GPUs: one chain split into
// contiguous segments, one per rank, with one exchange step per pass (§8(e)).
//
// Forward: every rank runs the forward kernel on its segment in the segment's
// own frame (identity at the previous segment's last C; residue 0 carries the
// omega bond, bb_forward_kernel segment mode) and exports the segment's
// aggregate transform A_s (12 floats per chain).  After an all-gather,
// segment_place_kernel moves the local coordinates to the chain frame with
// C_s = N(..N(A_0 A_1)..A_{s-1}) (r_i = M_i 0 with M_i = C_s M_i^local).
//
// Backward (from the coordinates, Eq. 2 via the rotation-axis identity):
// segment_totals_kernel reduces the segment's (S, T) = (sum g, sum (r - c) x g)
// about its first atom c; after an all-gather the backward kernel adds the
// later segments' totals (fixed order) to its suffix sums and closes omega of
// the segment's last residue with the next segment's first atom.
#include "common.cuh"
#include "kernels.h"

namespace tpl {

constexpr int kSegThreads = 256;

// (S, T about the first atom, first atom) per chain segment; one CTA per chain,
// fixed-order reduction (deterministic).
__global__ void __launch_bounds__(kSegThreads) segment_totals_kernel(const float* __restrict__ coords,
                                                                     const int* __restrict__ lengths, int B,
                                                                     int Lmax, const float* __restrict__ grad_coords,
                                                                     float* __restrict__ totals,
                                                                     unsigned* __restrict__ err) {
    __shared__ float red[kSegThreads / 32][6];
    const int b = blockIdx.x, tid = threadIdx.x;
    const int L = lengths[b];
    if (L < 1 || L > Lmax) {
        if (tid == 0) atomicOr(err, ERR_LENGTH);
        return;
    }
    const float* x = coords + (size_t)b * Lmax * 9;
    const float* g = grad_coords + (size_t)b * Lmax * 9;
    const float cx = x[0], cy = x[1], cz = x[2];
    float s6[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int i = tid; i < 3 * L; i += kSegThreads) {
        const float px = x[3 * i] - cx, py = x[3 * i + 1] - cy, pz = x[3 * i + 2] - cz;
        const float gx = g[3 * i], gy = g[3 * i + 1], gz = g[3 * i + 2];
        s6[0] += gx; s6[1] += gy; s6[2] += gz;
        s6[3] += fmaf(py, gz, -pz * gy);
        s6[4] += fmaf(pz, gx, -px * gz);
        s6[5] += fmaf(px, gy, -py * gx);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1)
#pragma unroll
        for (int q = 0; q < 6; ++q) s6[q] += __shfl_down_sync(0xffffffffu, s6[q], d);
    if ((tid & 31) == 0)
#pragma unroll
        for (int q = 0; q < 6; ++q) red[tid >> 5][q] = s6[q];
    __syncthreads();
    if (tid == 0) {
        float* o = totals + (size_t)b * 12;
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            float v = 0.f;
            for (int w = 0; w < kSegThreads / 32; ++w) v += red[w][q];
            o[q] = v;
        }
        o[6] = cx; o[7] = cy; o[8] = cz;
        o[9] = o[10] = o[11] = 0.f;
    }
}

// coords of segment `seg` (its own frame) -> the chain frame.  grid (tiles, B).
__global__ void __launch_bounds__(kSegThreads) segment_place_kernel(float* __restrict__ coords,
                                                                    const int* __restrict__ lengths, int B, int Lmax,
                                                                    const float* __restrict__ aggs, int seg, int ns,
                                                                    unsigned* __restrict__ err) {
    __shared__ float sC[12];
    const int b = blockIdx.y, tid = threadIdx.x;
    const int L = lengths[b];
    if (L < 1 || L > Lmax) {
        if (tid == 0 && blockIdx.x == 0) atomicOr(err, ERR_LENGTH);
        return;
    }
    const int i = blockIdx.x * kSegThreads + tid;
    if (blockIdx.x * kSegThreads >= 3 * L) return;
    if (tid == 0) {
        Aff C = aff_identity();
        for (int r = 0; r < seg; ++r) {  // fixed order (deterministic)
            C = aff_compose(C, load_aff(aggs + ((size_t)r * B + b) * 12));
            if (ns >= 1) aff_orthonormalize(C);
        }
        store_aff(sC, C);
    }
    __syncthreads();
    if (i >= 3 * L) return;
    const Aff C = load_aff(sC);
    float* p = coords + ((size_t)b * Lmax * 3 + i) * 3;
    float ox, oy, oz;
    apply(C, p[0], p[1], p[2], ox, oy, oz);
    p[0] = ox;
    p[1] = oy;
    p[2] = oz;
}

cudaError_t segment_totals_launch(const BBArgs& a, float* totals, cudaStream_t st) {
    segment_totals_kernel<<<a.B, kSegThreads, 0, st>>>(static_cast<const float*>(a.coords), a.lengths, a.B, a.Lmax,
                                                       a.grad_coords, totals, a.err);
    return cudaGetLastError();
}

cudaError_t segment_place_launch(const BBArgs& a, const float* aggs, int seg, cudaStream_t st) {
    dim3 grid((3 * a.Lmax + kSegThreads - 1) / kSegThreads, a.B);
    segment_place_kernel<<<grid, kSegThreads, 0, st>>>(a.coords, a.lengths, a.B, a.Lmax, aggs, seg, a.ns, a.err);
    return cudaGetLastError();
}

}  // namespace tpl
