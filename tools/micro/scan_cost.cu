// Micro-benchmark: latency of the block-wide affine scan (block_exclusive_scan) and of
// the pass-1 residue chain alone, 256 CTAs x 128 threads, one round per CTA.
#include <cstdio>
#include "../../paper_1812_01108_b200/csrc/common.cuh"

using namespace tpl;

template <int MODE>
__global__ void k(float* out, const float* ang, int reps) {
    __shared__ float scratch[4 * 12];
    __shared__ float total[12];
    const int tid = threadIdx.x;
    Aff M = aff_identity();
    long long t0 = clock64();
    if (MODE == 0) {  // 7 residues x 3 bonds, as pass 1
        for (int r = 0; r < reps; ++r)
#pragma unroll
            for (int q = 0; q < 7; ++q) {
                const float x[3] = {ang[(tid * 7 + q) * 3], ang[(tid * 7 + q) * 3 + 1], ang[(tid * 7 + q) * 3 + 2]};
                float s[3], c[3], mx = 0.f;
                tpl_sincos_hot<3>(x, s, c, &mx);
                aff_bond_bb<0>(M, c[0], s[0]);
                aff_bond_bb<1>(M, c[1], s[1]);
                aff_bond_bb<2>(M, c[2], s[2]);
            }
    } else {  // the block scan
        M.t0 = ang[tid];
        for (int r = 0; r < reps; ++r) {
            M = block_exclusive_scan<128, 1>(M, aff_identity(), scratch, total);
        }
    }
    long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = float(t1 - t0);
    out[gridDim.x + blockIdx.x * 128 + tid] = M.t0 + M.r00;
}

int main() {
    float *out, *ang;
    cudaMalloc(&out, (256 + 256 * 128) * sizeof(float));
    cudaMalloc(&ang, 128 * 7 * 3 * sizeof(float) + 4096);
    cudaMemset(ang, 0, 128 * 7 * 3 * sizeof(float) + 4096);
    float h[256];
    for (int mode = 0; mode < 2; ++mode) {
        for (int g : {1, 256}) {
            if (mode == 0) k<0><<<g, 128>>>(out, ang, 1); else k<1><<<g, 128>>>(out, ang, 1);
            cudaDeviceSynchronize();
            if (mode == 0) k<0><<<g, 128>>>(out, ang, 1); else k<1><<<g, 128>>>(out, ang, 1);
            cudaMemcpy(h, out, g * sizeof(float), cudaMemcpyDeviceToHost);
            double m = 0;
            for (int i = 0; i < g; ++i) m = h[i] > m ? h[i] : m;
            printf("%s grid %3d: max %.0f cycles (%.2f us at 1.965 GHz)\n", mode ? "block scan      " : "pass1 7 residues", g, m,
                   m / 1965.0);
        }
    }
    return 0;
}
