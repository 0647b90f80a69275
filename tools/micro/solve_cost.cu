// Latency of the per-chain LRMSD solve (lrmsd_math.cuh: T, eigenpair, U) on one
// thread: clock64 around lrmsd_solve for random-pair and near-superposed moments.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1812_01108_b200/csrc \
//        -I include tools/micro/solve_cost.cu -o tools/micro/solve_cost && tools/micro/solve_cost
#include <cstdio>

#define TPL_SOLVE_CLOCKS
#include "lrmsd_math.cuh"

__global__ void k(const double* mom, int n, long long* cyc, float* out) {
    float st[16], v;
    for (int i = 0; i < n; ++i) {
        const long long t0 = clock64();
        tpl::lrmsd_solve(mom + 17 * i, 2100.0, &v, st);
        const long long t1 = clock64();
        cyc[i * 8] = t1 - t0;
        for (int p = 1; p < 6; ++p) cyc[i * 8 + p] = tpl::g_solve_clk[p] - tpl::g_solve_clk[p - 1];
        cyc[i * 8 + 6] = tpl::g_solve_clk[0] - t0;
        cyc[i * 8 + 7] = t1 - tpl::g_solve_clk[5];
        out[i] = v + st[0];
    }
}

int main() {
    const int n = 4;
    double h[17 * n] = {};
    // random pair (centred moments): R ~ small relative to sxx, syy
    double* m = h;
    m[6] = 1.2e4; m[7] = -3.1e4; m[8] = 2.2e4; m[9] = 5.0e3; m[10] = 9.1e3; m[11] = -1.4e4; m[12] = 7.7e3;
    m[13] = 2.5e3; m[14] = -6.0e3; m[15] = 2.0e6; m[16] = 1.9e6;
    // near-superposed: R ~ diag(sxx) rotated a little
    m = h + 17;
    m[6] = 7.0e5; m[7] = 1.0e3; m[8] = -2.0e3; m[9] = -1.0e3; m[10] = 6.5e5; m[11] = 5.0e2; m[12] = 2.0e3;
    m[13] = -5.0e2; m[14] = 6.4e5; m[15] = 1.99e6; m[16] = 1.99e6;
    for (int i = 2; i < n; ++i)
        for (int k = 0; k < 17; ++k) h[17 * i + k] = h[17 * (i - 2) + k] * (1.0 + 0.01 * i);
    double* dm;
    long long* dc;
    float* dout;
    cudaMalloc(&dm, sizeof(h));
    cudaMalloc(&dc, 8 * n * sizeof(long long));
    cudaMalloc(&dout, n * sizeof(float));
    cudaMemcpy(dm, h, sizeof(h), cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 3; ++rep) k<<<1, 1>>>(dm, n, dc, dout);
    long long c[8 * n];
    cudaMemcpy(c, dc, sizeof(c), cudaMemcpyDeviceToHost);
    for (int i = 0; i < n; ++i)
        printf("solve %d: %lld cycles (%.2f us): pre %lld coeffs %lld approach %lld polish %lld adjugate %lld post %lld\n", i,
               c[8 * i], c[8 * i] / 1965.0, c[8 * i + 6], c[8 * i + 1], c[8 * i + 2], c[8 * i + 3], c[8 * i + 4] + c[8 * i + 5],
               c[8 * i + 7]);
    return 0;
}
