// Largest root of the LRMSD quartic (lrmsd_math.cuh, sym4_max_eigen_newton): cycles
// and iterations of three ways to reach it on one warp, over random, near-rotation,
// reflected and degenerate correlation matrices R.
//   V0: the library's loop (fp64 Laguerre with two reciprocals + rsqrt per step)
//   V1: the same start, lambda scaled by |R|_F and one reciprocal + one sqrt per step
//   V2: V1 started from a 32-lane bracket (two rounds of 32-section on [0, bound],
//       Fourier-Budan: the smallest sample where p, p', p'' > 0 (and lambda > 0) lies
//       above every root)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1812_01108_b200/csrc \
//        -I include tools/micro/polish.cu -o tools/micro/polish && tools/micro/polish
#include <cstdio>
#include <cstdlib>
#include <cmath>

#include "lrmsd_math.cuh"

using namespace tpl;

constexpr int NV = 9;
struct Coef { double c2, c1, c0, start; };

__device__ Coef coefs(const double R[3][3], double e0) {
    double T[4][4] = {
        {R[0][0] + R[1][1] + R[2][2], R[1][2] - R[2][1], R[2][0] - R[0][2], R[0][1] - R[1][0]},
        {R[1][2] - R[2][1], R[0][0] - R[1][1] - R[2][2], R[0][1] + R[1][0], R[0][2] + R[2][0]},
        {R[2][0] - R[0][2], R[0][1] + R[1][0], -R[0][0] + R[1][1] - R[2][2], R[1][2] + R[2][1]},
        {R[0][1] - R[1][0], R[0][2] + R[2][0], R[1][2] + R[2][1], -R[0][0] - R[1][1] + R[2][2]},
    };
    double c2 = 0.0;
    for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 3; ++c) c2 += R[a][c] * R[a][c];
    c2 *= -2.0;
    Coef k;
    k.c2 = c2;
    k.c1 = -8.0 * det3(R[0][0], R[0][1], R[0][2], R[1][0], R[1][1], R[1][2], R[2][0], R[2][1], R[2][2]);
    k.c0 = det4(T);
    k.start = fmin(e0 * (1.0 + 1e-5), sqrt(-1.5 * c2) * (1.0 + 1e-12));
    return k;
}

__device__ double v0(const Coef& k, int* its) {
    const double c2 = k.c2, c1 = k.c1, c0 = k.c0;
    double l = k.start;
    int it = 0;
    for (; it < 12; ++it) {
        const double l2 = l * l;
        const double p = (l2 + c2) * l2 + c1 * l + c0;
        if (!(p > 0.0)) break;
        const double dp = (4.0 * l2 + 2.0 * c2) * l + c1;
        const double ddp = 12.0 * l2 + 2.0 * c2;
        const double ip = rcp_full(p);
        const double G = dp * ip;
        const double H = fma(-ddp, ip, G * G);
        const double disc = 3.0 * fmax(4.0 * H - G * G, 0.0);
        const double den = G + (disc > 0.0 ? disc * rsqrt_full(disc) : 0.0);
        if (!(den > 0.0)) break;
        const double step = 4.0 * rcp_full(den);
        l -= step;
        if (step <= 1e-14 * fabs(l)) break;
    }
    *its = it;
    return l;
}

// scaled: mu = lambda / s, s = |R|_F = sqrt(-c2 / 2): q(mu) = mu^4 - 2 mu^2 + b1 mu + b0
__device__ double v1_from(const Coef& k, double s, double is, double mu, int* its) {
    const double b1 = k.c1 * is * is * is, b0 = k.c0 * (is * is) * (is * is);
    int it = 0;
    for (; it < 12; ++it) {
        const double m2 = mu * mu;
        const double p = fma(m2 - 2.0, m2, fma(b1, mu, b0));
        if (!(p > 0.0)) break;
        const double dp = fma(4.0 * m2 - 4.0, mu, b1);
        const double ddp = fma(12.0, m2, -4.0);
        // Laguerre (n = 4): step = 4 p / (p' + sqrt(3 (3 p'^2 - 4 p p'')))
        const double disc = fmax(fma(9.0 * dp, dp, -12.0 * p * ddp), 0.0);
        const double den = dp + (disc > 0.0 ? disc * rsqrt_full(disc) : 0.0);
        if (!(den > 0.0)) break;
        const double step = 4.0 * p * rcp_full(den);
        mu -= step;
        if (step <= 1e-14 * fabs(mu)) break;
    }
    *its = it;
    return mu * s;
}

__device__ double v1(const Coef& k, int* its) {
    const double s = sqrt(-0.5 * k.c2), is = 1.0 / s;
    return v1_from(k, s, is, k.start * is, its);
}

// V2: lanes sample mu in [0, hi]; the smallest sample with p, p', p'' > 0 bounds every root
__device__ double v2(const Coef& k, int* its) {
    const int lane = threadIdx.x & 31;
    const double s = sqrt(-0.5 * k.c2), is = 1.0 / s;
    const double b1 = k.c1 * is * is * is, b0 = k.c0 * (is * is) * (is * is);
    double lo = 0.0, hi = k.start * is;
    for (int round = 0; round < 2; ++round) {
        const double w = (hi - lo) * (1.0 / 32.0);
        const double mu = lo + w * double(lane + 1);  // lane 31 = hi (above every root)
        const double m2 = mu * mu;
        const double p = fma(m2 - 2.0, m2, fma(b1, mu, b0));
        const double dp = fma(4.0 * m2 - 4.0, mu, b1);
        const double ddp = fma(12.0, m2, -4.0);
        const unsigned above = __ballot_sync(0xffffffffu, p > 0.0 && dp > 0.0 && ddp > 0.0);
        // above-all-roots is an upper set of samples: its lowest member
        const int first = above ? __ffs(above) - 1 : 31;  // lane 31 (the bound) qualifies
        hi = lo + w * double(first + 1);
        lo = hi - w;
    }
    return v1_from(k, s, is, hi, its);
}

// V3: V2's bracket (rounds in fp64 across the lanes), then Laguerre with p in fp64 and
// the step in fp32 (a correction: its relative error only scales the remaining distance)
__device__ double v3_from(double b1, double b0, double mu, double tol, int* its) {
    const float b1f = float(b1);
    int it = 0;
    for (; it < 12; ++it) {
        const double m2 = mu * mu;
        const double p = fma(m2 - 2.0, m2, fma(b1, mu, b0));
        if (!(p > 0.0)) break;
        const float mf = float(mu), pf = float(p), m2f = mf * mf;
        const float dp = fmaf(4.f * m2f - 4.f, mf, b1f);
        const float ddp = fmaf(12.f, m2f, -4.f);
        const float disc = fmaxf(fmaf(9.f * dp, dp, -12.f * pf * ddp), 0.f);
        const float den = dp + disc * rsqrtf(fmaxf(disc, 1e-37f));
        if (!(den > 0.f)) break;
        const float step = 4.f * pf * __frcp_rn(den);
        mu -= double(step);
        if (double(step) <= tol * fabs(mu)) break;
    }
    *its = it;
    return mu;
}
template <int kRounds>
__device__ double v3(const Coef& k, double tol, int* its) {
    const int lane = threadIdx.x & 31;
    const double s = sqrt(-0.5 * k.c2), is = 1.0 / s;
    const double b1 = k.c1 * is * is * is, b0 = k.c0 * (is * is) * (is * is);
    double lo = 0.0, hi = k.start * is;
    for (int round = 0; round < kRounds; ++round) {
        const double w = (hi - lo) * (1.0 / 32.0);
        const double mu = lo + w * double(lane + 1);
        const double m2 = mu * mu;
        const double p = fma(m2 - 2.0, m2, fma(b1, mu, b0));
        const double dp = fma(4.0 * m2 - 4.0, mu, b1);
        const double ddp = fma(12.0, m2, -4.0);
        const unsigned above = __ballot_sync(0xffffffffu, p > 0.0 && dp > 0.0 && ddp > 0.0);
        const int first = above ? __ffs(above) - 1 : 31;
        hi = lo + w * double(first + 1);
        lo = hi - w;
    }
    return v3_from(b1, b0, hi, tol, its) * s;
}

__global__ void kern(const double* Rs, int n, long long* cyc, double* lam, int* its) {
    for (int i = 0; i < n; ++i) {
        double R[3][3];
        double e0 = 0.0;
        for (int a = 0; a < 9; ++a) R[a / 3][a % 3] = Rs[10 * i + a];
        e0 = Rs[10 * i + 9];
        const Coef k = coefs(R, e0);
        __syncwarp();
        for (int v = 0; v < NV; ++v) {
            int it = 0;
            __syncwarp();
            const long long t0 = clock64();
            double l;
            if (v == 0) l = v0(k, &it);
            else if (v == 1) l = v1(k, &it);
            else if (v == 2) l = v2(k, &it);
            else if (v == 3) l = v3<2>(k, 1e-14, &it);
            else if (v == 4) l = v3<2>(k, 1e-9, &it);
            else if (v == 5) l = v3<3>(k, 1e-9, &it);
            else if (v == 6) l = v3<1>(k, 1e-9, &it);
            else if (v == 7) {  // the whole single-thread rotation (library, before)
                __shared__ float U[9];
                if (threadIdx.x == 0) lrmsd_rotation(R, e0, U);
                __syncwarp();
                l = U[0];
            } else {            // the whole warp rotation (library, now)
                __shared__ float U[9];
                lrmsd_rotation_warp(R, U);
                __syncwarp();
                l = U[0];
            }
            // consume l before the clock (the loop's result)
            const long long t1 = clock64() + (l == 12345.0 ? 1 : 0);
            if (threadIdx.x == 0) {
                cyc[NV * i + v] = t1 - t0;
                lam[NV * i + v] = l;
                its[NV * i + v] = it;
            }
        }
    }
}

int main() {
    const int n = 64;
    static double h[10 * n];
    srand(7);
    auto rnd = [] { return (rand() + 0.5) / (RAND_MAX + 1.0); };
    auto gauss = [&] { return sqrt(-2 * log(rnd())) * cos(6.283185307179586 * rnd()); };
    for (int i = 0; i < n; ++i) {
        double* m = h + 10 * i;
        const int kind = i % 4;
        // random rotation Q from a random unit quaternion
        double q[4], qn = 0;
        for (int a = 0; a < 4; ++a) { q[a] = gauss(); qn += q[a] * q[a]; }
        for (int a = 0; a < 4; ++a) q[a] /= sqrt(qn);
        const double Q[9] = {q[0]*q[0]+q[1]*q[1]-q[2]*q[2]-q[3]*q[3], 2*(q[1]*q[2]-q[0]*q[3]), 2*(q[1]*q[3]+q[0]*q[2]),
                             2*(q[1]*q[2]+q[0]*q[3]), q[0]*q[0]-q[1]*q[1]+q[2]*q[2]-q[3]*q[3], 2*(q[2]*q[3]-q[0]*q[1]),
                             2*(q[1]*q[3]-q[0]*q[2]), 2*(q[2]*q[3]+q[0]*q[1]), q[0]*q[0]-q[1]*q[1]-q[2]*q[2]+q[3]*q[3]};
        double sig[3];
        if (kind == 0) { for (int a = 0; a < 9; ++a) m[a] = 3e4 * gauss(); m[9] = 2e6; }             // random pair
        else {
            if (kind == 1) { sig[0] = 7e5; sig[1] = 6.5e5; sig[2] = 6.4e5; }                          // near superposition
            else if (kind == 2) { sig[0] = 7e5; sig[1] = 6.5e5; sig[2] = -6.4e5; }                    // reflected
            else { sig[0] = 7e5; sig[1] = 7e5 * (1 + 1e-9 * i); sig[2] = 1e3; }                       // degenerate pair
            for (int a = 0; a < 3; ++a)
                for (int c = 0; c < 3; ++c) m[3 * a + c] = Q[3 * a + c] * sig[c] + 10.0 * gauss();
            m[9] = 1.0000001 * (fabs(sig[0]) + fabs(sig[1]) + fabs(sig[2]));
        }
    }
    double *dR, *dl;
    long long* dc;
    int* di;
    cudaMalloc(&dR, sizeof(h));
    cudaMalloc(&dc, NV * n * sizeof(long long));
    cudaMalloc(&dl, NV * n * sizeof(double));
    cudaMalloc(&di, NV * n * sizeof(int));
    cudaMemcpy(dR, h, sizeof(h), cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 3; ++rep) kern<<<1, 32>>>(dR, n, dc, dl, di);
    static long long c[NV * n];
    static double l[NV * n];
    static int it[NV * n];
    cudaMemcpy(c, dc, sizeof(c), cudaMemcpyDeviceToHost);
    cudaMemcpy(l, dl, sizeof(l), cudaMemcpyDeviceToHost);
    cudaMemcpy(it, di, sizeof(it), cudaMemcpyDeviceToHost);
    const char* kinds[4] = {"random", "near-sup", "reflect", "degen"};
    for (int kind = 0; kind < 4; ++kind) {
        double cs[NV] = {}, is[NV] = {}, dmax[NV] = {};
        int cnt = 0, imax[NV] = {};
        for (int i = kind; i < n; i += 4) {
            ++cnt;
            for (int v = 0; v < NV; ++v) {
                cs[v] += c[NV * i + v];
                is[v] += it[NV * i + v];
                imax[v] = it[NV * i + v] > imax[v] ? it[NV * i + v] : imax[v];
                const double d = v >= 7 ? fabs(l[NV * i + v] - l[NV * i + 7]) : fabs(l[NV * i + v] - l[NV * i]) / fabs(l[NV * i]);
                dmax[v] = d > dmax[v] ? d : dmax[v];
            }
        }
        for (int v = 0; v < NV; ++v)
            printf("%-9s V%d %6.0f cyc, its %.1f (max %d), |dl|/l vs V0 %.1e\n", kinds[kind], v, cs[v] / cnt, is[v] / cnt, imax[v], dmax[v]);
    }
    return 0;
}
