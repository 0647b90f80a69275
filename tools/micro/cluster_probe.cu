// Probe of the cluster exchange primitives used by bb_forward_cl_kernel:
// rank 0 sends 4 floats to rank 1's shared memory and arrives on its mbarrier.
// variant (argv[1]): 0 = full protocol, 1 = no cluster wait before the remote
// access, 2 = aligned cluster wait by all threads, 3 = no exchange at all.
#include <cstdio>
#include <cstdlib>
#include "../../paper_1812_01108_b200/csrc/common.cuh"
using namespace tpl;
namespace tpl { bool pdl_enabled() { return false; } }

__global__ void probe(float* out, int variant) {
    __shared__ __align__(16) uint64_t bar[2];
    __shared__ __align__(16) float slot[4];
    const unsigned rank = cluster_ctarank();
    if (threadIdx.x == 0) {
        mbar_init(bar + 1, 1);
        fence_mbarrier_init_cluster();
    }
    __syncthreads();
    cluster_arrive_relaxed();
    if (variant == 2) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    if (variant == 3) { out[blockIdx.x] = 1.f; return; }
    if (rank == 0 && threadIdx.x == 0) {
        if (variant == 0) asm volatile("barrier.cluster.wait;" ::: "memory");
        const uint32_t dst = mapa_shared(smem_u32(slot), 1);
        st_cluster_v4(dst, 1.f + blockIdx.x, 2.f, 3.f, 4.f);
        mbar_arrive_remote(mapa_shared(smem_u32(bar + 1), 1));
    }
    if (rank == 1) {
        mbar_wait_cluster(bar + 1, 0);
        if (threadIdx.x == 0) out[blockIdx.x] = slot[0] + slot[1] + slot[2] + slot[3];
    }
}

int main(int argc, char** argv) {
    const int variant = argc > 1 ? atoi(argv[1]) : 0;
    float* d;
    cudaMalloc(&d, 1024 * 4);
    cudaMemset(d, 0, 1024 * 4);
    cudaError_t e = launch_cluster(probe, 8, 2, 128, 0, (cudaStream_t)0, d, variant);
    printf("launch: %s\n", cudaGetErrorString(e));
    e = cudaDeviceSynchronize();
    printf("sync: %s\n", cudaGetErrorString(e));
    float h[8];
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 8; ++i) printf("%g ", h[i]);
    printf("\n");
    return 0;
}
