// Micro-benchmark: per-launch time of an empty kernel inside a CUDA graph (the
// floor under every kernel of the step), plain and with programmatic dependent launch.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void empty_kernel(int* p) {
    if (p && threadIdx.x == 0 && blockIdx.x == 1 << 30) p[0] = 1;
}
__global__ void empty_pdl(int* p) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (p && threadIdx.x == 0 && blockIdx.x == 1 << 30) p[0] = 1;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

static float run(int grid, int block, bool pdl, int n) {
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < n; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(block);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, pdl ? empty_pdl : empty_kernel, (int*)nullptr);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0, s);
        cudaGraphLaunch(ge, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best * 1e3f / n;
}

int main() {
    const int n = 200;
    int grids[] = {1, 148, 256, 592, 4096};
    for (int gi = 0; gi < 5; ++gi)
        printf("grid %5d x 128: %.2f us/launch, with PDL %.2f us/launch\n", grids[gi], run(grids[gi], 128, false, n),
               run(grids[gi], 128, true, n));
    return 0;
}
