// Chain of small dependent kernels captured in a CUDA graph, with and without
// programmatic dependent launch (PDL): per-kernel time at the latency floor.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 pdl_micro.cu -o pdl_micro
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_step(const double* __restrict__ x, double* __restrict__ y, int n, int pdl) {
    if (pdl) {
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        y[i] = 0.5 * x[i] + 1.0;
}

int main() {
    const int reps = 200;
    for (int n : {3 * 1089, 3 * 4225, 3 * 16641, 3 * 66049}) {
        double *a, *b;
        cudaMalloc(&a, n * 8);
        cudaMalloc(&b, n * 8);
        cudaMemset(a, 0, n * 8);
        cudaStream_t s;
        cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        const int grid = (n + 255) / 256;
        for (int pdl = 0; pdl < 2; ++pdl) {
            cudaGraph_t g;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
            for (int r = 0; r < reps; ++r) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(grid);
                cfg.blockDim = dim3(256);
                cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = pdl ? 1 : 0;
                const double* x = (r & 1) ? b : a;
                double* y = (r & 1) ? a : b;
                cudaLaunchKernelEx(&cfg, k_step, x, y, n, pdl);
            }
            cudaStreamEndCapture(s, &g);
            cudaGraphExec_t ge;
            if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed\n"); return 1; }
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaGraphLaunch(ge, s);
            cudaEventRecord(e0, s);
            for (int k = 0; k < 5; ++k) cudaGraphLaunch(ge, s);
            cudaEventRecord(e1, s);
            cudaStreamSynchronize(s);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("n %7d grid %4d pdl %d: %.2f us per kernel (%s)\n", n, grid, pdl, ms * 1e3 / (5 * reps),
                   cudaGetErrorString(cudaGetLastError()));
            cudaGraphExecDestroy(ge);
            cudaGraphDestroy(g);
        }
        cudaFree(a);
        cudaFree(b);
    }
    return 0;
}
