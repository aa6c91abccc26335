// Throughput of SM-issued stores into pinned host memory (UVA): one double per
// lane per instruction (coalesced 256 B per warp) vs lanes 2 apart (the sweep's
// pattern), alone and concurrent with a 100 MB H2D copy on another stream.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 hostwrite_micro.cu -o hostwrite_micro
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_write(const double* __restrict__ src, double* dst, long n, int stride2) {
    long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long step = (long)gridDim.x * blockDim.x;
    for (; i < n; i += step) {
        long j = i;
        if (stride2) {   // lane l writes 2l, then 2l + 1 of its 64-element block
            const long blk = i / 64, r = i % 64;
            j = blk * 64 + (r < 32 ? 2 * r : 2 * (r - 32) + 1);
        }
        dst[j] = src[j];
    }
}

int main() {
    const long n = 100786200 / 8;
    double *d, *dsrc, *h, *h2;
    cudaMalloc(&d, n * 8);
    cudaMalloc(&dsrc, n * 8);
    cudaMemset(dsrc, 0, n * 8);
    cudaHostAlloc(&h, n * 8, cudaHostAllocDefault);
    cudaHostAlloc(&h2, n * 8, cudaHostAllocDefault);
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int grid : {148 * 4, 148 * 16}) {
        for (int stride2 = 0; stride2 < 2; ++stride2) {
            for (int duplex = 0; duplex < 2; ++duplex) {
                float best = 1e9;
                for (int rep = 0; rep < 4; ++rep) {
                    cudaDeviceSynchronize();
                    cudaEventRecord(a, s1);
                    cudaStreamWaitEvent(s2, a, 0);
                    if (duplex) cudaMemcpyAsync(d, h2, n * 8, cudaMemcpyHostToDevice, s2);
                    k_write<<<grid, 256, 0, s1>>>(dsrc, h, n, stride2);
                    cudaEvent_t e;
                    cudaEventCreate(&e);
                    cudaEventRecord(e, s2);
                    cudaStreamWaitEvent(s1, e, 0);
                    cudaEventRecord(b, s1);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    if (ms < best) best = ms;
                }
                printf("grid %5d %s %s: %.3f ms, %.1f GB/s per direction (%s)\n", grid,
                       stride2 ? "lanes 2 apart" : "coalesced   ", duplex ? "+H2D" : "    ", best,
                       n * 8 / best / 1e6, cudaGetErrorString(cudaGetLastError()));
            }
        }
    }
    return 0;
}
