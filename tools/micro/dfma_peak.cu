// FP64 peak of this B200: DFMA, DADD/DMUL issue throughput, measured.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/micro/dfma_peak \
//        tools/micro/dfma_peak.cu && tools/micro/dfma_peak > profiles/fp64_peak.json
//
// Every thread runs ILP independent FMA chains (no memory traffic inside the
// loop); grids of 148 x {1..16} CTAs x 256 threads, best of 10 timed launches
// per grid with CUDA events.  Prints one JSON object: the best DFMA rate in
// TFLOP/s (2 flops per DFMA) and DFMA instructions per SM per clock (at the
// SM clock the driver reports during the run), which is the denominator of
// the FP64 fractions bench.py reports.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ILP = 8;

__global__ void __launch_bounds__(256) k_dfma(double* out, double a, double b, int iters) {
    double acc[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) acc[k] = threadIdx.x * 1e-9 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < ILP; ++k) acc[k] = fma(acc[k], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += acc[k];
    if (s == 12345.678) out[0] = s;   // never true: keeps the chains alive
}

__global__ void __launch_bounds__(256) k_dadd(double* out, double a, int iters) {
    double acc[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) acc[k] = threadIdx.x * 1e-9 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < ILP; ++k) acc[k] = acc[k] + a;
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += acc[k];
    if (s == 12345.678) out[0] = s;
}

int main() {
    cudaDeviceProp pr;
    cudaGetDeviceProperties(&pr, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 1 << 14;
    double best_fma = 0.0, best_add = 0.0;
    int best_cta = 0;
    for (int per_sm = 1; per_sm <= 16; per_sm *= 2) {
        const int grid = pr.multiProcessorCount * per_sm;
        for (int kind = 0; kind < 2; ++kind) {
            for (int rep = 0; rep < 11; ++rep) {
                cudaEventRecord(e0);
                if (kind == 0) k_dfma<<<grid, 256>>>(out, 0.999999, 1e-7, iters);
                else k_dadd<<<grid, 256>>>(out, 1e-7, iters);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0.f;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep == 0) continue;   // warm-up
                const double inst = (double)grid * 256 * iters * ILP;
                const double rate = inst / (ms * 1e-3);   // thread-instructions / s
                if (kind == 0 && rate > best_fma) { best_fma = rate; best_cta = per_sm; }
                if (kind == 1 && rate > best_add) best_add = rate;
            }
        }
    }
    if (cudaGetLastError() != cudaSuccess) { fprintf(stderr, "CUDA error\n"); return 1; }
    const double sms = pr.multiProcessorCount;
    const double ghz_max = clk_khz * 1e-6;
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"dfma_tflops\": %.2f, \"dfma_per_s\": %.4e, "
           "\"dadd_per_s\": %.4e, \"dfma_lanes_per_sm_per_clk_at_max_clock\": %.1f, "
           "\"sm_max_ghz\": %.3f, \"best_ctas_per_sm\": %d, \"ilp\": %d, "
           "\"how\": \"tools/micro/dfma_peak.cu: %d independent DFMA chains per thread, 256 "
           "threads per CTA, 148 x {1,2,4,8,16} CTAs, best of 10 CUDA-event-timed launches\"}\n",
           pr.name, pr.multiProcessorCount, 2.0 * best_fma * 1e-12, best_fma, best_add,
           best_fma / (sms * ghz_max * 1e9), ghz_max, best_cta, ILP, ILP);
    return 0;
}
