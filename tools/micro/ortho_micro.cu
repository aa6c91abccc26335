// Micro-benchmark: multi-row dot (r = V[0..k) . w, t = V[0..k) . v) and
// multi-row update (w -= V h) kernel variants on a 12.6M-element basis.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ortho_micro ortho_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int RB = 592, RT = 256;

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}
__device__ double block_sum(double v) {
    __shared__ double sh[RT / 32];
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    v = threadIdx.x < RT / 32 ? sh[threadIdx.x] : 0.0;
    if (wid == 0) v = warp_sum(v);
    return v;
}

// V1: batches of R rows, grid-stride, scalar loads
template <int R>
__global__ void __launch_bounds__(RT) dots_v1(long n, int k, const double* V, long ldv,
                                              const double* w, const double* vj, double* part) {
    for (int i0 = 0; i0 < k; i0 += R) {
        double ar[R], at[R];
        for (int r = 0; r < R; ++r) ar[r] = at[r] = 0.0;
        for (long e = (long)blockIdx.x * RT + threadIdx.x; e < n; e += (long)gridDim.x * RT) {
            const double we = w[e], ve = vj[e];
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (i0 + r < k) {
                    const double x = V[(long)(i0 + r) * ldv + e];
                    ar[r] = fma(x, we, ar[r]);
                    at[r] = fma(x, ve, at[r]);
                }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (i0 + r >= k) break;
            const double a = block_sum(ar[r]), b = block_sum(at[r]);
            if (threadIdx.x == 0) { part[(2 * (i0 + r)) * RB + blockIdx.x] = a; part[(2 * (i0 + r) + 1) * RB + blockIdx.x] = b; }
        }
    }
}

// V3: 2-D grid (element chunk x row batch), double2 loads, contiguous chunk per block
template <int R>
__global__ void __launch_bounds__(RT) dots_v3(long n2, int k, const double2* V, long ldv2,
                                              const double2* w, const double2* vj, double* part, long chunk) {
    const int i0 = blockIdx.y * R;
    double ar[R], at[R];
    for (int r = 0; r < R; ++r) ar[r] = at[r] = 0.0;
    const long e0 = (long)blockIdx.x * chunk, e1 = min(n2, e0 + chunk);
    for (long e = e0 + threadIdx.x; e < e1; e += RT) {
        const double2 we = w[e], ve = vj[e];
#pragma unroll
        for (int r = 0; r < R; ++r)
            if (i0 + r < k) {
                const double2 x = V[(long)(i0 + r) * ldv2 + e];
                ar[r] = fma(x.x, we.x, fma(x.y, we.y, ar[r]));
                at[r] = fma(x.x, ve.x, fma(x.y, ve.y, at[r]));
            }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        if (i0 + r >= k) break;
        const double a = block_sum(ar[r]), b = block_sum(at[r]);
        if (threadIdx.x == 0) { part[(2 * (i0 + r)) * gridDim.x + blockIdx.x] = a; part[(2 * (i0 + r) + 1) * gridDim.x + blockIdx.x] = b; }
    }
}

// update U1: runtime row loop
__global__ void __launch_bounds__(RT) upd_u1(long n, int k, const double* V, long ldv, const double* h, double* w, double* part) {
    double v = 0.0;
    for (long e = (long)blockIdx.x * RT + threadIdx.x; e < n; e += (long)gridDim.x * RT) {
        double acc = 0.0;
        for (int i = 0; i < k; ++i) acc = fma(h[i], V[(long)i * ldv + e], acc);
        const double we = w[e] - acc;
        w[e] = we;
        v = fma(we, we, v);
    }
    const double s = block_sum(v);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// update U2: double2, h in smem, rows unrolled by 8 with loads first, contiguous chunks
__global__ void __launch_bounds__(RT) upd_u2(long n2, int k, const double2* V, long ldv2, const double* h,
                                             double2* w, double* part, long chunk) {
    __shared__ double hs[1024];
    for (int i = threadIdx.x; i < k; i += RT) hs[i] = h[i];
    __syncthreads();
    double v = 0.0;
    const long e0 = (long)blockIdx.x * chunk, e1 = min(n2, e0 + chunk);
    for (long e = e0 + threadIdx.x; e < e1; e += RT) {
        double ax = 0.0, ay = 0.0;
        for (int i0 = 0; i0 < k; i0 += 8) {
            double2 x[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) x[r] = i0 + r < k ? V[(long)(i0 + r) * ldv2 + e] : make_double2(0.0, 0.0);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const double hr = i0 + r < k ? hs[i0 + r] : 0.0;
                ax = fma(hr, x[r].x, ax);
                ay = fma(hr, x[r].y, ay);
            }
        }
        double2 we = w[e];
        we.x -= ax;
        we.y -= ay;
        w[e] = we;
        v = fma(we.x, we.x, fma(we.y, we.y, v));
    }
    const double s = block_sum(v);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// update U3: scalar, rows in chunks of R with loads first
template <int R>
__global__ void __launch_bounds__(RT) upd_u3(long n, int k, const double* V, long ldv, const double* h, double* w, double* part) {
    __shared__ double hs[1024];
    for (int i = threadIdx.x; i < k; i += RT) hs[i] = h[i];
    __syncthreads();
    double v = 0.0;
    for (long e = (long)blockIdx.x * RT + threadIdx.x; e < n; e += (long)gridDim.x * RT) {
        double acc = 0.0;
        for (int i0 = 0; i0 < k; i0 += R) {
            double x[R];
#pragma unroll
            for (int r = 0; r < R; ++r) x[r] = i0 + r < k ? V[(long)(i0 + r) * ldv + e] : 0.0;
#pragma unroll
            for (int r = 0; r < R; ++r) acc = fma(i0 + r < k ? hs[i0 + r] : 0.0, x[r], acc);
        }
        const double we = w[e] - acc;
        w[e] = we;
        v = fma(we, we, v);
    }
    const double s = block_sum(v);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// update U4: two passes over rows in chunks of 4: out-of-place partial sums kept in w
// (w -= sum over 4 rows per pass; reads w once per 4 rows)
__global__ void __launch_bounds__(RT) upd_u4(long n, int k, const double* V, long ldv, const double* h, double* w, double* part) {
    __shared__ double hs[1024];
    for (int i = threadIdx.x; i < k; i += RT) hs[i] = h[i];
    __syncthreads();
    double v = 0.0;
    for (int i0 = 0; i0 < k; i0 += 4) {
        const bool last = i0 + 4 >= k;
        for (long e = (long)blockIdx.x * RT + threadIdx.x; e < n; e += (long)gridDim.x * RT) {
            double acc = 0.0;
#pragma unroll
            for (int r = 0; r < 4; ++r)
                if (i0 + r < k) acc = fma(hs[i0 + r], V[(long)(i0 + r) * ldv + e], acc);
            const double we = w[e] - acc;
            w[e] = we;
            if (last) v = fma(we, we, v);
        }
    }
    const double s = block_sum(v);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// update U5: rows in chunks of 8 with independent partial sums, 2 elements per thread
__global__ void __launch_bounds__(RT) upd_u5(long n, int k, const double* V, long ldv, const double* h, double* w, double* part) {
    __shared__ double hs[1024];
    for (int i = threadIdx.x; i < k; i += RT) hs[i] = h[i];
    __syncthreads();
    double v = 0.0;
    const long stride = (long)gridDim.x * RT;
    for (long e = (long)blockIdx.x * RT + threadIdx.x; e < n; e += 2 * stride) {
        const long e2 = e + stride;
        const bool two = e2 < n;
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
        int i = 0;
        for (; i + 1 < k; i += 2) {
            const double h0 = hs[i], h1 = hs[i + 1];
            const double* r0 = V + (long)i * ldv;
            const double* r1 = r0 + ldv;
            a0 = fma(h0, r0[e], a0);
            a1 = fma(h1, r1[e], a1);
            if (two) { b0 = fma(h0, r0[e2], b0); b1 = fma(h1, r1[e2], b1); }
        }
        if (i < k) {
            a0 = fma(hs[i], V[(long)i * ldv + e], a0);
            if (two) b0 = fma(hs[i], V[(long)i * ldv + e2], b0);
        }
        const double we = w[e] - (a0 + a1);
        w[e] = we;
        v = fma(we, we, v);
        if (two) {
            const double we2 = w[e2] - (b0 + b1);
            w[e2] = we2;
            v = fma(we2, we2, v);
        }
    }
    const double s = block_sum(v);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

int main() {
    const long n = 12598275, ldv = (n + 63) / 64 * 64, n2 = ldv / 2;
    const int m = 31;
    double *V, *w, *part, *h;
    cudaMalloc(&V, sizeof(double) * ldv * m);
    cudaMalloc(&w, sizeof(double) * ldv);
    cudaMalloc(&part, sizeof(double) * 2 * m * 4096);
    cudaMalloc(&h, sizeof(double) * m);
    cudaMemset(V, 0, sizeof(double) * ldv * m);
    cudaMemset(w, 0, sizeof(double) * ldv);
    cudaMemset(h, 0, sizeof(double) * m);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](const char* name, int k, double vecs, auto fn) {
        fn();
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) fn();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 5;
        printf("k=%2d %-28s %8.1f us  %.2f TB/s\n", k, name, ms * 1e3, vecs * n * 8 / (ms * 1e-3) / 1e12);
    };
    for (int k : {1, 8, 16, 30}) {
        const double dv = k + 2, uv = k + 2;
        timeit("dots v1 R=4", k, dv, [&] { dots_v1<4><<<RB, RT>>>(n, k, V, ldv, w, V, part); });
        timeit("upd u1", k, uv, [&] { upd_u1<<<RB, RT>>>(n, k, V, ldv, h, w, part); });
        timeit("upd u5 (2 elem, 2 chains)", k, uv, [&] { upd_u5<<<RB, RT>>>(n, k, V, ldv, h, w, part); });
        timeit("upd u5 x2 grid", k, uv, [&] { upd_u5<<<2 * RB, RT>>>(n, k, V, ldv, h, w, part); });
        timeit("upd u3 R=4", k, uv, [&] { upd_u3<4><<<RB, RT>>>(n, k, V, ldv, h, w, part); });
        timeit("upd u3 R=2", k, uv, [&] { upd_u3<2><<<RB, RT>>>(n, k, V, ldv, h, w, part); });
        timeit("upd u3 R=4 x2 grid", k, uv, [&] { upd_u3<4><<<2 * RB, RT>>>(n, k, V, ldv, h, w, part); });
        timeit("upd u4 (4-row passes)", k, uv, [&] { upd_u4<<<RB, RT>>>(n, k, V, ldv, h, w, part); });
        timeit("dots v1 R=2", k, dv, [&] { dots_v1<2><<<RB, RT>>>(n, k, V, ldv, w, V, part); });
        timeit("dots v1 R=4 x2 grid", k, dv, [&] { dots_v1<4><<<2 * RB, RT>>>(n, k, V, ldv, w, V, part); });
    }
    return 0;
}
