// pff_vec.cu -- fused vector kernels of the smoother and the Krylov solver.
//
// Chebyshev-Jacobi recurrence: src/multigrid.py:170-198.  Constraint masks of
// the V-cycle: src/multigrid.py:330-344.  Modified Gram-Schmidt of GMRES:
// src/krylov.py:76-79, fused as one "axpy(i) + dot(i+1)" pass per step with
// the coefficient kept on device.  All reductions run on a fixed grid of
// RED_BLOCKS blocks with a fixed tree order, so results are deterministic.
#include "pff_internal.cuh"

namespace pff {

namespace {

inline unsigned blocks(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

// layout 0: 3n [dir | dir | act]; 1: 2n [dir | dir]; 2: n [act]
__device__ __forceinline__ bool is_cons(uint8_t f, int layout, int comp) {
    if (layout == 2) return f & F_ACT;
    return comp < 2 ? (f & F_DIR) : (f & F_ACT);
}

// op 0: z = cons ? r : 0; op 1: z[cons] = 0; op 2: z[cons] = r[cons]
__global__ void k_cons(int64_t n, const uint8_t* __restrict__ flags, int layout, int op,
                       const double* __restrict__ r, double* __restrict__ z) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint8_t f = flags[i];
    const int nc = layout == 0 ? 3 : (layout == 1 ? 2 : 1);
    for (int c = 0; c < nc; ++c) {
        const int64_t k = c * n + i;
        const bool cons = is_cons(f, layout, c);
        if (op == 0)
            z[k] = cons ? r[k] : 0.0;
        else if (op == 3)
            z[k] = cons ? 0.0 : r[k];
        else if (cons)
            z[k] = op == 1 ? 0.0 : r[k];
    }
}

// first smoothing of a V-cycle level (z = 0 on entry): z = SELECT(r) (3n),
// res_u = EXCLUDE(r) on the u rows and the u block's Chebyshev
// d0 = invd_u res_u / theta -- the cons SELECT, cons EXCLUDE and cheb_init
// passes in one (same values bit for bit; z += d0 is left to the first
// fused step, pff_apply_cheb_first)
__global__ void k_smooth_init(int64_t n, const uint8_t* __restrict__ flags,
                              const double* __restrict__ r, double* __restrict__ z,
                              double* __restrict__ res_u, const double* __restrict__ invd_u,
                              double* __restrict__ d_u, double theta, bool add_d0) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint8_t f = flags[i];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int64_t k = c * n + i;
        const bool cons = is_cons(f, 0, c);
        const double rv = r[k];
        double zv = cons ? rv : 0.0;
        if (c < 2) {
            const double rr = cons ? 0.0 : rv;
            res_u[k] = rr;
            const double d0 = invd_u[k] * rr / theta;
            d_u[k] = d0;
            if (add_d0) zv += d0;   // exact: one of the two terms is zero
        }
        z[k] = zv;
    }
}

__global__ void k_cheb_init(int64_t n, const double* __restrict__ invd,
                            const double* __restrict__ rhs, double theta, double* __restrict__ d,
                            double* __restrict__ acc, int acc_mode) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double v = invd[i] * rhs[i] / theta;
    d[i] = v;
    if (acc_mode == 0) acc[i] = v;
    else if (acc_mode == 1) acc[i] += v;
}

__global__ void k_cheb_step(int64_t n, const double* __restrict__ invd,
                            const double* __restrict__ r, double c1, double c2,
                            double* __restrict__ d, double* __restrict__ acc) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double v = cheb_update(c1, d[i], c2, invd[i], r[i]);
    d[i] = v;
    acc[i] += v;
}

__global__ void k_axpby(int64_t n, double a, const double* __restrict__ x, double b,
                        double* __restrict__ y) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    y[i] = b == 0.0 ? a * x[i] : (a == 1.0 && b == 1.0 ? y[i] + x[i] : a * x[i] + b * y[i]);
}

__global__ void k_div(int64_t n, const double* __restrict__ x, const double* __restrict__ sdev,
                      double sval, double* __restrict__ y) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double s = sdev ? *sdev : sval;
    y[i] = x[i] / s;
}

__global__ void k_mul(int64_t n, const double* __restrict__ a, const double* __restrict__ x,
                      double* __restrict__ y) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    y[i] = a[i] * x[i];
}

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double sh[RED_THREADS / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double s = 0.0;
    if (wid == 0) {
        s = lane < RED_THREADS / 32 ? sh[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    }
    return s;  // valid in thread 0
}

// sum of RED_BLOCKS partials in a fixed order; every block gets the same bits
__device__ __forceinline__ double reduce_partials(const double* __restrict__ part) {
    double v = 0.0;
    for (int k = threadIdx.x; k < RED_BLOCKS; k += RED_THREADS) v += part[k];
    __shared__ double total;
    double s = block_sum(v);
    if (threadIdx.x == 0) total = s;
    __syncthreads();
    return total;
}

__global__ void __launch_bounds__(RED_THREADS)
k_dot_partials(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
               double* __restrict__ part) {
    double v = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * RED_THREADS + threadIdx.x; i < n;
         i += (int64_t)RED_BLOCKS * RED_THREADS)
        v = fma(x[i], y[i], v);
    double s = block_sum(v);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(RED_THREADS)
k_reduce_final(const double* __restrict__ part, double* out, int take_sqrt) {
    double s = reduce_partials(part);
    if (threadIdx.x == 0) *out = take_sqrt ? sqrt(s) : s;
}

// MGS step i of column j: h[i] = <partials_in>; w -= h[i] V[i];
// partials_out = V[i+1] . w (i < j) or w . w (i == j)
__global__ void __launch_bounds__(RED_THREADS)
k_mgs_step(int64_t n, const double* __restrict__ V, int64_t ldv, double* __restrict__ w,
           const double* __restrict__ pin, double* __restrict__ pout, double* __restrict__ h,
           int i, int j) {
    const double hi = reduce_partials(pin);
    if (blockIdx.x == 0 && threadIdx.x == 0) h[i] = hi;
    const double* vi = V + (int64_t)i * ldv;
    const double* vn = i < j ? V + (int64_t)(i + 1) * ldv : nullptr;
    double v = 0.0;
    for (int64_t k = (int64_t)blockIdx.x * RED_THREADS + threadIdx.x; k < n;
         k += (int64_t)RED_BLOCKS * RED_THREADS) {
        double wk = w[k] - hi * vi[k];
        w[k] = wk;
        v = fma(vn ? vn[k] : wk, wk, v);
    }
    double s = block_sum(v);
    if (threadIdx.x == 0) pout[blockIdx.x] = s;
}

// multi-dot: part[i][block] = sum over the block's elements of V[i] . w, 4 rows
// of V per pass (w re-read once per 4 rows); fixed grid -> deterministic
constexpr int MDOT_ROWS = 4;   // 8 rows per pass halves the achieved bandwidth (tools/micro/ortho_micro.cu)
__global__ void __launch_bounds__(RED_THREADS)
k_mdot_partials(int64_t n, int k, const double* __restrict__ V, int64_t ldv,
                const double* __restrict__ w, double* __restrict__ part) {
    for (int i0 = 0; i0 < k; i0 += MDOT_ROWS) {
        double acc[MDOT_ROWS];
#pragma unroll
        for (int r = 0; r < MDOT_ROWS; ++r) acc[r] = 0.0;
        for (int64_t e = (int64_t)blockIdx.x * RED_THREADS + threadIdx.x; e < n;
             e += (int64_t)RED_BLOCKS * RED_THREADS) {
            const double we = w[e];
#pragma unroll
            for (int r = 0; r < MDOT_ROWS; ++r)
                if (i0 + r < k) acc[r] = fma(V[(int64_t)(i0 + r) * ldv + e], we, acc[r]);
        }
#pragma unroll
        for (int r = 0; r < MDOT_ROWS; ++r) {
            if (i0 + r >= k) break;
            const double s = block_sum(acc[r]);
            if (threadIdx.x == 0) part[(int64_t)(i0 + r) * RED_BLOCKS + blockIdx.x] = s;
        }
    }
}

__global__ void __launch_bounds__(RED_THREADS)
k_mdot_final(const double* __restrict__ part, double* out) {
    const double s = reduce_partials(part + (int64_t)blockIdx.x * RED_BLOCKS);
    if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// Low-synchronisation MGS (inverse compact-WY form) for Arnoldi column j:
// one pass computes r = V[0..j] . w and the new Gram row t = V[0..j-1] . V[j];
// the MGS coefficients follow exactly from h_i = r_i - sum_{k<i} (v_i.v_k) h_k
// (the recurrence MGS evaluates with updated w), then one pass forms
// w -= V h and |w|^2.  4 basis rows per pass, fixed grid -> deterministic.
#ifndef LSMGS_ROWS
#define LSMGS_ROWS 4   // basis rows per pass of the low-sync partials (A/B knob at build time)
#endif
__global__ void __launch_bounds__(RED_THREADS)
k_lsmgs_partials(int64_t n, int j, const double* __restrict__ V, int64_t ldv,
                 const double* __restrict__ w, double* __restrict__ part) {
    constexpr int RR = LSMGS_ROWS;
    const double* vj = V + (int64_t)j * ldv;
    for (int i0 = 0; i0 <= j; i0 += RR) {
        double ar[RR], at[RR];
#pragma unroll
        for (int r = 0; r < RR; ++r) ar[r] = at[r] = 0.0;
        for (int64_t e = (int64_t)blockIdx.x * RED_THREADS + threadIdx.x; e < n;
             e += (int64_t)RED_BLOCKS * RED_THREADS) {
            const double we = w[e], ve = vj[e];
#pragma unroll
            for (int r = 0; r < RR; ++r)
                if (i0 + r <= j) {
                    const double vi = V[(int64_t)(i0 + r) * ldv + e];
                    ar[r] = fma(vi, we, ar[r]);
                    at[r] = fma(vi, ve, at[r]);
                }
        }
#pragma unroll
        for (int r = 0; r < RR; ++r) {
            if (i0 + r > j) break;
            const double sr = block_sum(ar[r]);
            const double st = block_sum(at[r]);
            if (threadIdx.x == 0) {
                part[(int64_t)(2 * (i0 + r)) * RED_BLOCKS + blockIdx.x] = sr;
                part[(int64_t)(2 * (i0 + r) + 1) * RED_BLOCKS + blockIdx.x] = st;
            }
        }
    }
}

// one block: finish the 2(j+1) sums (one warp per sum, fixed order), store
// the Gram row j, forward-substitute h
constexpr int SOLVE_THREADS = 1024;
__global__ void __launch_bounds__(SOLVE_THREADS)
k_lsmgs_solve(int j, const double* __restrict__ part, double* __restrict__ gram, int64_t ldg,
              double* __restrict__ h) {
    __shared__ double r[1024];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int q = wid; q < 2 * (j + 1); q += SOLVE_THREADS / 32) {
        const double* p = part + (int64_t)q * RED_BLOCKS;
        double v = 0.0;
        for (int k = lane; k < RED_BLOCKS; k += 32) v += p[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (lane == 0) {
            const int i = q >> 1;
            if ((q & 1) == 0) r[i] = v;
            else if (i < j) gram[(int64_t)j * ldg + i] = v;   // v_j . v_i, i < j
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 0; i <= j; ++i) {
            double hi = r[i];
            for (int k = 0; k < i; ++k) hi = fma(-gram[(int64_t)i * ldg + k], h[k], hi);
            h[i] = hi;
        }
    }
}

// w -= sum_i h[i] V[i]; part = per-block |w|^2.  Bandwidth form: h in shared
// memory, two elements per thread and the basis rows loaded in independent
// batches of 4 ahead of their FMAs (the per-element sum keeps the order
// i = 0..j); one pass over the j+1 rows.
constexpr int LSU_HMAX = 512;
__global__ void __launch_bounds__(RED_THREADS)
k_lsmgs_update(int64_t n, int j, const double* __restrict__ V, int64_t ldv,
               const double* __restrict__ h, double* __restrict__ w, double* __restrict__ part) {
    __shared__ double hs[LSU_HMAX];
    const bool sm = j < LSU_HMAX;
    if (sm)
        for (int i = threadIdx.x; i <= j; i += RED_THREADS) hs[i] = h[i];
    __syncthreads();
    const double* hp = sm ? hs : h;
    double v = 0.0;
    const int64_t stride = (int64_t)RED_BLOCKS * RED_THREADS * 2;
    for (int64_t e0 = (int64_t)blockIdx.x * RED_THREADS * 2 + threadIdx.x; e0 < n; e0 += stride) {
        const int64_t e1 = e0 + RED_THREADS;
        const bool two = e1 < n;
        const double w0 = w[e0], w1 = two ? w[e1] : 0.0;
        double a0 = 0.0, a1 = 0.0;
        int i = 0;
        for (; i + 4 <= j + 1; i += 4) {
            double x0[4], x1[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const double* vr = V + (int64_t)(i + r) * ldv;
                x0[r] = vr[e0];
                x1[r] = two ? vr[e1] : 0.0;
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                a0 = fma(hp[i + r], x0[r], a0);
                a1 = fma(hp[i + r], x1[r], a1);
            }
        }
        for (; i <= j; ++i) {
            const double* vr = V + (int64_t)i * ldv;
            a0 = fma(hp[i], vr[e0], a0);
            if (two) a1 = fma(hp[i], vr[e1], a1);
        }
        const double we0 = w0 - a0;
        w[e0] = we0;
        v = fma(we0, we0, v);
        if (two) {
            const double we1 = w1 - a1;
            w[e1] = we1;
            v = fma(we1, we1, v);
        }
    }
    const double s = block_sum(v);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// out = sum_i y[i] V[i]  (+ out)
__global__ void k_combine(int64_t n, int k, const double* __restrict__ V, int64_t ldv,
                          const double* __restrict__ y, double* __restrict__ out, int accumulate) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    double acc = 0.0;
    for (int i = 0; i < k; ++i) acc = fma(y[i], V[(int64_t)i * ldv + e], acc);
    out[e] = accumulate ? out[e] + acc : acc;
}

}  // namespace

cudaError_t launch_cons(const Level& L, int layout, int op, const double* r, double* z,
                        cudaStream_t s) {
    const int64_t n = L.local_n();
    k_cons<<<blocks(n), 256, 0, s>>>(n, L.flags, layout, op, r, z);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_smooth_init(const Level& L, const double* r, double* z, double* res_u,
                               const double* invd_u, double* d_u, double theta, bool add_d0,
                               cudaStream_t s) {
    const int64_t n = L.local_n();
    k_smooth_init<<<blocks(n), 256, 0, s>>>(n, L.flags, r, z, res_u, invd_u, d_u, theta, add_d0);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_cheb_init(int64_t n, const double* invd, const double* rhs, double theta,
                             double* d, double* acc, int acc_mode, cudaStream_t s) {
    k_cheb_init<<<blocks(n), 256, 0, s>>>(n, invd, rhs, theta, d, acc, acc_mode);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_cheb_step(int64_t n, const double* invd, const double* r, double c1,
                             double c2, double* d, double* acc, cudaStream_t s) {
    k_cheb_step<<<blocks(n), 256, 0, s>>>(n, invd, r, c1, c2, d, acc);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_axpby(int64_t n, double a, const double* x, double b, double* y,
                         cudaStream_t s) {
    k_axpby<<<blocks(n), 256, 0, s>>>(n, a, x, b, y);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_div(int64_t n, const double* x, const double* sdev, double sval, double* y,
                       cudaStream_t s) {
    k_div<<<blocks(n), 256, 0, s>>>(n, x, sdev, sval, y);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_dot(int64_t n, const double* x, const double* y, double* partials,
                       double* out, cudaStream_t s) {
    k_dot_partials<<<RED_BLOCKS, RED_THREADS, 0, s>>>(n, x, y, partials);
    if (out) k_reduce_final<<<1, RED_THREADS, 0, s>>>(partials, out, 0);
    count_launches(out ? 2 : 1);
    return cudaGetLastError();
}

cudaError_t launch_mgs(int64_t n, int j, const double* V, int64_t ldv, double* w,
                       double* partials, double* h, cudaStream_t s) {
    double* pa = partials;
    double* pb = partials + RED_BLOCKS;
    k_dot_partials<<<RED_BLOCKS, RED_THREADS, 0, s>>>(n, V, w, pa);
    for (int i = 0; i <= j; ++i) {
        k_mgs_step<<<RED_BLOCKS, RED_THREADS, 0, s>>>(n, V, ldv, w, pa, pb, h, i, j);
        double* t = pa;
        pa = pb;
        pb = t;
    }
    k_reduce_final<<<1, RED_THREADS, 0, s>>>(pa, h + j + 1, 1);
    count_launches(j + 3);
    return cudaGetLastError();
}

cudaError_t launch_lsmgs(int64_t n, int j, const double* V, int64_t ldv, double* w,
                         double* gram, int64_t ldg, double* partials, double* h, cudaStream_t s) {
    k_lsmgs_partials<<<RED_BLOCKS, RED_THREADS, 0, s>>>(n, j, V, ldv, w, partials);
    k_lsmgs_solve<<<1, SOLVE_THREADS, 0, s>>>(j, partials, gram, ldg, h);
    double* pn = partials + (int64_t)2 * (j + 1) * RED_BLOCKS;
    k_lsmgs_update<<<RED_BLOCKS, RED_THREADS, 0, s>>>(n, j, V, ldv, h, w, pn);
    k_reduce_final<<<1, RED_THREADS, 0, s>>>(pn, h + j + 1, 1);
    count_launches(4);
    return cudaGetLastError();
}

cudaError_t launch_mdot(int64_t n, int k, const double* V, int64_t ldv, const double* w,
                        double* partials, double* out, cudaStream_t s) {
    if (k <= 0) return cudaSuccess;
    k_mdot_partials<<<RED_BLOCKS, RED_THREADS, 0, s>>>(n, k, V, ldv, w, partials);
    k_mdot_final<<<k, RED_THREADS, 0, s>>>(partials, out);
    count_launches(2);
    return cudaGetLastError();
}

cudaError_t launch_combine(int64_t n, int k, const double* V, int64_t ldv, const double* y,
                           double* out, int accumulate, cudaStream_t s) {
    k_combine<<<blocks(n), 256, 0, s>>>(n, k, V, ldv, y, out, accumulate);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_lanczos_scale(int64_t n, const double* dhalf, const double* v, double* out,
                                 cudaStream_t s) {
    k_mul<<<blocks(n), 256, 0, s>>>(n, dhalf, v, out);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace pff
