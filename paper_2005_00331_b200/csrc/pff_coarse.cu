// pff_coarse.cu -- the coarse-level solve of the V-cycle as dense linear maps.
//
// The reference's coarse solve (src/multigrid.py:311-328) is a fixed number of
// Jacobi-Chebyshev sweeps on the u block, then the phi row with z_phi = 0, then
// Chebyshev on the phi block, then the constrained rows copied from r.  For a
// fixed linearisation point and fixed ranges each Chebyshev pass is a fixed
// matrix polynomial, so setup forms C_u = P_u(G_uu) and C_phi = P_phi(G_phiphi)
// once (multigrid.py _build_dense_coarse, the reference recurrence run on the
// identity) and every V-cycle applies
//     z_u = C_u r_u,  t = r_phi - G_phiu z_u,  z_phi = C_phi t,  z[c] = r[c]
// in ONE single-CTA launch instead of ~130 small operator launches.  Row sums
// run lane-strided then through a fixed shuffle tree: deterministic.
#include "pff_internal.cuh"

namespace pff {

namespace {

constexpr int CD_THREADS = 512;
constexpr int CD_NMAX = 256;   // scalar nodes of the coarse level (3n <= 768)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// y[i] = (b ? b[i] : 0) - sgn * sum_j M[i, j] x[j] for i < rows (M row-major, ld = cols)
__device__ __forceinline__ void matvec(int rows, int cols, const double* __restrict__ M,
                                       const double* x, const double* b, double sgn, double* y) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int i = wid; i < rows; i += CD_THREADS / 32) {
        const double* mi = M + (int64_t)i * cols;
        double acc = 0.0;
        for (int j = lane; j < cols; j += 32) acc = fma(mi[j], x[j], acc);
        acc = warp_sum(acc);
        if (lane == 0) y[i] = (b ? b[i] : 0.0) - sgn * acc;
    }
}

__global__ void __launch_bounds__(CD_THREADS)
k_coarse_dense(int n, const double* __restrict__ Cu, const double* __restrict__ Gpu,
               const double* __restrict__ Cp, const uint8_t* __restrict__ cmask,
               const double* __restrict__ r, double* __restrict__ z) {
    __shared__ double rs[3 * CD_NMAX], zu[2 * CD_NMAX], t[CD_NMAX], zp[CD_NMAX];
    for (int k = threadIdx.x; k < 3 * n; k += CD_THREADS) rs[k] = r[k];
    __syncthreads();
    matvec(2 * n, 2 * n, Cu, rs, nullptr, -1.0, zu);          // z_u = C_u r_u
    __syncthreads();
    matvec(n, 2 * n, Gpu, zu, rs + 2 * n, 1.0, t);             // t = r_phi - G_phiu z_u
    __syncthreads();
    matvec(n, n, Cp, t, nullptr, -1.0, zp);                    // z_phi = C_phi t
    __syncthreads();
    for (int k = threadIdx.x; k < 3 * n; k += CD_THREADS) {
        const double v = k < 2 * n ? zu[k] : zp[k - 2 * n];
        z[k] = cmask[k] ? rs[k] : v;                           // constrained rows copy r
    }
}

// y = M x, M row-major (rows x cols), one warp per row, lane-strided columns
// and a fixed shuffle tree (deterministic); M stays L2-resident across calls
__global__ void __launch_bounds__(256)
k_dense_matvec(int rows, int cols, const double* __restrict__ M, const double* __restrict__ x,
               double* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (row >= rows) return;
    const double* mr = M + (int64_t)row * cols;
    double acc = 0.0;
    for (int j = lane; j < cols; j += 32) acc = fma(mr[j], x[j], acc);
    acc = warp_sum(acc);
    if (lane == 0) y[row] = acc;
}

}  // namespace

int coarse_dense_nmax() { return CD_NMAX; }

cudaError_t launch_dense_matvec(int rows, int cols, const double* M, const double* x, double* y,
                                cudaStream_t s) {
    if (rows < 1 || cols < 1) return cudaErrorInvalidValue;
    k_dense_matvec<<<(rows + 7) / 8, 256, 0, s>>>(rows, cols, M, x, y);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_coarse_dense(int n, const double* Cu, const double* Gpu, const double* Cp,
                                const uint8_t* cmask, const double* r, double* z,
                                cudaStream_t s) {
    if (n < 1 || n > CD_NMAX) return cudaErrorInvalidValue;
    k_coarse_dense<<<1, CD_THREADS, 0, s>>>(n, Cu, Gpu, Cp, cmask, r, z);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace pff
