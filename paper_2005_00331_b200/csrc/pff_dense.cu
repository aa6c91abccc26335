// pff_dense.cu -- small dense fp64 linear algebra for the multigrid setup:
// the masked dense Jacobian of a coarse level, GEMM, and row-scaled updates.
//
// The GMG setup composes the coarse solve and the level-3 V-cycle as dense
// maps (multigrid.py _build_dense_coarse / _build_dense_level: the reference's
// coarse Chebyshev passes and the V-cycle from level 3 down, src/multigrid.py:
// 311-344, are fixed linear maps for a fixed setup).  These kernels build them
// without a library GEMM, sparse assembly or framework elementwise kernels.
// Matrices are row-major.  fp64 has no tcgen05 kind on B200 and its DMMA rate
// equals the DFMA rate, so the GEMM is a shared-memory-tiled DFMA kernel; the
// matrices are <= ~900^2 (L2-resident).
#include "pff_internal.cuh"

namespace pff {

namespace {

// Masked dense Jacobian G (3n x 3n) of a whole-mesh level from its cell
// matrices gk[cell][3 NL][3 NL] (pff_cell_matrices): one thread per entry
// (r, c) sums the cells containing both nodes in increasing cell index;
// constrained rows/columns are identity (src/pff_operator.py:343-377).
template <int P>
__global__ void k_dense_jacobian(Mesh m, const double* __restrict__ gk,
                                 const uint8_t* __restrict__ flags, double* __restrict__ G) {
    constexpr int N1 = P + 1, NL = N1 * N1, NC = 3 * NL;
    const int64_t n = m.n, N = 3 * n;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N * N) return;
    const int64_t r = t / N, c = t - r * N;
    const int cr = (int)(r / n), cc = (int)(c / n);
    const int64_t gr = r - cr * n, gc = c - cc * n;
    const uint8_t fr = flags[gr], fc = flags[gc];
    const bool cons_r = cr < 2 ? (fr & F_DIR) : (fr & F_ACT);
    const bool cons_c = cc < 2 ? (fc & F_DIR) : (fc & F_ACT);
    if (cons_r || cons_c) {
        G[t] = r == c ? 1.0 : 0.0;
        return;
    }
    double acc = 0.0;
    node_cells(m, gr, 0, m.nside, [&](int cx, int cy, int a, int b) {
        const int64_t cell = (int64_t)cy * m.nside + cx;
#pragma unroll 1
        for (int bc = 0; bc < N1; ++bc)
            for (int ac = 0; ac < N1; ++ac)
                if (m.node(cx, cy, ac, bc) == gc)
                    acc += gk[(cell * NC + cr * NL + b * N1 + a) * NC + cc * NL + bc * N1 + ac];
    });
    G[t] = acc;
}

// C = alpha A B + beta C (row-major; A m x k, B k x n): GT x GT tiles per
// 256-thread block, k in steps of 16 through shared memory.  beta == 0 ignores
// C's previous contents.
// Tile GT x GT (64: 4 x 4 outputs per thread; 32: 2 x 2 -- the small matrices of
// the coarse maps, where 64-wide tiles leave a handful of blocks with long
// serial chains).  Every output sums over k in increasing order: the tile size
// does not change a bit of the result.
constexpr int GK = 16;
template <int GT>
__global__ void __launch_bounds__(256)
k_dgemm(int m, int n, int k, double alpha, const double* __restrict__ A, int lda,
        const double* __restrict__ B, int ldb, double beta, double* __restrict__ C, int ldc) {
    constexpr int TO = GT / 16;   // outputs per thread and dimension
    __shared__ double As[GK][GT + 1];
    __shared__ double Bs[GK][GT + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int row0 = blockIdx.y * GT, col0 = blockIdx.x * GT;
    double acc[TO][TO] = {};
    for (int k0 = 0; k0 < k; k0 += GK) {
        for (int e = threadIdx.x; e < GT * GK; e += 256) {
            const int i = e / GK, kk = e - i * GK;          // A tile: rows i, cols kk
            const int gi = row0 + i, gk = k0 + kk;
            As[kk][i] = (gi < m && gk < k) ? A[(int64_t)gi * lda + gk] : 0.0;
            const int kb = e / GT, j = e - kb * GT;          // B tile: rows kb, cols j
            const int gkb = k0 + kb, gj = col0 + j;
            Bs[kb][j] = (gkb < k && gj < n) ? B[(int64_t)gkb * ldb + gj] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < GK; ++kk) {
            double a[TO], b[TO];
#pragma unroll
            for (int u = 0; u < TO; ++u) {
                a[u] = As[kk][ty * TO + u];
                b[u] = Bs[kk][tx * TO + u];
            }
#pragma unroll
            for (int u = 0; u < TO; ++u)
#pragma unroll
                for (int v = 0; v < TO; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < TO; ++u) {
        const int gi = row0 + ty * TO + u;
        if (gi >= m) continue;
#pragma unroll
        for (int v = 0; v < TO; ++v) {
            const int gj = col0 + tx * TO + v;
            if (gj >= n) continue;
            double* cp = C + (int64_t)gi * ldc + gj;
            *cp = beta == 0.0 ? alpha * acc[u][v] : fma(alpha, acc[u][v], beta * *cp);
        }
    }
}

// Y = a Y + b diag(s) X  (s == nullptr: the identity; a == 0: Y overwritten)
__global__ void k_dmat_axpby(int m, int n, double a, double* Y, int ldy, double b,
                             const double* __restrict__ s, const double* X, int ldx) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)m * n) return;
    const int i = (int)(t / n), j = (int)(t - (int64_t)i * n);
    const double x = (s ? s[i] : 1.0) * X[(int64_t)i * ldx + j];
    double* y = Y + (int64_t)i * ldy + j;
    *y = a == 0.0 ? b * x : fma(a, *y, b * x);
}

// Y = diag(s)  (s == nullptr: the identity)
__global__ void k_dmat_diag(int n, const double* __restrict__ s, double* Y, int ldy) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)n * n) return;
    const int i = (int)(t / n), j = (int)(t - (int64_t)i * n);
    Y[(int64_t)i * ldy + j] = i == j ? (s ? s[i] : 1.0) : 0.0;
}

// y = 1 / x (mode 0) or 1 / sqrt(x) (mode 1): the inverse block diagonals of
// the smoother and the D^-1/2 scaling of the Lanczos runs
__global__ void k_recip(int64_t n, const double* __restrict__ x, double* __restrict__ y, int mode) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    y[i] = mode ? 1.0 / sqrt(x[i]) : 1.0 / x[i];
}

// constraint flags <-> masks (mode 0: flags = dir | act << 1; mode 1: unpack)
__global__ void k_flags(int64_t n, uint8_t* dir, uint8_t* act, uint8_t* flags, int mode) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (mode == 0) {
        flags[i] = (uint8_t)((dir[i] ? F_DIR : 0) | (act[i] ? F_ACT : 0));
    } else {
        const uint8_t f = flags[i];
        dir[i] = (f & F_DIR) ? 1 : 0;
        act[i] = (f & F_ACT) ? 1 : 0;
    }
}

inline unsigned blocks256(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

cudaError_t launch_dense_jacobian(const Level& L, const double* gk, double* G, cudaStream_t s) {
    if (L.windowed() || !L.flags) return cudaErrorInvalidValue;
    const int64_t N = 3 * L.mesh.n;
    const unsigned g = blocks256(N * N);
    switch (L.mesh.p) {
        case 1: k_dense_jacobian<1><<<g, 256, 0, s>>>(L.mesh, gk, L.flags, G); break;
        case 2: k_dense_jacobian<2><<<g, 256, 0, s>>>(L.mesh, gk, L.flags, G); break;
        case 3: k_dense_jacobian<3><<<g, 256, 0, s>>>(L.mesh, gk, L.flags, G); break;
        case 4: k_dense_jacobian<4><<<g, 256, 0, s>>>(L.mesh, gk, L.flags, G); break;
        default: return cudaErrorInvalidValue;
    }
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_dgemm(int m, int n, int k, double alpha, const double* A, int lda, const double* B,
                         int ldb, double beta, double* C, int ldc, cudaStream_t s) {
    if (m <= 0 || n <= 0) return cudaSuccess;
    // fewer than half a wave of 64-wide tiles: the 32-wide form (four times the blocks)
    if ((int64_t)((n + 63) / 64) * ((m + 63) / 64) < 64) {
        dim3 grid((n + 31) / 32, (m + 31) / 32);
        k_dgemm<32><<<grid, 256, 0, s>>>(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
    } else {
        dim3 grid((n + 63) / 64, (m + 63) / 64);
        k_dgemm<64><<<grid, 256, 0, s>>>(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
    }
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_dmat_axpby(int m, int n, double a, double* Y, int ldy, double b, const double* sv,
                              const double* X, int ldx, cudaStream_t s) {
    if (m <= 0 || n <= 0) return cudaSuccess;
    k_dmat_axpby<<<blocks256((int64_t)m * n), 256, 0, s>>>(m, n, a, Y, ldy, b, sv, X, ldx);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_dmat_diag(int n, const double* sv, double* Y, int ldy, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    k_dmat_diag<<<blocks256((int64_t)n * n), 256, 0, s>>>(n, sv, Y, ldy);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_recip(int64_t n, const double* x, double* y, int mode, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    k_recip<<<blocks256(n), 256, 0, s>>>(n, x, y, mode);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_flags(int64_t n, uint8_t* dir, uint8_t* act, uint8_t* flags, int mode, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    k_flags<<<blocks256(n), 256, 0, s>>>(n, dir, act, flags, mode);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace pff
