// pff_internal.cuh -- host-side launch interface shared by the .cu files.
#pragma once
#include "pff_common.cuh"

namespace pff {

// kernels (and memsets) enqueued by this library; see pff_launch_counter()
void count_launches(int k);

// Local window of a level as seen by the generic (any-degree) kernels: cells
// of rows [row0, row0 + ncell/nside); global node id g lives at local index
// g - shift (grid rows) or dupl + (g - n_grid) (slit copies); n = local length.
struct Win {
    int row0;
    int64_t ncell, shift, dupl, n;
    int64_t own_lo, own_hi;   // owned node rows
    int owns_dup;
    __host__ __device__ __forceinline__ int64_t loc(const Mesh& m, int64_t g) const {
        return g >= m.n_grid ? dupl + (g - m.n_grid) : g - shift;
    }
    // t-th owned node (grid rows first, then the slit copies) -> global id
    __host__ __device__ __forceinline__ int64_t owned_global(const Mesh& m, int64_t t) const {
        const int64_t cnt = (own_hi - own_lo) * m.np1;
        return t < cnt ? own_lo * m.np1 + t : m.n_grid + (t - cnt);
    }
    __host__ __device__ __forceinline__ int64_t n_owned(const Mesh& m) const {
        return (own_hi - own_lo) * m.np1 + (owns_dup ? m.n_dup : 0);
    }
};

// smallest mesh (cells per side) on the Q2 sweep kernel (PFF_SWEEP_MIN_NSIDE);
// below it the generic cooperative kernel runs (pff_sweep.cu)
int sweep_min_nside();
void set_sweep_min_nside(int nside);

// Per-level handle contents (the C-ABI's opaque pff_level).
struct Level {
    Mesh mesh;
    Shape shape;
    Embed embed;       // coarse basis at this level's child support points
    Material mat;
    int miehe;
    // bound linearisation point (device pointers owned by the caller)
    const double* U = nullptr;          // 3n: u0x | u0y | phi0
    const double* phi_tilde = nullptr;  // n
    const uint8_t* flags = nullptr;     // n: F_DIR | F_ACT
    double* qcache = nullptr;           // qcache_len() doubles

    // Slab window (multi-GPU): this handle owns cell rows
    // [win_begin, win_end) of the global mesh and holds LOCAL arrays with node
    // rows [j_lo, j_hi] (p ghost rows below, 1 above) followed by the upper slit
    // copies when row i_mid lies in that range.  win_end < 0: whole mesh.
    int win_begin = 0, win_end = -1;
    bool windowed() const { return win_end >= 0; }
    int cy_begin() const { return windowed() ? win_begin : 0; }
    int cy_end() const { return windowed() ? win_end : mesh.nside; }
    int q_row0() const { return cy_begin() > 0 ? cy_begin() - 1 : 0; }   // first computed cell row
    int q_rows() const { return cy_end() - q_row0(); }
    int64_t j_lo() const { return (int64_t)mesh.p * q_row0(); }
    int64_t j_hi() const { return (int64_t)mesh.p * cy_end(); }
    bool local_dup() const { return mesh.n_dup > 0 && mesh.i_mid >= j_lo() && mesh.i_mid <= j_hi(); }
    int64_t local_n() const {
        return windowed() ? (j_hi() - j_lo() + 1) * mesh.np1 + (local_dup() ? mesh.n_dup : 0) : mesh.n;
    }
    // offset of the slit copies relative to the row-shifted base (base - j_lo*np1)
    int64_t dupoff() const { return windowed() ? (j_hi() + 1) * mesh.np1 : mesh.n_grid; }
    int64_t row_shift() const { return windowed() ? j_lo() * mesh.np1 : 0; }

    // owned node rows [own_lo, own_hi) and slit copies
    int64_t own_lo() const { return (int64_t)mesh.p * cy_begin(); }
    int64_t own_hi() const {
        return (int64_t)mesh.p * cy_end() + (cy_end() == mesh.nside ? 1 : 0);
    }
    bool owns_dup() const { return mesh.n_dup > 0 && mesh.i_mid >= own_lo() && mesh.i_mid < own_hi(); }
    // cell window of the generic kernels: cells of rows [q_row0, cy_end)
    int64_t local_cells() const { return (int64_t)q_rows() * mesh.nside; }
    Win win() const {
        Win w;
        w.row0 = q_row0();
        w.ncell = local_cells();
        w.shift = row_shift();
        w.dupl = dupoff() - row_shift();
        w.n = local_n();
        w.own_lo = own_lo();
        w.own_hi = own_hi();
        w.owns_dup = owns_dup() ? 1 : 0;
        return w;
    }

    // generic q-point cache (layout [field][k][cell], 6 fields) over the window's cells
    int64_t generic_len() const { return 6 * (int64_t)(mesh.p + 1) * (mesh.p + 1) * local_cells(); }
    // Q2 strip-tiled q-point cache of the sweep kernel (pff_sweep.cu): per
    // (strip of 31 cells + 1 halo, cell row) one block [iq][array][jq][lane]
    bool q2_struct = false;   // N[1] = (0,1,0), D[1] = (-1,0,1) at the middle Gauss point
    int min_nside = 64;       // sweep_min_nside() when the level was created (fixes its layout)
    bool sweep_ok() const {   // the sweep kernel stages with 32-bit node indices
        return mesh.p == 2 && mesh.nside >= min_nside && q2_struct &&
               mesh.n < (int64_t(1) << 31);
    }
    int n_strips() const { return (mesh.nside + 30) / 31; }
    // Miehe: +-g, +-gamma, cos/sin 2 theta, 2 eigen-frame coupling coefficients, pc;
    // none: g w, coupling (3), pc
    int tile_nq() const { return miehe ? 7 : 5; }
    int tile4_nq() const { return miehe ? 7 : 5; }   // Q4: the same arrays
    int64_t tile_block() const { return (int64_t)tile_nq() * 9 * 32; }
    int64_t tile_len() const { return sweep_ok() ? (int64_t)n_strips() * q_rows() * tile_block() : 0; }
    // element-vector scratch of the generic application and of the restriction
    // into this level: [component][cell][local node], 3 x cells x (p+1)^2
    int64_t ev_len() const { return 3 * (int64_t)(mesh.p + 1) * (mesh.p + 1) * local_cells(); }
    // weighted tangent cache of the generic application (Miehe levels without
    // the sweep kernel), in warp groups of gtan_group() cells (the cooperative
    // kernel's cells per warp): [group][array T00 T01 T02 T11 T12 T22 cw0 cw1 cw2
    // pc][jq][cell in group][iq] -- a warp's load for one (array, jq) is one
    // contiguous run over its (cell, iq) lanes
    // (none: [g w][cw0 cw1 cw2][pc], 5 arrays)
    int gtan_group() const { return 32 / (mesh.p + 1); }
    int gtan_arrays() const { return miehe ? 10 : 5; }
    int64_t gtan_len() const {
        const int64_t cg = gtan_group();
        const int64_t cells = (local_cells() + cg - 1) / cg * cg;
        return !sweep_ok() ? gtan_arrays() * (int64_t)(mesh.p + 1) * (mesh.p + 1) * cells : 0;
    }
    // Q4 sweep kernel (pff_sweep4.cu): strips of 6 cells (5 own + the left
    // neighbour), per (strip, cell row) one tangent block [array][jq][cell][iq]
    bool q4_struct = false;   // mirror-symmetric 5-point basis (even-odd contractions)
    bool sweep4_ok() const {
        return mesh.p == 4 && !windowed() && mesh.nside >= min_nside && q4_struct &&
               mesh.n < (int64_t(1) << 31);
    }
    int n_strips4() const { return (mesh.nside + 4) / 5; }
    int64_t tile4_block() const { return (int64_t)tile4_nq() * 25 * 6; }
    int64_t tile4_len() const { return sweep4_ok() ? (int64_t)n_strips4() * mesh.nside * tile4_block() : 0; }
    int64_t qcache_len() const {
        return generic_len() + tile_len() + gtan_len() + ev_len() + tile4_len();
    }
    double* qtile4() const { return ev() + ev_len(); }
    double* qtile() const { return qcache + generic_len(); }
    double* gtan() const { return qcache + generic_len() + tile_len(); }
    double* ev() const { return qcache + generic_len() + tile_len() + gtan_len(); }
};

// Cells containing scalar node g (global id) in increasing cell index, with
// the node's local (a, b) in each; cells of rows outside [row_lo, row_hi) are
// skipped.  The slit copies: the grid id of a slit node belongs to the lower
// cell row only, the appended copy n_grid + i to the upper one.
template <class F>
__device__ __forceinline__ void node_cells(const Mesh& m, int64_t g, int row_lo, int row_hi,
                                           F&& f) {
    const int p = m.p, ns = m.nside;
    int64_t i, j;
    int cy_lo = row_lo, cy_hi = row_hi < ns ? row_hi : ns;
    if (g < m.n_grid) {
        j = g / m.np1;
        i = g - j * m.np1;
        if (m.level >= 1 && j == m.i_mid && i < m.i_mid && cy_hi > (ns >> 1)) cy_hi = ns >> 1;
    } else {
        i = g - m.n_grid;
        j = m.i_mid;
        if (cy_lo < (ns >> 1)) cy_lo = ns >> 1;
    }
    const int cy0 = j > 0 ? (int)((j - 1) / p) : 0, cy1 = (int)(j / p);
    const int cx0 = i > 0 ? (int)((i - 1) / p) : 0, cx1 = (int)(i / p);
    for (int cy = cy0; cy <= cy1; ++cy) {
        if (cy < cy_lo || cy >= cy_hi) continue;
        const int b = (int)(j - (int64_t)cy * p);
        if (b < 0 || b > p) continue;
        for (int cx = cx0; cx <= cx1 && cx < ns; ++cx) {
            const int a = (int)(i - (int64_t)cx * p);
            if (a < 0 || a > p) continue;
            f(cx, cy, a, b);
        }
    }
}

// node_cells with the degree P at compile time and 32-bit index math (levels
// with fewer than 2^31 nodes): no 64-bit divisions -- the per-node gathers
// are instruction-bound on those.  Same cells, same order.
template <int P, class F>
__device__ __forceinline__ void node_cells_p(const Mesh& m, int64_t g, int row_lo, int row_hi,
                                             F&& f) {
    if (m.n >= (int64_t(1) << 31)) {
        node_cells(m, g, row_lo, row_hi, f);
        return;
    }
    const int ns = m.nside, np1 = (int)m.np1, imid = (int)m.i_mid;
    const int g32 = (int)g, ngrid = (int)m.n_grid;
    int i, j;
    int cy_lo = row_lo, cy_hi = row_hi < ns ? row_hi : ns;
    if (g32 < ngrid) {
        j = (int)((unsigned)g32 / (unsigned)np1);
        i = g32 - j * np1;
        if (m.level >= 1 && j == imid && i < imid && cy_hi > (ns >> 1)) cy_hi = ns >> 1;
    } else {
        i = g32 - ngrid;
        j = imid;
        if (cy_lo < (ns >> 1)) cy_lo = ns >> 1;
    }
    // at most two cell rows and columns, visited in increasing cell index (the
    // same cells and order as node_cells), unrolled
    const int cy0 = j > 0 ? (j - 1) / P : 0, cy1 = j / P;
    const int cx0 = i > 0 ? (i - 1) / P : 0, cx1 = i / P;
#pragma unroll
    for (int ry = 0; ry < 2; ++ry) {
        const int cy = ry ? cy1 : cy0;
        if ((ry && cy1 == cy0) || cy < cy_lo || cy >= cy_hi) continue;
        const int b = j - cy * P;
#pragma unroll
        for (int rx = 0; rx < 2; ++rx) {
            const int cx = rx ? cx1 : cx0;
            if ((rx && cx1 == cx0) || cx >= ns) continue;
            f(cx, cy, i - cx * P, b);
        }
    }
}

// a Chebyshev step fused into a block application (pff_apply_cheb): after
// cr = cr - G d, d_out = c1 d + c2 invd cr and acc += d_out, per component
struct ChebArgs {
    const double* invd;
    double* dout;
    double* acc;
    double c1, c2;
    // acc_src: acc += d + d' (the first step after a producer emitted d0 = d;
    // (acc + d) + d' rounds exactly like the separate pff_cheb_init pass)
    int acc_src = 0;
    // last: the final step of a pass -- only acc is consumed, so the residual
    // (dst) and d' (dout) stores are skipped
    int last = 0;
    // noacc: the step leaves acc alone (the next step adds both, acc_src)
    int noacc = 0;
    // residual producers (fused form, no dout): d0 = invd * dst / theta on the
    // first emit_nc output components (pff_cheb_init's d, same rounding)
    double* emit = nullptr;
    double theta = 1.0;
    int emit_nc = 0;
};

// small dense algebra of the GMG setup (pff_dense.cu)
cudaError_t launch_dense_jacobian(const Level& L, const double* gk, double* G, cudaStream_t s);
cudaError_t launch_dgemm(int m, int n, int k, double alpha, const double* A, int lda, const double* B,
                         int ldb, double beta, double* C, int ldc, cudaStream_t s);
cudaError_t launch_dmat_axpby(int m, int n, double a, double* Y, int ldy, double b, const double* sv,
                              const double* X, int ldx, cudaStream_t s);
cudaError_t launch_dmat_diag(int n, const double* sv, double* Y, int ldy, cudaStream_t s);
cudaError_t launch_recip(int64_t n, const double* x, double* y, int mode, cudaStream_t s);
cudaError_t launch_flags(int64_t n, uint8_t* dir, uint8_t* act, uint8_t* flags, int mode, cudaStream_t s);

// options (pff_set_option)
void set_generic_apply(bool on);
void set_sweep_rows_per_chunk(int rows);
void set_sweep_colring(int mode);   // -1 auto (env / measured default), 0 row stages, 1 column ring

// Q2 sweep kernel (pff_sweep.cu)
cudaError_t launch_refresh_tiled(const Level& L, cudaStream_t s);
// Q4 sweep kernel (pff_sweep4.cu)
cudaError_t launch_refresh_tile4(const Level& L, cudaStream_t s);
cudaError_t launch_sweep4_apply(const Level& L, int mode, const double* src, double* dst,
                                const double* rhs, cudaStream_t s, bool* handled);
cudaError_t launch_sweep_apply(const Level& L, int mode, const double* src, double* dst,
                               const double* rhs, cudaStream_t s, bool* handled,
                               const ChebArgs* cheb = nullptr);
cudaError_t launch_sweep_apply_rows(const Level& L, int mode, const double* src, double* dst,
                                    const double* rhs, int cy_begin, int cy_end, cudaStream_t s,
                                    bool* handled, const ChebArgs* cheb = nullptr);

// operator family (pff_ops.cu)
cudaError_t launch_refresh(const Level& L, cudaStream_t s);
cudaError_t launch_apply(const Level& L, int mode, const double* src, double* dst,
                         const double* rhs, cudaStream_t s, const ChebArgs* cheb = nullptr);
cudaError_t launch_diagonal(const Level& L, double* dx, double* dy, double* dp, int invert,
                            cudaStream_t s);
cudaError_t launch_residual(const Level& L, double* out, int mask_dirichlet, int mask_active,
                            cudaStream_t s);

// coarse-level solve as dense linear maps (pff_coarse.cu)
int coarse_dense_nmax();
cudaError_t launch_coarse_dense(int n, const double* Cu, const double* Gpu, const double* Cp,
                                const uint8_t* cmask, const double* r, double* z,
                                cudaStream_t s);

cudaError_t launch_dense_matvec(int rows, int cols, const double* M, const double* x, double* y,
                                cudaStream_t s);

// dense per-cell matrices (pff_assemble.cu)
cudaError_t launch_cell_matrices(const Level& L, double* gk, cudaStream_t s);

// active-set loop (pff_active.cu)
cudaError_t launch_lumped_mass(const Level& L, double* out, cudaStream_t s);
cudaError_t launch_active_set(int64_t n, const double* rhs_phi, double* phi,
                              const double* phi_old, const double* m_diag, double c,
                              const uint8_t* prev, uint8_t* active, unsigned long long* stats,
                              cudaStream_t s);

// transfers (pff_transfer.cu)
cudaError_t launch_prolongate(const Level& fine, const Level& coarse, const double* xc,
                              double* yf, int add_masked, cudaStream_t s);
cudaError_t launch_restrict(const Level& fine, const Level& coarse, const double* yf,
                            double* xc, int zero_cons, cudaStream_t s);
cudaError_t launch_inject_f64(const Level& fine, const Level& coarse, const double* src,
                              double* dst, int ncomp, cudaStream_t s);
cudaError_t launch_inject_u8(const Level& fine, const Level& coarse, const uint8_t* src,
                             uint8_t* dst, cudaStream_t s);

// vectors (pff_vec.cu)
constexpr int RED_BLOCKS = 592;   // 4 x 148 SMs: fixed, so reductions are deterministic
constexpr int RED_THREADS = 256;
cudaError_t launch_cons(const Level& L, int layout, int op, const double* r, double* z,
                        cudaStream_t s);
cudaError_t launch_smooth_init(const Level& L, const double* r, double* z, double* res_u,
                               const double* invd_u, double* d_u, double theta, bool add_d0,
                               cudaStream_t s);
cudaError_t launch_cheb_init(int64_t n, const double* invd, const double* rhs, double theta,
                             double* d, double* acc, int acc_mode, cudaStream_t s);
cudaError_t launch_cheb_step(int64_t n, const double* invd, const double* r, double c1,
                             double c2, double* d, double* acc, cudaStream_t s);
cudaError_t launch_axpby(int64_t n, double a, const double* x, double b, double* y,
                         cudaStream_t s);
cudaError_t launch_div(int64_t n, const double* x, const double* sdev, double sval, double* y,
                       cudaStream_t s);
cudaError_t launch_dot(int64_t n, const double* x, const double* y, double* partials,
                       double* out, cudaStream_t s);
cudaError_t launch_mgs(int64_t n, int j, const double* V, int64_t ldv, double* w,
                       double* partials, double* h, cudaStream_t s);
cudaError_t launch_lsmgs(int64_t n, int j, const double* V, int64_t ldv, double* w,
                         double* gram, int64_t ldg, double* partials, double* h, cudaStream_t s);
cudaError_t launch_mdot(int64_t n, int k, const double* V, int64_t ldv, const double* w,
                        double* partials, double* out, cudaStream_t s);
cudaError_t launch_combine(int64_t n, int k, const double* V, int64_t ldv, const double* y,
                           double* out, int accumulate, cudaStream_t s);
cudaError_t launch_lanczos_scale(int64_t n, const double* dhalf, const double* v, double* out,
                                 cudaStream_t s);

// batched Lanczos range estimates (pff_lanczos.cu)
cudaError_t lanczos_ranges(int nruns, const Level* const* levels, const int* modes,
                           const int64_t* ns, const double* const* dhalf, double* const* work,
                           int max_it, double* lo_hi, double* partials, double* dots,
                           cudaStream_t s);

}  // namespace pff
