/*
 * pff_b200.h -- C ABI of libpff_b200.so, the B200 (sm_100a) implementation
 * of the matrix-free phase-field-fracture hot path of fracturekit 0.1.0
 * (arXiv 2005.00331).  `src/` below is /root/reference/pkg/src/fracturekit/.
 *
 * Conventions
 *  - Every entry point returns 0 on success, a cudaError_t value (> 0) for a
 *    CUDA failure or a negative PFF_E* code; it never throws or aborts.
 *    pff_last_error() gives a message for the calling thread.
 *  - All vector pointers are DEVICE pointers (fp64 unless stated), laid out
 *    exactly as the reference's numpy vectors: component-major
 *    [u_x | u_y | phi], each n_scalar long, grid node (i, j) at j*(p*2^l+1)+i,
 *    upper slit copies appended (src/mesh_hierarchy.py:156-189).
 *  - The caller owns all device memory.  A pff_level owns only its tables.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Every call is
 *    asynchronous on that stream and CUDA-graph capturable; none synchronises.
 *  - src and dst of one call must not alias; dst may alias rhs.
 */
#ifndef PFF_B200_H
#define PFF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PFF_ABI_VERSION 1

enum { PFF_E_ARG = -1, PFF_E_STATE = -2, PFF_E_UNBOUND = -3 };

/* operator modes (src/pff_operator.py:262-302) */
enum {
    PFF_MODE_FULL = 0,    /* apply_jacobian:     3n -> 3n */
    PFF_MODE_UU = 1,      /* apply_block_uu:     2n -> 2n */
    PFF_MODE_PHIPHI = 2,  /* apply_block_phiphi:  n ->  n */
    PFF_MODE_PHIROW = 3   /* apply_phi_row:      3n ->  n */
};

/* constraint flag bits, one byte per scalar node (constrained_mask(),
 * src/pff_operator.py:148-150) */
enum { PFF_FLAG_DIRICHLET = 1, PFF_FLAG_ACTIVE = 2 };

/* vector layouts for the masking helpers */
enum { PFF_LAYOUT_FULL = 0, PFF_LAYOUT_UU = 1, PFF_LAYOUT_PHI = 2 };
/* SELECT: z = cons ? r : 0;  ZERO: z[cons] = 0;  COPY: z[cons] = r[cons];
 * EXCLUDE: z = cons ? 0 : r  (= r - G z0 for z0 = SELECT(r): the first smoother
 * residual of a V-cycle level, without an operator application) */
enum { PFF_CONS_SELECT = 0, PFF_CONS_ZERO = 1, PFF_CONS_COPY = 2, PFF_CONS_EXCLUDE = 3 };

/* MaterialParams, src/material_model.py:20-44 */
typedef struct {
    double lame_lambda, mu, g_c, kappa, eps;
} pff_material;

typedef struct pff_level pff_level;

int pff_abi_version(void);
const char* pff_last_error(void);

/* number of kernels (and memsets) this library has enqueued so far; the
 * benchmark reads it around its timed region */
int64_t pff_launch_counter(void);

/* tuning / testing knobs (process-wide):
 *   PFF_OPT_GENERIC_APPLY: 1 = route pff_apply through the generic per-cell
 *     atomic kernel for every degree (the Q2 sweep kernel is the default)
 *   PFF_OPT_SWEEP_ROWS: cell rows per warp chunk of the Q2 sweep (0 = auto)
 *   PFF_OPT_SWEEP_MIN_NSIDE: smallest Q2 mesh (cells per side) on the sweep
 *     kernel for levels created AFTER the call (a level keeps the layout it was
 *     created with); 0 = PFF_SWEEP_MIN_NSIDE or the default 64, minimum 4 */
/*   PFF_OPT_SWEEP_COLRING: staging of the Q2 sweep's tangent block: 1 = the
 *     single-buffered Gauss-column ring, 0 = two whole-row stages, -1 = the
 *     measured per-mode default (the results are bitwise the same either way) */
enum { PFF_OPT_GENERIC_APPLY = 1, PFF_OPT_SWEEP_ROWS = 2, PFF_OPT_SWEEP_MIN_NSIDE = 3,
       PFF_OPT_SWEEP_COLRING = 4 };
int pff_set_option(int key, int value);

/* One mesh level (replaces DofMap + LinearizationState's static data,
 * src/pff_operator.py:74-101).  N, D: host (p+1)x(p+1) row-major shape
 * values/derivatives at the Gauss points, w: (p+1) weights
 * (src/tensor_basis.py:66-81); embed: host 2x(p+1)x(p+1) coarse basis at
 * the child support points (src/multigrid.py:58-61).  split: 0 none, 1 miehe. */
int pff_level_create(pff_level** out, int degree, int level, int split,
                     const pff_material* mat, const double* N, const double* D,
                     const double* w, const double* embed);
int pff_level_destroy(pff_level* L);
int64_t pff_level_n_scalar(const pff_level* L);
int64_t pff_level_n_cells(const pff_level* L);
int64_t pff_level_qcache_len(const pff_level* L);
/* 1 when the level's applications run the Q2 sweep kernel (fixed at creation,
 * PFF_OPT_SWEEP_MIN_NSIDE), 0 for the generic cooperative kernel, -1 on NULL */
int pff_level_uses_sweep(const pff_level* L);

/* Slab window for multi-GPU runs: the handle then owns cell
 * rows [cy_begin, cy_end) of the global mesh and every array bound to it or
 * passed to pff_apply is LOCAL: node rows [j_lo, j_hi] = [p*max(cy_begin-1,0),
 * p*cy_end] (p ghost rows below, one above), x fastest, followed by the n_dup
 * upper slit copies when row i_mid lies in that range; pff_level_n_scalar()
 * returns that local length.  pff_apply writes only the owned node rows
 * [p*cy_begin, p*cy_end) (plus row p*2^l for the top slab, and the slit copies
 * on the slab owning row i_mid).  Q2 and >= 64x64 cells only; (0, 2^l) resets.
 * pff_level_window: rows = {j_lo, j_hi, has_slit_copies, local index of the
 * first slit copy, cy_begin, cy_end}. */
int pff_level_set_window(pff_level* L, int cy_begin, int cy_end);
int pff_level_window(const pff_level* L, int64_t* rows);

/* Bind the linearisation point: U (3n), phi_tilde (n), flags (n bytes, readable
 * for 16 bytes past the end: the sweeps stage them in aligned units) and a
 * caller-allocated q-point cache of pff_level_qcache_len() doubles (q-point
 * state, the Q2 tangent tiles, and the element-vector scratch that the generic
 * application and the restriction INTO this level use -- so a level's
 * applications and restrictions into it must be ordered, e.g. one stream). */
int pff_level_bind(pff_level* L, const double* U, const double* phi_tilde,
                   const uint8_t* flags, double* qcache);

/* LinearizationState.refresh_cache -> cache_kernel (src/pff_operator.py:154-184) */
int pff_level_refresh(pff_level* L, void* stream);

/* Jacobian family with identity rows/columns on constraints
 * (src/pff_operator.py:262-302 -> src/_kernels.py:555-693).
 * rhs == NULL: dst = G src.  rhs != NULL: dst = rhs - G src (fused residual,
 * e.g. `r - apply_jacobian(z)` of src/multigrid.py:298,336). */
int pff_apply(const pff_level* L, int mode, const double* src, double* dst,
              const double* rhs, void* stream);

/* pff_apply restricted to the owned cell rows [cy_begin, cy_end) of the
 * level: writes the node rows [p*cy_begin, p*cy_end) (plus the top row / the
 * slit copies when they fall in the range) and reads node rows
 * [p*(cy_begin-1), p*cy_end].  Lets a caller pipeline host<->device transfers
 * of row chunks with the computation.  Q2 sweep levels (>= 64x64 cells) only. */
int pff_apply_rows(const pff_level* L, int mode, const double* src, double* dst,
                   const double* rhs, int cy_begin, int cy_end, void* stream);

/* pff_apply from HOST buffers (the reference's operator takes host arrays,
 * src/pff_operator.py:262-302): xh (inputs of the mode, component-major as
 * pff_apply) -> yh, pipelined over cell-row chunks -- every H2D chunk queued
 * first on an internal copy stream, the row sweep of chunk k on `stream` once
 * its rows are resident, its D2H on a second copy stream -- so both PCIe
 * directions and the kernel overlap.  xd / yd are device work buffers of the
 * input / output size.  Asynchronous: ordered after the work already on
 * `stream`, and `stream` waits for the last copy, so synchronising `stream`
 * makes yh valid.  xh / yh should be page-locked for the overlap.
 * nchunks == 0: the default ramp of chunk sizes; 1..64: equal chunks.
 * Whole-mesh Q2 sweep levels (>= 64x64 cells) only. */
int pff_apply_host(const pff_level* L, int mode, const double* xh, double* yh, double* xd,
                   double* yd, int nchunks, void* stream);

/* block_diagonal (src/pff_operator.py:305-327 -> src/_kernels.py:700-746):
 * diag_uu (2n), diag_pp (n); constrained entries 1; invert != 0 stores 1/d. */
int pff_diagonal(const pff_level* L, double* diag_uu, double* diag_pp, int invert,
                 void* stream);

/* One Chebyshev smoothing step fused into the block application
 * (src/multigrid.py:186-195): cr = rhs - G d (mode PFF_MODE_UU or
 * PFF_MODE_PHIPHI, identity rows/columns as pff_apply; rhs may alias cr), then
 * d_out = c1 d + c2 invd .* cr and acc += d_out, per entry in the same pass.
 * d_out must not alias d.  Bitwise identical to pff_apply(mode, d, cr, rhs)
 * followed by pff_cheb_step. */
int pff_apply_cheb(const pff_level* L, int mode, const double* d, double* d_out,
                   const double* rhs, double* cr, const double* invd, double* acc, double c1,
                   double c2, void* stream);

/* residual (src/pff_operator.py:218-241 -> src/_kernels.py:319-440), 3n */
int pff_residual(const pff_level* L, double* out, int mask_dirichlet, int mask_active,
                 void* stream);

/* dense per-cell Jacobian matrices G_k (src/pff_operator.py:328-340 ->
 * src/_kernels.py:754-826) for the assembled comparison path: gk holds
 * n_cells x (3 (p+1)^2)^2 doubles, [cell][row][col], rows/cols ordered
 * (u_x | u_y | phi) x local node b*(p+1)+a.  Needs a refreshed state; whole
 * mesh only. */
int pff_cell_matrices(const pff_level* L, double* gk, void* stream);

/* Small dense fp64 algebra of the GMG setup (the coarse solve and the level-3
 * V-cycle as dense maps, src/multigrid.py:311-344 for a fixed setup).
 * Row-major matrices.
 * pff_dense_jacobian: G (3n x 3n) = the level's Jacobian assembled from its
 *   cell matrices gk (pff_cell_matrices), identity on constrained rows and
 *   columns (src/pff_operator.py:343-377); whole-mesh levels, 3n <= 8192.
 * pff_dgemm: C = alpha A B + beta C (A m x k, B k x n; beta = 0 overwrites).
 * pff_dmat_axpby: Y = a Y + b diag(s) X (s NULL: identity; a = 0 overwrites).
 * pff_dmat_diag: Y (n x n) = diag(s) (s NULL: identity).
 * pff_recip: y = 1/x (mode 0) or 1/sqrt(x) (mode 1).
 * pff_flags: mode 0 packs the Dirichlet / active byte masks into the level
 *   flags (bit0 | bit1), mode 1 unpacks them (src/pff_operator.py:
 *   constrained_mask). */
int pff_dense_jacobian(const pff_level* L, const double* gk, double* G, void* stream);
int pff_dgemm(int m, int n, int k, double alpha, const double* A, int lda, const double* B,
              int ldb, double beta, double* C, int ldc, void* stream);
int pff_dmat_axpby(int m, int n, double a, double* Y, int ldy, double b, const double* s,
                   const double* X, int ldx, void* stream);
int pff_dmat_diag(int n, const double* s, double* Y, int ldy, void* stream);
int pff_recip(int64_t n, const double* x, double* y, int mode, void* stream);
int pff_flags(int64_t n, uint8_t* dir, uint8_t* act, uint8_t* flags, int mode, void* stream);

/* lumped phi mass diagonal (src/active_set_solver.py:60-69 -> src/_kernels.py:828-843):
 * row sums of the scalar mass matrix over the level's local nodes; bitwise the
 * reference's summation order.  Needs no bound state. */
int pff_lumped_mass(const pff_level* L, double* out, void* stream);

/* one complementarity pass of the active-set loop (src/active_set_solver.py:72-82,
 * 113-118): active[i] = rhs_phi[i]/m[i] + c (phi[i] - phi_old[i]) > 0; freshly
 * activated dofs with phi != phi_old are reset to phi_old IN PLACE; stats (3
 * uint64, device) = {|A|, reset dofs, |A xor prev|} (prev may be NULL). */
int pff_active_set(int64_t n, const double* rhs_phi, double* phi, const double* phi_old,
                   const double* m_diag, double c, const uint8_t* prev, uint8_t* active,
                   uint64_t* stats, void* stream);

/* TransferOperator (src/multigrid.py:97-120) between fine = coarse + 1.
 * A windowed fine level (slab) transfers its OWNED fine nodes only: restrict
 * accumulates their P^T contributions into the whole-mesh coarse vector (sum
 * the ranks' partial coarse vectors with an all-reduce), prolongate fills /
 * updates its owned fine rows from a whole-mesh coarse vector.
 * prolongate: yf = P xc, or with add_masked: yf += where(cons_f, 0, P xc)
 * (src/multigrid.py:340-342).  restrict: xc = P^T yf, zero_cons: xc[cons_c]=0. */
int pff_prolongate(const pff_level* fine, const pff_level* coarse, const double* xc,
                   double* yf, int add_masked, void* stream);
int pff_restrict(const pff_level* fine, const pff_level* coarse, const double* yf,
                 double* xc, int zero_cons, void* stream);

/* MeshHierarchy.injection gathers (src/mesh_hierarchy.py:316-338), one level */
int pff_inject_f64(const pff_level* fine, const pff_level* coarse, const double* src,
                   double* dst, int ncomp, void* stream);
int pff_inject_u8(const pff_level* fine, const pff_level* coarse, const uint8_t* src,
                  uint8_t* dst, void* stream);

/* constraint masking on a level's vector (layout PFF_LAYOUT_*, op PFF_CONS_*) */
int pff_cons(const pff_level* L, int layout, int op, const double* r, double* z,
             void* stream);

/* chebyshev_apply pieces (src/multigrid.py:170-198):
 * init: d = invd*rhs/theta; acc_mode 0: acc = d, 1: acc += d, 2: untouched
 * step: d = c1*d + c2*(invd*r); acc += d */
int pff_cheb_init(int64_t n, const double* invd, const double* rhs, double theta,
                  double* d, double* acc, int acc_mode, void* stream);
int pff_cheb_step(int64_t n, const double* invd, const double* r, double c1, double c2,
                  double* d, double* acc, void* stream);

/* y = a x + b y;  y = x / s (s = *sdev if sdev else sval);  y = a .* x */
int pff_axpby(int64_t n, double a, const double* x, double b, double* y, void* stream);
int pff_div(int64_t n, const double* x, const double* sdev, double sval, double* y,
            void* stream);
int pff_mul(int64_t n, const double* a, const double* x, double* y, void* stream);

/* Lanczos range estimates of several block operators at once
 * (src/multigrid.py:123-162 for every level and block of GmgPreconditioner,
 * 259-275): run r applies mode modes[r] (PFF_MODE_UU or PFF_MODE_PHIPHI) of
 * levels[r] scaled by dhalf[r] = diag^-1/2 (ns[r] entries) for at most
 * max_iterations steps; work[r] holds 4 ns[r] doubles whose first ns[r] are the
 * start vector on entry.  The runs advance in lockstep with the recurrence's
 * scalars kept on the device; the host's stopping tests trail the GPU by one
 * round (a stopped run's extra round is discarded: same ranges bit for bit);
 * lo_hi (host, 2 nruns) receives the extreme Ritz values; partials: nruns *
 * pff_reduce_scratch_len() doubles, dots: 2 nruns doubles (device: alpha,
 * beta^2 per run).  Synchronises the stream. */
int pff_lanczos_ranges(int nruns, const pff_level* const* levels, const int* modes,
                       const int64_t* ns, const double* const* dhalf, double* const* work,
                       int max_iterations, double* lo_hi, double* partials, double* dots,
                       void* stream);

/* Copy `count` entries of each of `ncomp` components spaced `stride` entries
 * apart (component-major vectors; host<->device or device<->device, UVA) in
 * one strided copy -- the chunk transfers of the pipelined host path. */
int pff_copy_components(double* dst, const double* src, int64_t count, int ncomp,
                        int64_t stride, void* stream);

/* deterministic dot: partials = pff_reduce_scratch_len() doubles, out = 1 double */
int64_t pff_reduce_scratch_len(void);
int pff_dot(int64_t n, const double* x, const double* y, double* partials, double* out,
            void* stream);

/* Arnoldi column j of GMRES (src/krylov.py:76-80): V holds rows 0..j (row
 * stride ldv), w is overwritten by the MGS-orthogonalised vector;
 * h[0..j] = coefficients, h[j+1] = ||w||. */
int pff_mgs(int64_t n, int j, const double* V, int64_t ldv, double* w, double* partials,
            double* h, void* stream);

/* Arnoldi column j orthogonalised by low-synchronisation MGS (inverse
 * compact-WY form of src/krylov.py:76-84): h[0..j] are the MGS coefficients,
 * computed from V[0..j] . w and the Gram rows gram[i][k] = v_i . v_k (k < i,
 * row-major, leading dimension ldg > j; row j is written by this call, rows
 * < j must hold the earlier calls' rows of the same restart cycle); w is
 * replaced by w - V h and h[j+1] = |w|.  Two passes over V instead of MGS's
 * 2(j+1) dependent steps.  partials: (2 j + 3) * pff_reduce_scratch_len() / 2
 * doubles. */
int pff_mgs_lowsync(int64_t n, int j, const double* V, int64_t ldv, double* w, double* gram,
                    int64_t ldg, double* partials, double* h, void* stream);

/* pff_apply_cheb with the accumulator update acc += d + d' instead of
 * acc += d': the first fused step after a producer emitted d = d0 (the
 * separate pff_cheb_init pass's `acc += d0`, same rounding). */
int pff_apply_cheb_first(const pff_level* L, int mode, const double* d, double* d_out,
                         const double* rhs, double* cr, const double* invd, double* acc,
                         double c1, double c2, void* stream);

/* pff_apply_cheb with options: PFF_CHEB_FIRST = pff_apply_cheb_first's
 * acc += d + d'; PFF_CHEB_LAST = the last step of a pass: only acc is
 * written (cr and d_out are not stored; nothing reads them afterwards). */
/* PFF_CHEB_NOACC: the step leaves acc alone; the NEXT step then runs with
 * PFF_CHEB_FIRST and adds this step's d' (its own d) and its d' in the same
 * order, (acc + d) + d' -- bitwise the two separate updates, one acc read and
 * write fewer. */
enum { PFF_CHEB_FIRST = 1, PFF_CHEB_LAST = 2, PFF_CHEB_NOACC = 4 };
int pff_apply_cheb_ex(const pff_level* L, int mode, const double* d, double* d_out,
                      const double* rhs, double* cr, const double* invd, double* acc, double c1,
                      double c2, int flags, void* stream);

/* Fused residual dst = rhs - G src (mode FULL, UU or PHIROW) that also emits the
 * next smoothing block's Chebyshev start d0 = invd * dst / theta (FULL / UU: the
 * two u components, invd/d0 of length 2n; PHIROW: the phi output, length n).
 * UU: the u rows of the FULL residual alone -- bitwise the same values, the
 * Jacobian has no u-phi block (src/_kernels.py:611-669) -- for the smoother's
 * u-block residual, whose phi rows nothing reads (src/multigrid.py:262-276)
 * -- pff_cheb_init folded into the residual's store. */
int pff_apply_emit(const pff_level* L, int mode, const double* src, double* dst,
                   const double* rhs, const double* invd, double* d0, double theta,
                   void* stream);

/* First smoothing of a V-cycle level: z = r on constrained rows, 0 elsewhere
 * (3n); res_u = r[:2n] with constrained rows zeroed; d_u = invd_u res_u / theta
 * (pff_cons SELECT + EXCLUDE + pff_cheb_init in one pass). */
int pff_smooth_init(const pff_level* L, const double* r, double* z, double* res_u,
                    const double* invd_u, double* d_u, double theta, void* stream);
/* flags & PFF_SMOOTH_ADD_D0: z[:2n] also takes the Chebyshev start, z_u = d_u on
 * unconstrained rows (exactly 0 + d_u; d_u is 0 on constrained rows) -- the
 * `z += d` of src/multigrid.py:185, so the first fused step needs no PFF_CHEB_FIRST */
enum { PFF_SMOOTH_ADD_D0 = 1 };
int pff_smooth_init_ex(const pff_level* L, const double* r, double* z, double* res_u,
                       const double* invd_u, double* d_u, double theta, int flags, void* stream);

/* y = M x for a row-major dense device matrix M (rows x cols); x != y.  The
 * V-cycle below a small level as one precomputed linear map. */
int pff_dense_matvec(int64_t rows, int64_t cols, const double* M, const double* x, double* y,
                     void* stream);

/* Coarse-level solve of the V-cycle (replaces the coarse Chebyshev passes of
 * src/multigrid.py:311-328 on a coarse level of n <= 256 scalar nodes):
 * z_u = Cu r_u, t = r_phi - Gpu z_u, z_phi = Cp t, then z = r on the rows
 * with cmask != 0.  Cu (2n x 2n), Gpu (n x 2n), Cp (n x n): row-major device
 * matrices formed at setup (Cu, Cp: the fixed Chebyshev polynomials of the
 * masked diagonal blocks; Gpu: the masked phi-row's u columns); r, z: 3n. */
int pff_coarse_dense(int64_t n, const double* Cu, const double* Gpu, const double* Cp,
                     const uint8_t* cmask, const double* r, double* z, void* stream);

/* multi-dot out[i] = V[i] . w for i < k (CGS2 orthogonalisation of the
 * distributed GMRES); partials = k * pff_reduce_scratch_len() / 2 doubles */
int pff_mdot(int64_t n, int k, const double* V, int64_t ldv, const double* w, double* partials,
             double* out, void* stream);

/* out = sum_{i<k} y[i] V[i] (+ out if accumulate); y is a device array */
int pff_combine(int64_t n, int k, const double* V, int64_t ldv, const double* y, double* out,
                int accumulate, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PFF_B200_H */
