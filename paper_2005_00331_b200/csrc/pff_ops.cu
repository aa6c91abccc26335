// pff_ops.cu -- operator family on device: q-point refresh, Jacobian
// application (full / uu / phiphi / phi-row, optional fused r - J z),
// block diagonals, nonlinear residual.
//
// Generic path (any p in 1..4): one thread per cell, sum-factorised 1-D
// contractions in registers, q-point physics restated from
// src/_kernels.py:555-693.  No atomics anywhere, so results are identical run
// to run: the application writes per-cell element vectors into the level's
// scratch and a per-node gather sums them in increasing cell index (two
// launches, full parallelism -- the coarse levels of the V-cycle are latency
// bound); diagonals and residual add in four colour passes (cx mod 2,
// cy mod 2: cells of one colour share no node).  Identity rows/columns as in
// src/pff_operator.py:262-302.  The Q2 fast path lives in pff_sweep.cu.
#include "pff_internal.cuh"

namespace pff {

namespace {

constexpr int CELL_THREADS = 128;

inline unsigned grid_for(int64_t n, int threads) {
    return (unsigned)((n + threads - 1) / threads);
}

// One colour class of the cells in rows [row0, row0 + rows): colour bit 0 is
// the parity of cx, bit 1 the parity of cy.
struct Colour {
    int c, hx, hy, cy0;
    __host__ __device__ Colour(int colour, int ns, int row0, int rows) : c(colour) {
        hx = (ns - (colour & 1) + 1) >> 1;
        cy0 = row0 + (((row0 & 1) != (colour >> 1)) ? 1 : 0);
        const int left = row0 + rows - cy0;
        hy = left > 0 ? (left + 1) >> 1 : 0;
        if (hx < 0) hx = 0;
    }
    __host__ __device__ int64_t count() const { return (int64_t)hx * hy; }
    __device__ void cell(int64_t t, int& cx, int& cy) const {
        cx = (c & 1) + 2 * (int)(t % hx);
        cy = cy0 + 2 * (int)(t / hx);
    }
};

template <int N1>
__device__ __forceinline__ void cell_ids(const Mesh& m, int cx, int cy, int64_t (&gid)[N1][N1]) {
#pragma unroll
    for (int b = 0; b < N1; ++b)
#pragma unroll
        for (int a = 0; a < N1; ++a) gid[b][a] = m.node(cx, cy, a, b);
}

// value + reference gradients of a nodal field at the q x q points
template <int N1>
__device__ __forceinline__ void grad_q(const Shape& S, const double (&c)[N1][N1],
                                       double (&gx)[N1][N1], double (&gy)[N1][N1]) {
    double tx[N1][N1], td[N1][N1];
    fwd_x<N1>(S.N, c, tx);
    fwd_x<N1>(S.D, c, td);
    fwd_y<N1>(S.D, tx, gy);
    fwd_y<N1>(S.N, td, gx);
}

// ------------------------------------------------------------ refresh
// q-point linearisation cache, src/_kernels.py:447-516.  Layout
// qc[f][k][cell], f in {e11, e22, e12, g(phi~), g'(phi), pc}, k = jq*q+iq.
template <int P, bool MIEHE>
__global__ void __launch_bounds__(CELL_THREADS)
k_refresh(Mesh m, Win w, Shape S, Material M, const double* __restrict__ U,
          const double* __restrict__ pt, double* __restrict__ qc) {
    constexpr int N1 = P + 1, QQ = N1 * N1;
    const int64_t nc = w.ncell;
    int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (cell >= nc) return;
    int cx = (int)(cell % m.nside), cy = w.row0 + (int)(cell / m.nside);
    int64_t gid[N1][N1];
    cell_ids<N1>(m, cx, cy, gid);
#pragma unroll
    for (int b = 0; b < N1; ++b)
#pragma unroll
        for (int a = 0; a < N1; ++a) gid[b][a] = w.loc(m, gid[b][a]);
    const int64_t n = w.n;
    double cu[N1][N1], cv[N1][N1], cp[N1][N1], ct[N1][N1];
#pragma unroll
    for (int b = 0; b < N1; ++b)
#pragma unroll
        for (int a = 0; a < N1; ++a) {
            cu[b][a] = U[gid[b][a]];
            cv[b][a] = U[n + gid[b][a]];
            cp[b][a] = U[2 * n + gid[b][a]];
            ct[b][a] = pt[gid[b][a]];
        }
    double gxu[N1][N1], gyu[N1][N1], gxv[N1][N1], gyv[N1][N1], vp[N1][N1], vt[N1][N1];
    double tx[N1][N1];
    grad_q<N1>(S, cu, gxu, gyu);
    grad_q<N1>(S, cv, gxv, gyv);
    fwd_x<N1>(S.N, cp, tx);
    fwd_y<N1>(S.N, tx, vp);
    fwd_x<N1>(S.N, ct, tx);
    fwd_y<N1>(S.N, tx, vt);
    const double inv_h = 1.0 / m.h, gce = M.gc / M.eps, gdd = 2.0 * (1.0 - M.kappa);
#pragma unroll
    for (int jq = 0; jq < N1; ++jq)
#pragma unroll
        for (int iq = 0; iq < N1; ++iq) {
            double e11 = gxu[jq][iq] * inv_h;
            double e22 = gyv[jq][iq] * inv_h;
            double e12 = 0.5 * (gyu[jq][iq] + gxv[jq][iq]) * inv_h;
            double tre = e11 + e22;
            double g_t = (1.0 - M.kappa) * vt[jq][iq] * vt[jq][iq] + M.kappa;
            double esp = MIEHE ? esplus2(M.lam, M.mu, tre, eig2(e11, e22, e12))
                               : 0.5 * M.lam * tre * tre +
                                     M.mu * (e11 * e11 + e22 * e22 + 2.0 * e12 * e12);
            double* q = qc + (int64_t)(jq * N1 + iq) * nc + cell;
            const int64_t fs = (int64_t)QQ * nc;
            q[0] = e11;
            q[fs] = e22;
            q[2 * fs] = e12;
            q[3 * fs] = g_t;
            q[4 * fs] = gdd * vp[jq][iq];
            q[5 * fs] = gdd * esp + gce;
        }
}

// Weighted tangent cache of the generic path (Miehe): the reference's
// cache_tensors quantities (src/_kernels.py:517-548) per (q-point, cell) from
// the q-point cache, weight w_jq w_iq h^2 folded in; symmetric form
// (ds11, ds22, 2 ds12) = T (d11, d22, d12) as in the Q2 tiles (pff_sweep.cu)
template <int P, bool MIEHE>
__global__ void k_refresh_gtan(Mesh m, Win w, Shape S, Material M, const double* __restrict__ qc,
                               double* __restrict__ gt) {
    constexpr int N1 = P + 1, QQ = N1 * N1;
    const int64_t nc = w.ncell, fs = (int64_t)QQ * nc;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= fs) return;
    const int k = (int)(t / nc);
    const int jq = k / N1, iq = k - jq * N1;
    const double h = m.h, wv = S.w[jq] * S.w[iq] * h * h;
    const double* q = qc + t;
    const double e11 = q[0], e22 = q[fs], e12 = q[2 * fs], g = q[3 * fs], dg = q[4 * fs];
    const double tre = e11 + e22;
    // warp-group layout (Level::gtan_len): [group][array][jq][cell in group][iq]
    constexpr int CG = 32 / N1;
    const int64_t cell = t - (int64_t)k * nc, grp = cell / CG;
    const int cig = (int)(cell - grp * CG);
    const int64_t ag = (int64_t)QQ * CG;              // array stride within a group
    if (!MIEHE) {   // [g w][cw (sigma(e) x g' w)][pc w], as the Q2 tiles' none form
        double* o = gt + grp * (5 * ag) + (int64_t)(jq * CG + cig) * N1 + iq;
        o[0] = wv * g;
        o[ag] = wv * dg * (M.lam * tre + 2.0 * M.mu * e11);
        o[2 * ag] = wv * dg * (M.lam * tre + 2.0 * M.mu * e22);
        o[3 * ag] = wv * dg * 2.0 * (2.0 * M.mu * e12);
        o[4 * ag] = wv * q[5 * fs];
        return;
    }
    const double mm = 0.5 * (e11 + e22), dh = 0.5 * (e11 - e22);
    const double r = sqrt(dh * dh + e12 * e12);
    const Eig e = eig2(e11, e22, e12);
    const bool gap_ok = (e.ev1 - e.ev2) > 1e-12 * scale2(e11, e22, e12);
    const MieheQ mq = miehe_q(mm, gap_ok ? r : -r, e.c, e.s);
    double Mc[3][3], sp;
    miehe_dsig(M, g, mq, 1.0, 0.0, 0.0, Mc[0][0], Mc[1][0], Mc[2][0], sp);
    miehe_dsig(M, g, mq, 0.0, 1.0, 0.0, Mc[0][1], Mc[1][1], Mc[2][1], sp);
    miehe_dsig(M, g, mq, 0.0, 0.0, 1.0, Mc[0][2], Mc[1][2], Mc[2][2], sp);
    double q11, q22, q12;
    sigplus2(M.lam, M.mu, tre, e, q11, q22, q12);
    double* o = gt + grp * (10 * ag) + (int64_t)(jq * CG + cig) * N1 + iq;
    o[0] = wv * Mc[0][0];
    o[ag] = wv * 0.5 * (Mc[0][1] + Mc[1][0]);
    o[2 * ag] = wv * 0.5 * (Mc[0][2] + 2.0 * Mc[2][0]);
    o[3 * ag] = wv * Mc[1][1];
    o[4 * ag] = wv * 0.5 * (Mc[1][2] + 2.0 * Mc[2][1]);
    o[5 * ag] = wv * 2.0 * Mc[2][2];
    o[6 * ag] = wv * dg * q11;
    o[7 * ag] = wv * dg * q22;
    o[8 * ag] = wv * dg * 2.0 * q12;
    o[9 * ag] = wv * q[5 * fs];
}

// ----------------------------------------------------- Jacobian (generic)
template <int MODE>
struct ModeTraits {
    static constexpr bool DO_UU = MODE == MODE_FULL || MODE == MODE_UU;
    static constexpr bool DO_PP = MODE != MODE_UU;
    static constexpr bool DO_COUP = MODE == MODE_FULL || MODE == MODE_PHIROW;
    static constexpr bool NEED_U = DO_UU || DO_COUP;
};

// dst rows: constrained -> src (identity row); free -> 0, or for the fused
// Per-node gather of the element vectors (fixed cell order) with the identity
// rows of src/pff_operator.py:262-302; fused form dst = rhs - J src.
template <int P, int MODE>
__global__ void k_apply_gather(Mesh m, const uint8_t* __restrict__ flags,
                               const double* __restrict__ src, const double* __restrict__ rhs,
                               const double* __restrict__ ev, double* __restrict__ dst,
                               ChebArgs cheb) {
    constexpr int N1 = P + 1, QQ = N1 * N1;
    const int64_t n = m.n, nc = m.n_cells();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint8_t f = flags[i];
    // output components: (element-vector component, src offset, constraint bit)
    constexpr int NO = MODE == MODE_FULL ? 3 : MODE == MODE_UU ? 2 : 1;
    int comp[3], soff[3];
    bool cons[3];
    for (int c = 0; c < NO; ++c) {
        comp[c] = (MODE == MODE_FULL || MODE == MODE_UU) ? c : 2;
        soff[c] = MODE == MODE_PHIROW ? 2 : (MODE == MODE_PHIPHI ? 0 : c);
        cons[c] = comp[c] < 2 ? (f & F_DIR) : (f & F_ACT);
    }
    double acc[3] = {0.0, 0.0, 0.0};
    node_cells_p<P>(m, i, 0, m.nside, [&](int cx, int cy, int a, int b) {
        const int64_t cell = (int64_t)cy * m.nside + cx;
#pragma unroll
        for (int c = 0; c < NO; ++c)
            acc[c] += ev[((int64_t)comp[c] * nc + cell) * QQ + b * N1 + a];
    });
#pragma unroll
    for (int c = 0; c < NO; ++c) {
        const double sv = src[soff[c] * n + i];
        const double v = cons[c] ? sv : acc[c];
        const double x = rhs ? rhs[c * n + i] - v : v;
        if (!cheb.last) dst[c * n + i] = x;
        if (cheb.dout) {   // fused Chebyshev step on the residual just formed
            const double dn = cheb_update(cheb.c1, sv, cheb.c2, cheb.invd[c * n + i], x);
            if (!cheb.last) cheb.dout[c * n + i] = dn;
            if (!cheb.noacc) {
                const double av = cheb.acc[c * n + i];
                cheb.acc[c * n + i] = (cheb.acc_src ? av + sv : av) + dn;
            }
        } else if (c < cheb.emit_nc) {   // the next block's Chebyshev d0
            cheb.emit[c * n + i] = cheb.invd[c * n + i] * x / cheb.theta;
        }
    }
}

// Cooperative variant: p+1 lanes per cell (32/(p+1) cells per warp).  Lane t
// owns node row b = t for the x-passes and Gauss column iq = t for the
// y-passes and the q-point physics; the two transposes go through shared
// memory.  Per-lane state is ~1/(p+1) of the thread-per-cell kernel, so high
// orders neither spill nor thrash the instruction cache, and the latency of a
// cell on the small multigrid levels drops by ~(p+1).  Same arithmetic
// (src/_kernels.py:555-693), same element-vector output.
constexpr int COOP_WARPS = 4;
#ifndef COOP_MIN_BLOCKS
#define COOP_MIN_BLOCKS 3
#endif

template <int P, bool MIEHE, int MODE, bool TC = false>
__global__ void __launch_bounds__(32 * COOP_WARPS, COOP_MIN_BLOCKS)
k_apply_coop(Mesh m, Shape S, Material M, const double* __restrict__ qc,
             const uint8_t* __restrict__ flags, const double* __restrict__ sx,
             const double* __restrict__ sy, const double* __restrict__ sp,
             double* __restrict__ ev, const double* __restrict__ gt) {
    using T = ModeTraits<MODE>;
    constexpr int N1 = P + 1, QQ = N1 * N1, CPW = 32 / N1;
    constexpr int NA = 6;   // staged arrays per cell
    __shared__ double buf[COOP_WARPS][CPW][NA][N1][N1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = lane / N1, t = lane - c * N1;
    const int64_t nc = m.n_cells();
    const int64_t cell = ((int64_t)blockIdx.x * COOP_WARPS + warp) * CPW + c;
    const bool on = c < CPW && cell < nc;
    const int cx = on ? (int)(cell % m.nside) : 0, cy = on ? (int)(cell / m.nside) : 0;
    const double h = m.h, inv_h = 1.0 / h;
    double (&B)[NA][N1][N1] = buf[warp][c < CPW ? c : 0];

    // ---- phase 1: node row b = t, x-pass (value and derivative) per field
    if (on) {
        double ux[N1], uy[N1], up[N1];
#pragma unroll
        for (int a = 0; a < N1; ++a) {
            const int64_t g = m.node(cx, cy, a, t);
            const uint8_t f = flags[g];
            ux[a] = uy[a] = up[a] = 0.0;
            if (T::NEED_U) {
                ux[a] = (f & F_DIR) ? 0.0 : sx[g];
                uy[a] = (f & F_DIR) ? 0.0 : sy[g];
            }
            if (T::DO_PP) up[a] = (f & F_ACT) ? 0.0 : sp[g];
        }
#pragma unroll
        for (int iq = 0; iq < N1; ++iq) {
            double xn_u = 0.0, xd_u = 0.0, xn_v = 0.0, xd_v = 0.0, xn_p = 0.0, xd_p = 0.0;
#pragma unroll
            for (int a = 0; a < N1; ++a) {
                const double na = S.N[iq][a], da = S.D[iq][a];
                if (T::NEED_U) {
                    xn_u = fma(na, ux[a], xn_u);
                    xd_u = fma(da, ux[a], xd_u);
                    xn_v = fma(na, uy[a], xn_v);
                    xd_v = fma(da, uy[a], xd_v);
                }
                if (T::DO_PP) {
                    xn_p = fma(na, up[a], xn_p);
                    xd_p = fma(da, up[a], xd_p);
                }
            }
            B[0][t][iq] = xn_u;
            B[1][t][iq] = xd_u;
            B[2][t][iq] = xn_v;
            B[3][t][iq] = xd_v;
            B[4][t][iq] = xn_p;
            B[5][t][iq] = xd_p;
        }
    }
    __syncwarp();
    // ---- phase 2: Gauss column iq = t: y-pass, physics, backward y-pass
    double X[NA][N1];
#pragma unroll
    for (int A = 0; A < NA; ++A)
#pragma unroll
        for (int b = 0; b < N1; ++b) X[A][b] = on ? B[A][b][t] : 0.0;
    double Tr[NA][N1];   // uD uN vD vN pN pD
#pragma unroll
    for (int A = 0; A < NA; ++A)
#pragma unroll
        for (int b = 0; b < N1; ++b) Tr[A][b] = 0.0;
    if (on) {
        const int iq = t;
        const int64_t fs = (int64_t)QQ * nc;
#pragma unroll
        for (int jq = 0; jq < N1; ++jq) {
            double yn[NA], yd[NA];
#pragma unroll
            for (int A = 0; A < NA; ++A) {
                double sn = 0.0, sd = 0.0;
#pragma unroll
                for (int b = 0; b < N1; ++b) {
                    sn = fma(S.N[jq][b], X[A][b], sn);
                    sd = fma(S.D[jq][b], X[A][b], sd);
                }
                yn[A] = sn;
                yd[A] = sd;
            }
            const double wq = S.w[jq] * S.w[iq];
            const double wg = wq * h, wv = wq * h * h;
            const double* q = qc + (int64_t)(jq * N1 + iq) * nc + cell;
            double s11 = 0.0, s22 = 0.0, s12 = 0.0, coup = 0.0;
            const double d11 = yn[1] * inv_h;                 // N_y (D_x u)
            const double d22 = yd[2] * inv_h;                 // D_y (N_x v)
            const double d12 = 0.5 * (yd[0] + yn[3]) * inv_h;
            // warp-group layout: this warp's group is its cell block, lanes (c, iq) contiguous
            constexpr int NARR = MIEHE ? 10 : 5, GCW = MIEHE ? 6 : 1, GPC = GCW + 3;
            const double* g = TC ? gt + ((int64_t)blockIdx.x * COOP_WARPS + warp) * (NARR * QQ * CPW) +
                                       (int64_t)(jq * CPW + c) * N1 + iq
                                 : nullptr;
            constexpr int64_t gs = (int64_t)QQ * CPW;   // array stride
            if (T::NEED_U && TC) {
                // cached weighted tangent (x wv); the backward passes expect x wg = wv / h
                if (T::DO_UU && MIEHE) {
                    const double t00 = g[0], t01 = g[gs], t02 = g[2 * gs];
                    const double t11 = g[3 * gs], t12 = g[4 * gs], t22 = g[5 * gs];
                    s11 = fma(t00, d11, fma(t01, d22, t02 * d12)) * inv_h;
                    s22 = fma(t01, d11, fma(t11, d22, t12 * d12)) * inv_h;
                    s12 = 0.5 * fma(t02, d11, fma(t12, d22, t22 * d12)) * inv_h;
                } else if (T::DO_UU) {   // none: g w (lambda tr de I + 2 mu de)
                    const double gw = g[0] * inv_h;
                    const double lt = M.lam * (d11 + d22), mu2 = 2.0 * M.mu;
                    s11 = gw * fma(mu2, d11, lt);
                    s22 = gw * fma(mu2, d22, lt);
                    s12 = (gw * mu2) * d12;
                }
                if (T::DO_COUP)
                    coup = fma(g[GCW * gs], d11, fma(g[(GCW + 1) * gs], d22, g[(GCW + 2) * gs] * d12));   // x wv
            } else if (T::NEED_U) {
                double ds11, ds22, ds12, spde;
                dsig<MIEHE>(M.lam, M.mu, q[3 * fs], q[0], q[fs], q[2 * fs], d11, d22, d12, ds11,
                            ds22, ds12, spde);
                coup = q[4 * fs] * spde;
                s11 = ds11 * wg;
                s22 = ds22 * wg;
                s12 = ds12 * wg;
            }
            double fv = 0.0, fgx = 0.0, fgy = 0.0;
            if (T::DO_PP) {
                if (TC) {
                    fv = g[GPC * gs] * yn[4];
                    if (T::DO_COUP) fv += coup;
                } else {
                    double pval = q[5 * fs] * yn[4];
                    if (T::DO_COUP) pval += coup;
                    fv = pval * wv;
                }
                fgx = M.gc * M.eps * yn[5] * inv_h * wg;
                fgy = M.gc * M.eps * yd[4] * inv_h * wg;
            }
#pragma unroll
            for (int b = 0; b < N1; ++b) {
                const double nb = S.N[jq][b], db = S.D[jq][b];
                if (T::DO_UU) {
                    Tr[0][b] = fma(nb, s11, Tr[0][b]);
                    Tr[1][b] = fma(db, s12, Tr[1][b]);
                    Tr[2][b] = fma(nb, s12, Tr[2][b]);
                    Tr[3][b] = fma(db, s22, Tr[3][b]);
                }
                if (T::DO_PP) {
                    Tr[4][b] = fma(db, fgy, fma(nb, fv, Tr[4][b]));
                    Tr[5][b] = fma(nb, fgx, Tr[5][b]);
                }
            }
        }
    }
    __syncwarp();
    if (on) {
#pragma unroll
        for (int A = 0; A < NA; ++A)
#pragma unroll
            for (int b = 0; b < N1; ++b) B[A][b][t] = Tr[A][b];
    }
    __syncwarp();
    // ---- phase 3: node row b = t, backward x-pass, element vectors
    if (!on) return;
    double Rr[NA][N1];
#pragma unroll
    for (int A = 0; A < NA; ++A)
#pragma unroll
        for (int iq = 0; iq < N1; ++iq) Rr[A][iq] = B[A][t][iq];
#pragma unroll
    for (int a = 0; a < N1; ++a) {
        double ru = 0.0, rv = 0.0, rp = 0.0;
#pragma unroll
        for (int iq = 0; iq < N1; ++iq) {
            const double na = S.N[iq][a], da = S.D[iq][a];
            if (T::DO_UU) {
                ru = fma(da, Rr[0][iq], fma(na, Rr[1][iq], ru));
                rv = fma(da, Rr[2][iq], fma(na, Rr[3][iq], rv));
            }
            if (T::DO_PP) rp = fma(na, Rr[4][iq], fma(da, Rr[5][iq], rp));
        }
        const int loc = t * N1 + a;
        if (T::DO_UU) {
            ev[cell * QQ + loc] = ru;
            ev[(nc + cell) * QQ + loc] = rv;
        }
        if (T::DO_PP) ev[(2 * nc + cell) * QQ + loc] = rp;
    }
}

// ---------------------------------------------------------- diagonals
// src/_kernels.py:700-746, with the state eigensystem computed once per
// quadrature point instead of once per (node, point).
template <int P, bool MIEHE>
__global__ void __launch_bounds__(CELL_THREADS)
k_diag_cells(Mesh m, Win w, Shape S, Material M, const double* __restrict__ qc, double* dx,
             double* dy, double* dp, Colour col) {
    constexpr int N1 = P + 1, QQ = N1 * N1;
    const int64_t nc = w.ncell;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= col.count()) return;
    int cx, cy;
    col.cell(tid, cx, cy);
    const int64_t cell = (int64_t)(cy - w.row0) * m.nside + cx;
    const double h = m.h, inv_h = 1.0 / h;
    const int64_t fs = (int64_t)QQ * nc;
    double ax[N1][N1] = {}, ay[N1][N1] = {}, ap[N1][N1] = {};
#pragma unroll
    for (int jq = 0; jq < N1; ++jq)
#pragma unroll
        for (int iq = 0; iq < N1; ++iq) {
            const double wq = S.w[jq] * S.w[iq] * h * h;
            const double* q = qc + (int64_t)(jq * N1 + iq) * nc + cell;
            const double e11 = q[0], e22 = q[fs], e12 = q[2 * fs], g_t = q[3 * fs],
                         pc = q[5 * fs];
            // Miehe: the split tangent is linear in the direction strain, so its three unit
            // columns (one dsig_split_pre each, per q-point) replace the two evaluations
            // per (node, q-point) of src/_kernels.py:700-746: t[i][k] = s_i for unit
            // direction k, (s11, s22, s12) over (d11, d22, d12)
            double t[3][3] = {};
            if (MIEHE) {
                const Eig e = eig2(e11, e22, e12);
                const double scale = scale2(e11, e22, e12), tre = e11 + e22;
                double unused;
                dsig_split_pre(M.lam, M.mu, g_t, e, scale, tre, 1.0, 0.0, 0.0, t[0][0], t[1][0],
                               t[2][0], unused);
                dsig_split_pre(M.lam, M.mu, g_t, e, scale, tre, 0.0, 1.0, 0.0, t[0][1], t[1][1],
                               t[2][1], unused);
                dsig_split_pre(M.lam, M.mu, g_t, e, scale, tre, 0.0, 0.0, 1.0, t[0][2], t[1][2],
                               t[2][2], unused);
            }
#pragma unroll
            for (int b = 0; b < N1; ++b)
#pragma unroll
                for (int a = 0; a < N1; ++a) {
                    double gx = S.D[iq][a] * S.N[jq][b] * inv_h;
                    double gy = S.N[iq][a] * S.D[jq][b] * inv_h;
                    double val = S.N[iq][a] * S.N[jq][b];
                    double x11, x12, y12, y22;
                    if (MIEHE) {
                        // u_x direction (gx, 0, gy/2), u_y direction (0, gy, gx/2)
                        x11 = fma(t[0][2], 0.5 * gy, t[0][0] * gx);
                        x12 = fma(t[2][2], 0.5 * gy, t[2][0] * gx);
                        y22 = fma(t[1][2], 0.5 * gx, t[1][1] * gy);
                        y12 = fma(t[2][2], 0.5 * gx, t[2][1] * gy);
                    } else {
                        x11 = g_t * (M.lam + 2.0 * M.mu) * gx;
                        x12 = g_t * M.mu * gy;
                        y22 = g_t * (M.lam + 2.0 * M.mu) * gy;
                        y12 = g_t * M.mu * gx;
                    }
                    ax[b][a] += (x11 * gx + x12 * gy) * wq;
                    ay[b][a] += (y12 * gx + y22 * gy) * wq;
                    ap[b][a] += (pc * val * val + M.gc * M.eps * (gx * gx + gy * gy)) * wq;
                }
        }
#pragma unroll
    for (int b = 0; b < N1; ++b)
#pragma unroll
        for (int a = 0; a < N1; ++a) {
            int64_t g = w.loc(m, m.node(cx, cy, a, b));
            dx[g] += ax[b][a];
            dy[g] += ay[b][a];
            dp[g] += ap[b][a];
        }
}

// constrained entries -> 1 (src/pff_operator.py:320-326), optional reciprocal
__global__ void k_diag_finalize(int64_t n, const uint8_t* __restrict__ flags, double* dx,
                                double* dy, double* dp, int invert) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint8_t f = flags[i];
    double x = (f & F_DIR) ? 1.0 : dx[i];
    double y = (f & F_DIR) ? 1.0 : dy[i];
    double p = (f & F_ACT) ? 1.0 : dp[i];
    if (invert) {
        x = 1.0 / x;
        y = 1.0 / y;
        p = 1.0 / p;
    }
    dx[i] = x;
    dy[i] = y;
    dp[i] = p;
}

// ------------------------------------------------------------ residual
// src/_kernels.py:319-440 (the Newton right-hand side)
template <int P, bool MIEHE>
__global__ void __launch_bounds__(CELL_THREADS)
k_residual_cells(Mesh m, Shape S, Material M, const double* __restrict__ U,
                 const double* __restrict__ pt, double* out, Colour col) {
    constexpr int N1 = P + 1;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= col.count()) return;
    int cx, cy;
    col.cell(tid, cx, cy);
    const int64_t n = m.n;
    int64_t gid[N1][N1];
    cell_ids<N1>(m, cx, cy, gid);
    double cu[N1][N1], cv[N1][N1], cp[N1][N1], ct[N1][N1];
#pragma unroll
    for (int b = 0; b < N1; ++b)
#pragma unroll
        for (int a = 0; a < N1; ++a) {
            cu[b][a] = U[gid[b][a]];
            cv[b][a] = U[n + gid[b][a]];
            cp[b][a] = U[2 * n + gid[b][a]];
            ct[b][a] = pt[gid[b][a]];
        }
    double gxu[N1][N1], gyu[N1][N1], gxv[N1][N1], gyv[N1][N1];
    double vp[N1][N1], gxp[N1][N1], gyp[N1][N1], vt[N1][N1], tx[N1][N1], td[N1][N1];
    grad_q<N1>(S, cu, gxu, gyu);
    grad_q<N1>(S, cv, gxv, gyv);
    fwd_x<N1>(S.N, cp, tx);
    fwd_x<N1>(S.D, cp, td);
    fwd_y<N1>(S.N, tx, vp);
    fwd_y<N1>(S.D, tx, gyp);
    fwd_y<N1>(S.N, td, gxp);
    fwd_x<N1>(S.N, ct, tx);
    fwd_y<N1>(S.N, tx, vt);
    const double h = m.h, inv_h = 1.0 / h, gce = M.gc / M.eps;
    double s11[N1][N1], s22[N1][N1], s12[N1][N1], fv[N1][N1], fgx[N1][N1], fgy[N1][N1];
#pragma unroll
    for (int jq = 0; jq < N1; ++jq)
#pragma unroll
        for (int iq = 0; iq < N1; ++iq) {
            const double wq = S.w[jq] * S.w[iq];
            const double wg = wq * h, wv = wq * h * h;
            double e11 = gxu[jq][iq] * inv_h;
            double e22 = gyv[jq][iq] * inv_h;
            double e12 = 0.5 * (gyu[jq][iq] + gxv[jq][iq]) * inv_h;
            double tre = e11 + e22;
            double phv = vp[jq][iq], ptv = vt[jq][iq];
            double g_t = (1.0 - M.kappa) * ptv * ptv + M.kappa;
            double sp11, sp22, sp12, sm11 = 0.0, sm22 = 0.0, sm12 = 0.0, esp;
            if (MIEHE) {
                Eig e = eig2(e11, e22, e12);
                sigplus2(M.lam, M.mu, tre, e, sp11, sp22, sp12);
                sm11 = M.lam * tre + 2.0 * M.mu * e11 - sp11;
                sm22 = M.lam * tre + 2.0 * M.mu * e22 - sp22;
                sm12 = 2.0 * M.mu * e12 - sp12;
                esp = esplus2(M.lam, M.mu, tre, e);
            } else {
                sp11 = M.lam * tre + 2.0 * M.mu * e11;
                sp22 = M.lam * tre + 2.0 * M.mu * e22;
                sp12 = 2.0 * M.mu * e12;
                esp = 0.5 * M.lam * tre * tre + M.mu * (e11 * e11 + e22 * e22 + 2.0 * e12 * e12);
            }
            s11[jq][iq] = (g_t * sp11 + sm11) * wg;
            s22[jq][iq] = (g_t * sp22 + sm22) * wg;
            s12[jq][iq] = (g_t * sp12 + sm12) * wg;
            double dgv = 2.0 * (1.0 - M.kappa) * phv;
            fv[jq][iq] = (dgv * esp - gce * (1.0 - phv)) * wv;
            fgx[jq][iq] = M.gc * M.eps * gxp[jq][iq] * inv_h * wg;
            fgy[jq][iq] = M.gc * M.eps * gyp[jq][iq] * inv_h * wg;
        }
    double t[N1][N1], ru[N1][N1] = {}, rv[N1][N1] = {}, rp[N1][N1] = {};
    bwd_y<N1>(S.N, s11, t);
    bwd_x_add<N1>(S.D, t, ru);
    bwd_y<N1>(S.D, s12, t);
    bwd_x_add<N1>(S.N, t, ru);
    bwd_y<N1>(S.N, s12, t);
    bwd_x_add<N1>(S.D, t, rv);
    bwd_y<N1>(S.D, s22, t);
    bwd_x_add<N1>(S.N, t, rv);
    bwd_y<N1>(S.N, fv, t);
    bwd_x_add<N1>(S.N, t, rp);
    bwd_y<N1>(S.N, fgx, t);
    bwd_x_add<N1>(S.D, t, rp);
    bwd_y<N1>(S.D, fgy, t);
    bwd_x_add<N1>(S.N, t, rp);
#pragma unroll
    for (int b = 0; b < N1; ++b)
#pragma unroll
        for (int a = 0; a < N1; ++a) {
            out[gid[b][a]] += ru[b][a];
            out[n + gid[b][a]] += rv[b][a];
            out[2 * n + gid[b][a]] += rp[b][a];
        }
}

__global__ void k_residual_mask(int64_t n, const uint8_t* __restrict__ flags, double* out,
                                int mask_dirichlet, int mask_active) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint8_t f = flags[i];
    if (mask_dirichlet && (f & F_DIR)) {
        out[i] = 0.0;
        out[n + i] = 0.0;
    }
    if (mask_active && (f & F_ACT)) out[2 * n + i] = 0.0;
}

// ------------------------------------------------------------ dispatch
template <template <int, bool> class F, typename... A>
cudaError_t dispatch_p_split(int p, bool miehe, A... args) {
    switch (p * 2 + (miehe ? 1 : 0)) {
        case 2: return F<1, false>::run(args...);
        case 3: return F<1, true>::run(args...);
        case 4: return F<2, false>::run(args...);
        case 5: return F<2, true>::run(args...);
        case 6: return F<3, false>::run(args...);
        case 7: return F<3, true>::run(args...);
        case 8: return F<4, false>::run(args...);
        case 9: return F<4, true>::run(args...);
    }
    return cudaErrorInvalidValue;
}

template <int P, bool MIEHE>
struct RefreshL {
    static cudaError_t run(const Level* L, cudaStream_t s) {
        const Mesh& m = L->mesh;
        const Win w = L->win();
        k_refresh<P, MIEHE><<<grid_for(w.ncell, CELL_THREADS), CELL_THREADS, 0, s>>>(
            m, w, L->shape, L->mat, L->U, L->phi_tilde, L->qcache);
        count_launches(1);
        if (L->gtan_len() > 0) {
            const int64_t nq = (int64_t)(P + 1) * (P + 1) * w.ncell;
            k_refresh_gtan<P, MIEHE><<<grid_for(nq, 256), 256, 0, s>>>(m, w, L->shape, L->mat, L->qcache,
                                                               L->gtan());
            count_launches(1);
        }
        return cudaGetLastError();
    }
};

template <int P, bool MIEHE>
struct ApplyL {
    static cudaError_t run(const Level* L, int mode, const double* src, double* dst,
                           const double* rhs, cudaStream_t s, const ChebArgs* cheb) {
        ChebArgs cb{nullptr, nullptr, nullptr, 0.0, 0.0};
        if (cheb) cb = *cheb;
        const Mesh& m = L->mesh;
        const int64_t n = m.n;
        const unsigned gi = grid_for(n, 256);
        constexpr int CPB = COOP_WARPS * (32 / (P + 1));   // cells per block
        const unsigned gc = grid_for(m.n_cells(), CPB);
        const double* q = L->qcache;
        const uint8_t* f = L->flags;
        double* ev = L->ev();
        const bool tc = L->gtan_len() > 0;
        const double* gt = tc ? L->gtan() : nullptr;
        switch (mode) {
            case MODE_FULL:
                (tc ? k_apply_coop<P, MIEHE, MODE_FULL, true> : k_apply_coop<P, MIEHE, MODE_FULL, false>)<<<gc, 32 * COOP_WARPS, 0, s>>>(
                    m, L->shape, L->mat, q, f, src, src + n, src + 2 * n, ev, gt);
                k_apply_gather<P, MODE_FULL><<<gi, 256, 0, s>>>(m, f, src, rhs, ev, dst, cb);
                break;
            case MODE_UU:
                (tc ? k_apply_coop<P, MIEHE, MODE_UU, true> : k_apply_coop<P, MIEHE, MODE_UU, false>)<<<gc, 32 * COOP_WARPS, 0, s>>>(
                    m, L->shape, L->mat, q, f, src, src + n, nullptr, ev, gt);
                k_apply_gather<P, MODE_UU><<<gi, 256, 0, s>>>(m, f, src, rhs, ev, dst, cb);
                break;
            case MODE_PHIPHI:
                (tc ? k_apply_coop<P, MIEHE, MODE_PHIPHI, true> : k_apply_coop<P, MIEHE, MODE_PHIPHI, false>)<<<gc, 32 * COOP_WARPS, 0, s>>>(
                    m, L->shape, L->mat, q, f, nullptr, nullptr, src, ev, gt);
                k_apply_gather<P, MODE_PHIPHI><<<gi, 256, 0, s>>>(m, f, src, rhs, ev, dst, cb);
                break;
            case MODE_PHIROW:
                (tc ? k_apply_coop<P, MIEHE, MODE_PHIROW, true> : k_apply_coop<P, MIEHE, MODE_PHIROW, false>)<<<gc, 32 * COOP_WARPS, 0, s>>>(
                    m, L->shape, L->mat, q, f, src, src + n, src + 2 * n, ev, gt);
                k_apply_gather<P, MODE_PHIROW><<<gi, 256, 0, s>>>(m, f, src, rhs, ev, dst, cb);
                break;
            default:
                return cudaErrorInvalidValue;
        }
        count_launches(2);
        return cudaGetLastError();
    }
};

template <int P, bool MIEHE>
struct DiagL {
    static cudaError_t run(const Level* L, double* dx, double* dy, double* dp, int invert,
                           cudaStream_t s) {
        const Mesh& m = L->mesh;
        const Win w = L->win();
        cudaMemsetAsync(dx, 0, sizeof(double) * w.n, s);
        cudaMemsetAsync(dy, 0, sizeof(double) * w.n, s);
        cudaMemsetAsync(dp, 0, sizeof(double) * w.n, s);
        count_launches(3);
        for (int c = 0; c < 4; ++c) {
            const Colour col(c, m.nside, w.row0, (int)(w.ncell / m.nside));
            if (col.count() == 0) continue;
            k_diag_cells<P, MIEHE><<<grid_for(col.count(), CELL_THREADS), CELL_THREADS, 0, s>>>(
                m, w, L->shape, L->mat, L->qcache, dx, dy, dp, col);
            count_launches(1);
        }
        k_diag_finalize<<<grid_for(w.n, 256), 256, 0, s>>>(w.n, L->flags, dx, dy, dp, invert);
        count_launches(1);
        return cudaGetLastError();
    }
};

template <int P, bool MIEHE>
struct ResidualL {
    static cudaError_t run(const Level* L, double* out, int md, int ma, cudaStream_t s) {
        const Mesh& m = L->mesh;
        cudaMemsetAsync(out, 0, sizeof(double) * 3 * m.n, s);
        count_launches(1);
        for (int c = 0; c < 4; ++c) {
            const Colour col(c, m.nside, 0, m.nside);
            if (col.count() == 0) continue;
            k_residual_cells<P, MIEHE><<<grid_for(col.count(), CELL_THREADS), CELL_THREADS, 0, s>>>(
                m, L->shape, L->mat, L->U, L->phi_tilde, out, col);
            count_launches(1);
        }
        k_residual_mask<<<grid_for(m.n, 256), 256, 0, s>>>(m.n, L->flags, out, md, ma);
        count_launches(1);
        return cudaGetLastError();
    }
};

}  // namespace

cudaError_t launch_refresh(const Level& L, cudaStream_t s) {
    cudaError_t e = dispatch_p_split<RefreshL>(L.mesh.p, L.miehe, &L, s);
    if (e == cudaSuccess && L.sweep_ok()) e = launch_refresh_tiled(L, s);
    if (e == cudaSuccess && L.sweep4_ok()) e = launch_refresh_tile4(L, s);
    return e;
}

static bool g_generic_apply = false;
void set_generic_apply(bool on) { g_generic_apply = on; }

cudaError_t launch_apply(const Level& L, int mode, const double* src, double* dst,
                         const double* rhs, cudaStream_t s, const ChebArgs* cheb) {
    bool handled = false;
    if (cheb && cheb->dout && (!rhs || (mode != MODE_UU && mode != MODE_PHIPHI) || cheb->dout == src))
        return cudaErrorInvalidValue;
    if (cheb && !cheb->dout &&
        (!rhs || !cheb->emit || !cheb->invd || mode == MODE_PHIPHI ||
         cheb->emit_nc != (mode == MODE_PHIROW ? 1 : 2)))
        return cudaErrorInvalidValue;
    if (L.windowed()) {   // slabs run the write-once sweep kernel only
        cudaError_t e = launch_sweep_apply(L, mode, src, dst, rhs, s, &handled, cheb);
        return handled ? e : cudaErrorNotSupported;
    }
    if (!g_generic_apply) {
        cudaError_t e = launch_sweep_apply(L, mode, src, dst, rhs, s, &handled, cheb);
        if (handled || e != cudaSuccess) return e;
        if (!cheb) {   // Q4 write-once sweep (plain and fused forms)
            e = launch_sweep4_apply(L, mode, src, dst, rhs, s, &handled);
            if (handled || e != cudaSuccess) return e;
        }
    }
    return dispatch_p_split<ApplyL>(L.mesh.p, L.miehe, &L, mode, src, dst, rhs, s, cheb);
}

cudaError_t launch_diagonal(const Level& L, double* dx, double* dy, double* dp, int invert,
                            cudaStream_t s) {
    return dispatch_p_split<DiagL>(L.mesh.p, L.miehe, &L, dx, dy, dp, invert, s);
}

cudaError_t launch_residual(const Level& L, double* out, int md, int ma, cudaStream_t s) {
    if (L.windowed()) return cudaErrorNotSupported;
    return dispatch_p_split<ResidualL>(L.mesh.p, L.miehe, &L, out, md, ma, s);
}

}  // namespace pff
