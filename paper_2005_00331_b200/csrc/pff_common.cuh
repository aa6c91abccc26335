// pff_common.cuh -- shared device definitions for the B200 PFF hot path.
//
// Vector layout is exactly the reference's (src/mesh_hierarchy.py:10-13,
// 156-189): component-major [u_x | u_y | phi], each n = n_grid + n_dup
// scalar nodes, grid node (i, j) at j*np1 + i (x fastest), upper slit
// copies appended at n_grid + i.  The connectivity array of the reference
// is replaced by the closed form in Mesh::node().
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pff {

constexpr int PMAX = 4;
constexpr int NMAX = PMAX + 1;

// 1-D shape data at Gauss points (src/tensor_basis.py:66-81), row = quad
// point, column = support point.  Passed by value: lives in the kernel
// parameter bank, so compile-time-indexed reads become constant operands.
struct Shape {
    double N[NMAX][NMAX];
    double D[NMAX][NMAX];
    double w[NMAX];
};

// Coarse-basis values at the fine support points of child 0/1
// (src/multigrid.py:58-61): E[child][k][m] = l_m((child + x_k) / 2).
struct Embed {
    double E[2][NMAX][NMAX];
};

struct Material {
    double lam, mu, gc, kappa, eps;
};

enum Mode : int { MODE_FULL = 0, MODE_UU = 1, MODE_PHIPHI = 2, MODE_PHIROW = 3 };
enum Flag : uint8_t { F_DIR = 1, F_ACT = 2 };

struct Mesh {
    int p, level, nside;
    int64_t np1, n_grid, n_dup, i_mid, n;
    double h;

    __host__ __device__ static Mesh make(int p, int level) {
        Mesh m;
        m.p = p;
        m.level = level;
        m.nside = 1 << level;
        m.np1 = (int64_t)p * m.nside + 1;
        m.n_grid = m.np1 * m.np1;
        m.i_mid = (int64_t)p * m.nside / 2;
        m.n_dup = level >= 1 ? m.i_mid : 0;
        m.n = m.n_grid + m.n_dup;
        m.h = 1.0 / (double)m.nside;
        return m;
    }
    __host__ __device__ int64_t n_cells() const { return (int64_t)nside * nside; }
    // src/mesh_hierarchy.py:180-187
    __host__ __device__ __forceinline__ int64_t node(int cx, int cy, int a, int b) const {
        int64_t j = (int64_t)cy * p + b;
        int64_t i = (int64_t)cx * p + a;
        if (level >= 1 && cy >= (nside >> 1) && j == i_mid && i < i_mid) return n_grid + i;
        return j * np1 + i;
    }
};

// Chebyshev smoother update d' = c1 d + c2 D^-1 r (src/multigrid.py:189-195),
// one explicit rounding sequence shared by the standalone step and the
// steps fused into the block applications (bitwise identical results)
__device__ __forceinline__ double cheb_update(double c1, double d, double c2, double invd,
                                             double r) {
    return fma(c2, invd * r, c1 * d);
}

// ------------------------------------------------------------- physics
// 2-D symmetric tensors as (11, 22, 12) triples; restated from
// src/_kernels.py:26-123 (same branch structure, selects instead of ifs).

struct Eig {
    double ev1, ev2, c, s;
};

__device__ __forceinline__ double posp(double x) { return x > 0.0 ? x : 0.0; }

__device__ __forceinline__ Eig eig2(double a11, double a22, double a12) {
    Eig e;
    double m = 0.5 * (a11 + a22);
    double dh = 0.5 * (a11 - a22);
    double r = sqrt(dh * dh + a12 * a12);
    e.ev1 = m + r;
    e.ev2 = m - r;
    bool left = dh <= 0.0;
    double vx = left ? a12 : r + dh;
    double vy = left ? r - dh : a12;
    double nrm = sqrt(vx * vx + vy * vy);
    bool ok = nrm > 0.0;
    e.c = ok ? vx / nrm : 1.0;
    e.s = ok ? vy / nrm : 0.0;
    return e;
}

__device__ __forceinline__ double scale2(double e11, double e22, double e12) {
    double f = sqrt(e11 * e11 + e22 * e22 + 2.0 * e12 * e12);
    return f > 1.0 ? f : 1.0;
}

__device__ __forceinline__ void dpos2(const Eig& e, double scale, double d11, double d22,
                                      double d12, double& o11, double& o22, double& o12) {
    double c = e.c, s = e.s;
    double t0 = d11 * c + d12 * s;
    double t1 = d12 * c + d22 * s;
    double dl1 = c * t0 + s * t1;
    double dl2 = s * s * d11 - 2.0 * s * c * d12 + c * c * d22;
    double dl1p = e.ev1 >= 0.0 ? dl1 : 0.0;
    double dl2p = e.ev2 >= 0.0 ? dl2 : 0.0;
    double l1p = posp(e.ev1), l2p = posp(e.ev2);
    double gap = e.ev1 - e.ev2;
    double alpha = gap > 1e-12 * scale ? (c * t1 - s * t0) / gap : 0.0;
    double rot = alpha * (l1p - l2p);
    o11 = dl1p * c * c + dl2p * s * s - 2.0 * rot * s * c;
    o22 = dl1p * s * s + dl2p * c * c + 2.0 * rot * s * c;
    o12 = (dl1p - dl2p) * c * s + rot * (c * c - s * s);
}

__device__ __forceinline__ void sigplus2(double lam, double mu, double tre, const Eig& e,
                                         double& p11, double& p22, double& p12) {
    double trp = posp(tre), l1p = posp(e.ev1), l2p = posp(e.ev2);
    double c = e.c, s = e.s;
    p11 = lam * trp + 2.0 * mu * (l1p * c * c + l2p * s * s);
    p22 = lam * trp + 2.0 * mu * (l1p * s * s + l2p * c * c);
    p12 = 2.0 * mu * (l1p - l2p) * c * s;
}

__device__ __forceinline__ double esplus2(double lam, double mu, double tre, const Eig& e) {
    double trp = posp(tre), l1p = posp(e.ev1), l2p = posp(e.ev2);
    return 0.5 * lam * trp * trp + mu * (l1p * l1p + l2p * l2p);
}

// g dsigma+ + dsigma- and sigma+ : de (src/_kernels.py:102-123), with the
// eigensystem of the state strain precomputed (it does not depend on de).
__device__ __forceinline__ void dsig_split_pre(double lam, double mu, double g, const Eig& e,
                                               double scale, double tre, double d11,
                                               double d22, double d12, double& s11,
                                               double& s22, double& s12, double& spde) {
    double o11, o22, o12;
    dpos2(e, scale, d11, d22, d12, o11, o22, o12);
    double trde = d11 + d22;
    double tt = tre < 0.0 ? 0.0 : trde;
    double dp11 = lam * tt + 2.0 * mu * o11;
    double dp22 = lam * tt + 2.0 * mu * o22;
    double dp12 = 2.0 * mu * o12;
    double f11 = lam * trde + 2.0 * mu * d11;
    double f22 = lam * trde + 2.0 * mu * d22;
    double f12 = 2.0 * mu * d12;
    double sp11, sp22, sp12;
    sigplus2(lam, mu, tre, e, sp11, sp22, sp12);
    spde = sp11 * d11 + sp22 * d22 + 2.0 * sp12 * d12;
    s11 = g * dp11 + (f11 - dp11);
    s22 = g * dp22 + (f22 - dp22);
    s12 = g * dp12 + (f12 - dp12);
}

__device__ __forceinline__ void dsig_split(double lam, double mu, double g, double e11,
                                           double e22, double e12, double d11, double d22,
                                           double d12, double& s11, double& s22, double& s12,
                                           double& spde) {
    dsig_split_pre(lam, mu, g, eig2(e11, e22, e12), scale2(e11, e22, e12), e11 + e22, d11, d22,
                   d12, s11, s22, s12, spde);
}

// isotropic ("none") tangent and sigma(e):de (src/_kernels.py:645-653)
__device__ __forceinline__ void dsig_none(double lam, double mu, double g, double e11,
                                          double e22, double e12, double d11, double d22,
                                          double d12, double& s11, double& s22, double& s12,
                                          double& spde) {
    double trde = d11 + d22;
    s11 = g * (lam * trde + 2.0 * mu * d11);
    s22 = g * (lam * trde + 2.0 * mu * d22);
    s12 = g * 2.0 * mu * d12;
    double tre = e11 + e22;
    spde = (lam * tre + 2.0 * mu * e11) * d11 + (lam * tre + 2.0 * mu * e22) * d22 +
           2.0 * (2.0 * mu * e12) * d12;
}

template <bool MIEHE>
__device__ __forceinline__ void dsig(double lam, double mu, double g, double e11, double e22,
                                     double e12, double d11, double d22, double d12,
                                     double& s11, double& s22, double& s12, double& spde) {
    if (MIEHE)
        dsig_split(lam, mu, g, e11, e22, e12, d11, d22, d12, s11, s22, s12, spde);
    else
        dsig_none(lam, mu, g, e11, e22, e12, d11, d22, d12, s11, s22, s12, spde);
}

// ------------------------------------------------- 1-D sum factorisation
// Same contraction order as the reference (src/_kernels.py:257-304).

template <int N1>
__device__ __forceinline__ void fwd_x(const double (&M)[NMAX][NMAX], const double (&c)[N1][N1],
                                      double (&t)[N1][N1]) {
#pragma unroll
    for (int b = 0; b < N1; ++b)
#pragma unroll
        for (int iq = 0; iq < N1; ++iq) {
            double acc = M[iq][0] * c[b][0];
#pragma unroll
            for (int a = 1; a < N1; ++a) acc = fma(M[iq][a], c[b][a], acc);
            t[b][iq] = acc;
        }
}

template <int N1>
__device__ __forceinline__ void fwd_y(const double (&M)[NMAX][NMAX], const double (&t)[N1][N1],
                                      double (&o)[N1][N1]) {
#pragma unroll
    for (int jq = 0; jq < N1; ++jq)
#pragma unroll
        for (int iq = 0; iq < N1; ++iq) {
            double acc = M[jq][0] * t[0][iq];
#pragma unroll
            for (int b = 1; b < N1; ++b) acc = fma(M[jq][b], t[b][iq], acc);
            o[jq][iq] = acc;
        }
}

template <int N1>
__device__ __forceinline__ void bwd_y(const double (&M)[NMAX][NMAX], const double (&f)[N1][N1],
                                      double (&t)[N1][N1]) {
#pragma unroll
    for (int b = 0; b < N1; ++b)
#pragma unroll
        for (int iq = 0; iq < N1; ++iq) {
            double acc = M[0][b] * f[0][iq];
#pragma unroll
            for (int jq = 1; jq < N1; ++jq) acc = fma(M[jq][b], f[jq][iq], acc);
            t[b][iq] = acc;
        }
}

template <int N1>
__device__ __forceinline__ void bwd_x_add(const double (&M)[NMAX][NMAX],
                                          const double (&t)[N1][N1], double (&r)[N1][N1]) {
#pragma unroll
    for (int b = 0; b < N1; ++b)
#pragma unroll
        for (int a = 0; a < N1; ++a) {
            double acc = r[b][a];
#pragma unroll
            for (int iq = 0; iq < N1; ++iq) acc = fma(M[iq][a], t[b][iq], acc);
            r[b][a] = acc;
        }
}

// Miehe tangent with the state eigensystem given as (m, +-r, c, s):
// ev1 = m + r, ev2 = m - r, tr e = 2m (bit-identical to src/_kernels.py:28-33),
// the gap test of _dpos2s (line 66) is the sign of the stored r.
struct MieheQ {
    Eig e;
    double tre;
    bool gap_ok;
};
__device__ __forceinline__ MieheQ miehe_q(double m, double rs, double c, double s) {
    MieheQ q;
    const double r = fabs(rs);
    q.e.ev1 = m + r;
    q.e.ev2 = m - r;
    q.e.c = c;
    q.e.s = s;
    q.tre = 2.0 * m;
    q.gap_ok = rs > 0.0;
    return q;
}

__device__ __forceinline__ void miehe_dsig(const Material& M, double g, const MieheQ& q,
                                           double d11, double d22, double d12, double& s11,
                                           double& s22, double& s12, double& spde) {
    const double c = q.e.c, s = q.e.s, lam = M.lam, mu = M.mu;
    const double t0 = d11 * c + d12 * s;
    const double t1 = d12 * c + d22 * s;
    const double dl1 = c * t0 + s * t1;
    const double dl2 = s * s * d11 - 2.0 * s * c * d12 + c * c * d22;
    const double dl1p = q.e.ev1 >= 0.0 ? dl1 : 0.0;
    const double dl2p = q.e.ev2 >= 0.0 ? dl2 : 0.0;
    const double l1p = posp(q.e.ev1), l2p = posp(q.e.ev2);
    const double alpha = q.gap_ok ? (c * t1 - s * t0) / (q.e.ev1 - q.e.ev2) : 0.0;
    const double rot = alpha * (l1p - l2p);
    const double o11 = dl1p * c * c + dl2p * s * s - 2.0 * rot * s * c;
    const double o22 = dl1p * s * s + dl2p * c * c + 2.0 * rot * s * c;
    const double o12 = (dl1p - dl2p) * c * s + rot * (c * c - s * s);
    const double trde = d11 + d22;
    const double tt = q.tre < 0.0 ? 0.0 : trde;
    const double dp11 = lam * tt + 2.0 * mu * o11;
    const double dp22 = lam * tt + 2.0 * mu * o22;
    const double dp12 = 2.0 * mu * o12;
    const double f11 = lam * trde + 2.0 * mu * d11;
    const double f22 = lam * trde + 2.0 * mu * d22;
    const double f12 = 2.0 * mu * d12;
    double sp11, sp22, sp12;
    sigplus2(lam, mu, q.tre, q.e, sp11, sp22, sp12);
    spde = sp11 * d11 + sp22 * d22 + 2.0 * sp12 * d12;
    s11 = g * dp11 + (f11 - dp11);
    s22 = g * dp22 + (f22 - dp22);
    s12 = g * dp12 + (f12 - dp12);
}

}  // namespace pff
