// pff_sweep4.cu -- write-once Q4 operator kernel (configs[2]: 512^2 Q4 cells).
//
// Same operator as k_apply_coop<4> (src/_kernels.py:555-693 with the identity
// rows/columns of src/pff_operator.py:262-302), without the element-vector
// round trip and the per-node gather pass:
//
//  * one warp owns a strip of 6 cells (5 own + the left neighbour, recomputed)
//    and sweeps upward over a chunk of cell rows; p+1 = 5 lanes per cell: lane
//    t owns node row b = t in the x-passes and Gauss column iq = t in the
//    y-passes and the q-point physics, the transposes go through shared memory
//    (the cooperative layout of k_apply_coop);
//  * every 1-D contraction uses the even-odd decomposition of the mirror-
//    symmetric 5-point basis (N[4-q][4-a] = N[q][a], D[4-q][4-a] = -D[q][a],
//    checked on the host): per 5x5 contraction 13 multiplies instead of 25;
//  * each lane stages its own node row (5 nodes x the used direction fields +
//    the flag words) one cell row ahead into shared memory by cp.async (no
//    registers held across the row step); the cell row's weighted tangent block
//    ([array][jq][cell][iq], the reference's cache_tensors quantities with the
//    quadrature weight folded in, as the Q2 tiles) arrives in shared memory by
//    one TMA bulk copy (cp.async.bulk + mbarrier) issued as soon as the previous
//    block is consumed;
//  * a cell's right node column goes to the next cell's lanes by shuffle, its
//    top node row is carried (lane 4 -> lane 0 of the cell) into the next cell
//    row; every dst entry is written exactly once (deterministic), identity
//    rows and the optional fused rhs - G src applied at the store;
//  * the slit: the upper cell row reads the upper copies (n_grid + i), lower
//    and upper copies are stored apart.
#include <cstdlib>

#include "pff_bulk.cuh"
#include "pff_internal.cuh"

namespace pff {

namespace {
using namespace bulk;

constexpr int P4 = 4, N4 = 5;
constexpr int C4 = 6;                 // cells per strip (cell 0: the left neighbour)
constexpr int OWN4 = C4 - 1;          // own cells per strip
constexpr int QA4 = N4 * N4 * C4;     // doubles per tangent array of a block (150)
// per-cell stride of the transpose buffer: 6 arrays x 5 x 5 doubles padded to
// 153 (= 5 mod 16 in 8-byte banks) -- the row-major writes/reads of the
// x-passes are conflict-free, the column accesses of the y-passes 2-way
constexpr int BXS = 153;

enum Field4 { GX = 0, GY, GP, NF4 };

template <int MODE, bool MIEHE>
struct Use4 {
    static constexpr bool ux = MODE != MODE_PHIPHI;
    static constexpr bool ph = MODE != MODE_UU;
    static constexpr bool DO_UU = MODE == MODE_FULL || MODE == MODE_UU;
    static constexpr bool DO_PP = MODE != MODE_UU;
    static constexpr bool DO_COUP = MODE == MODE_FULL || MODE == MODE_PHIROW;
    // tangent block arrays: none [g w][cw0 cw1 cw2][pc]; Miehe the eigen-frame form
    // of the Q2 sweep (pff_sweep.cu): [+-g w][+-gamma w][c2][s2][q1/2][q2/2][pc]
    static constexpr int NT = MIEHE ? 4 : 1;
    static constexpr int NCW = MIEHE ? 2 : 3;
    static constexpr int NQT = NT + NCW + 1;
    static constexpr int Q0 = MODE == MODE_PHIROW ? (MIEHE ? 2 : NT)
                              : MODE == MODE_PHIPHI ? NQT - 1 : 0;
    static constexpr int NQ = MODE == MODE_FULL ? NQT : MODE == MODE_UU ? NT
                              : MODE == MODE_PHIROW ? NQT - Q0 : 1;
    static constexpr int QC2 = 2 - Q0;     // local index of c2 (Miehe, not PHIPHI)
    static constexpr int QCW = NT - Q0;
    static constexpr int QPC = NQ - 1;
    static constexpr bool used(int f) { return (f == GX || f == GY) ? ux : ph; }
    static constexpr int slot(int f) {
        int s = 0;
        for (int g = 0; g < f; ++g) s += used(g) ? 1 : 0;
        return s;
    }
    static constexpr int NF = slot(NF4);
};

template <int NF, int NQ>
struct __align__(16) Smem4 {
    double q[NQ * QA4];                    // the cell row's tangent block (TMA destination)
    double bx[C4 * BXS];                   // x-pass results / backward-y results per cell
    double st[2][NF * 5][32];              // staged node rows (cp.async), [buffer][field x node][lane]
    unsigned fw[2][3][32];                 // staged flag words
    unsigned fo[2][32];                    // byte offsets of the flag words
    unsigned long long bar;
};

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// even-odd coefficients of the 5-point basis, prepared on the host; Dh = D / h
// (h = 2^-l: exact).  Pairs q in {0, 1} with 4-q, a in {0, 1} with 4-a.
struct EO4 {
    double NE[2][2], NO[2][2];   // (N[q][a] +- N[q][4-a]) / 2
    double DE[2][2], DO[2][2];   // (Dh[q][a] +- Dh[q][4-a]) / 2
    double NM[2], DM[2];         // N[q][2], Dh[q][2]
    double N2E[2], N22, D2O[2];  // (N[2][a] + N[2][4-a]) / 2, N[2][2], (Dh[2][a] - Dh[2][4-a]) / 2
    double w[5];                 // Gauss weights
    double cg;                   // gc eps h^2
    double h2;                   // h^2 (the Miehe eigen-frame form weights its constants)
    double lam, mu2;
    double lamh, muh, mu;        // lam / 2, mu / 2, mu
};

// v[q] = sum_a N[q][a] u[a], d[q] = sum_a Dh[q][a] u[a], q = 0..4
template <bool V, bool D>
__device__ __forceinline__ void fwd5(const EO4& K, const double (&u)[5], double (&v)[5],
                                     double (&d)[5]) {
    const double e0 = u[0] + u[4], e1 = u[1] + u[3];
    const double o0 = u[0] - u[4], o1 = u[1] - u[3], mid = u[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        if (V) {
            const double ev = fma(K.NE[q][0], e0, fma(K.NE[q][1], e1, K.NM[q] * mid));
            const double ov = fma(K.NO[q][0], o0, K.NO[q][1] * o1);
            v[q] = ev + ov;
            v[4 - q] = ev - ov;
        }
        if (D) {
            const double ed = fma(K.DE[q][0], e0, fma(K.DE[q][1], e1, K.DM[q] * mid));
            const double od = fma(K.DO[q][0], o0, K.DO[q][1] * o1);
            d[q] = ed + od;
            d[4 - q] = od - ed;
        }
    }
    if (V) v[2] = fma(K.N2E[0], e0, fma(K.N2E[1], e1, K.N22 * mid));
    if (D) d[2] = fma(K.D2O[0], o0, K.D2O[1] * o1);
}

// r[a] = sum_q N[q][a] t1[q] + Dh[q][a] t2[q], a = 0..4 (the transposed pass)
template <bool T1, bool T2>
__device__ __forceinline__ void bwd5(const EO4& K, const double (&t1)[5], const double (&t2)[5],
                                     double (&r)[5]) {
    double te0 = 0.0, te1 = 0.0, to0 = 0.0, to1 = 0.0, tm = 0.0;
    double se0 = 0.0, se1 = 0.0, so0 = 0.0, so1 = 0.0, sm = 0.0;
    if (T1) {
        te0 = t1[0] + t1[4]; te1 = t1[1] + t1[3];
        to0 = t1[0] - t1[4]; to1 = t1[1] - t1[3]; tm = t1[2];
    }
    if (T2) {
        se0 = t2[0] + t2[4]; se1 = t2[1] + t2[3];
        so0 = t2[0] - t2[4]; so1 = t2[1] - t2[3]; sm = t2[2];
    }
#pragma unroll
    for (int a = 0; a < 2; ++a) {
        double E = 0.0, O = 0.0;
        if (T1) {
            E = fma(K.NE[0][a], te0, fma(K.NE[1][a], te1, K.N2E[a] * tm));
            O = fma(K.NO[0][a], to0, K.NO[1][a] * to1);
        }
        if (T2) {
            E = fma(K.DE[0][a], so0, fma(K.DE[1][a], so1, E));
            O = fma(K.DO[0][a], se0, fma(K.DO[1][a], se1, fma(K.D2O[a], sm, O)));
        }
        r[a] = E + O;
        r[4 - a] = E - O;
    }
    double mid = 0.0;
    if (T1) mid = fma(K.NM[0], te0, fma(K.NM[1], te1, K.N22 * tm));
    if (T2) mid = fma(K.DM[0], so0, fma(K.DM[1], so1, mid));
    r[2] = mid;
}

struct Sweep4Args {
    EO4 K;
    Mesh m;
    const double* fld[NF4];   // ux uy phi of the direction
    const uint8_t* flags;
    const double* qtile;      // strip-tiled tangent cache
    int64_t qblock;           // doubles per (strip, cell row) block
    double* dst[3];
    const double* src_out[3];
    const double* rhs[3];
    int n_strips, rows_per_chunk, n_items;
};

// ------------------------------------------------------------- tiled refresh
// Per (strip, cell row) block [array][jq][cell c][iq] from the generic q-point
// cache (k_refresh): the direction-independent part of the reference's
// cache_tensors form (src/_kernels.py:517-548), weight w_jq w_iq h^2 folded in --
// none: g w, the coupling vector (3), pc; Miehe: the 7-array eigen-frame form of
// the Q2 sweep (pff_sweep.cu: +-g w, +-gamma w, cos / sin of twice the
// eigen-angle, two eigen-frame coupling coefficients, pc).
template <bool MIEHE>
__global__ void k_refresh_tile4(Mesh m, Shape S, Material M, const double* __restrict__ qc,
                                double* __restrict__ qt, int n_strips, int64_t qblock) {
    const int ns = m.nside;
    const int64_t total = (int64_t)n_strips * ns * QA4;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= total) return;
    const int within = (int)(t % QA4);
    const int64_t blk = t / QA4;                    // strip * ns + cy
    const int strip = (int)(blk / ns), cy = (int)(blk - (int64_t)strip * ns);
    const int jq = within / 30, r = within - 30 * jq, c = r / 5, iq = r - 5 * c;
    const int cx = strip * OWN4 - 1 + c;
    double* o = qt + blk * qblock + within;
    constexpr int NQT = MIEHE ? 7 : 5;
    if (cx < 0 || cx >= ns) {
#pragma unroll
        for (int a = 0; a < NQT; ++a) o[a * QA4] = 0.0;
        return;
    }
    const int64_t nc = m.n_cells(), fs = 25 * nc;
    const int64_t cell = (int64_t)cy * ns + cx;
    const double* q = qc + (int64_t)(jq * N4 + iq) * nc + cell;
    const double h = m.h, wv = S.w[jq] * S.w[iq] * h * h;
    const double e11 = q[0], e22 = q[fs], e12 = q[2 * fs], g = q[3 * fs], dg = q[4 * fs];
    const double tre = e11 + e22;
    if (!MIEHE) {
        o[0] = wv * g;
        o[QA4] = wv * dg * (M.lam * tre + 2.0 * M.mu * e11);
        o[2 * QA4] = wv * dg * (M.lam * tre + 2.0 * M.mu * e22);
        o[3 * QA4] = wv * dg * 2.0 * (2.0 * M.mu * e12);
        o[4 * QA4] = wv * q[5 * fs];
        return;
    }
    // the eigen-frame split tangent of k_refresh_tiled (pff_sweep.cu), with the weight
    // folded into g and gamma (the kernel rebuilds w_jq w_iq h^2 for the undegraded terms)
    const Eig e = eig2(e11, e22, e12);
    const bool gap_ok = (e.ev1 - e.ev2) > 1e-12 * scale2(e11, e22, e12);
    const double l1p = posp(e.ev1), l2p = posp(e.ev2), trp = posp(tre);
    const double beta = gap_ok ? (l1p - l2p) / (e.ev1 - e.ev2) : 0.0;
    const double gam = fma(g, beta, 1.0 - beta);
    const bool htr = !(tre < 0.0), h1 = e.ev1 >= 0.0, h2 = e.ev2 >= 0.0;
    const bool bb = htr ? h2 : h1;
    o[0] = htr ? wv * g : -(wv * g);
    o[QA4] = bb ? wv * gam : -(wv * gam);
    o[2 * QA4] = e.c * e.c - e.s * e.s;
    o[3 * QA4] = 2.0 * e.c * e.s;
    o[4 * QA4] = 0.5 * wv * dg * (M.lam * trp + 2.0 * M.mu * l1p);
    o[5 * QA4] = 0.5 * wv * dg * (M.lam * trp + 2.0 * M.mu * l2p);
    o[6 * QA4] = wv * q[5 * fs];
}

// ------------------------------------------------------------------ the kernel
template <int MODE, bool MIEHE, bool FUSED>
__global__ void __launch_bounds__(32) k_sweep_q4(const Sweep4Args A) {
    using U = Use4<MODE, MIEHE>;
    constexpr int NF = U::NF, NQ = U::NQ;
    constexpr int NC = U::DO_UU ? (U::DO_PP ? 3 : 2) : 1;   // output components
    using Smem = Smem4<NF, NQ>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& W = *reinterpret_cast<Smem*>(smem_raw);
    const int lane = threadIdx.x;
    const int c = lane / N4, t = lane - N4 * c;   // cell of the strip, node row / Gauss column
    const bool lane_on = c < C4;                  // lanes 30, 31 idle
    const int cs = lane_on ? c : 0;

    const Mesh& m = A.m;
    const EO4& K = A.K;
    const int ns = m.nside, np1i = (int)m.np1, imid = (int)m.i_mid, ngrid = (int)m.n_grid;
    const int half = ns >> 1;
    // this lane's Gauss weight (iq = t) times gc eps h^2
    const double wt = t == 0 ? K.w[0] : t == 1 ? K.w[1] : t == 2 ? K.w[2] : t == 3 ? K.w[3] : K.w[4];
    const double cgl = K.cg * wt;
    const double wth2 = wt * K.h2;   // w_iq h^2

    if (lane == 0) {
        mbar_init(&W.bar);
        fence_mbar_init();
    }
    __syncwarp();
    unsigned qphase = 0u;

    for (int item = blockIdx.x; item < A.n_items; item += gridDim.x) {
        const int strip = item % A.n_strips, chunk = item / A.n_strips;
        const int c0 = chunk * A.rows_per_chunk;
        const int c1 = min(ns, c0 + A.rows_per_chunk);
        const int cstart = c0 > 0 ? c0 - 1 : 0;
        const int cx = strip * OWN4 - 1 + cs;
        const bool active = lane_on && cx >= 0 && cx < ns;
        const bool owner = active && c > 0;

        auto issue_qblock = [&](int cy) {
            PFF_DCHECK(cy >= 0 && cy < ns);
            const double* src = A.qtile + ((int64_t)strip * ns + cy) * A.qblock + U::Q0 * QA4;
            mbar_expect_tx(&W.bar, (unsigned)(NQ * QA4 * 8));
            bulk_g2s(W.q, src, (unsigned)(NQ * QA4 * 8), &W.bar);
        };
        // this lane's node row b = t of cell row cy into staging buffer sb: the used
        // fields' 5 nodes (8-byte cp.async each) and the flag bytes (the two 4-byte
        // words around nodes 0..3 and the word of node 4 -- node 4 is not contiguous
        // on the crack tip); the closed-form numbering reads the upper slit copies
        // on the upper cell row.  Asynchronous: no registers held across the step.
        auto stage_row = [&](int cy, int sb) {
            if (active) {
                const int g0 = (int)m.node(cx, cy, 0, t), g4 = (int)m.node(cx, cy, 4, t);
#pragma unroll
                for (int a = 0; a < 5; ++a) {
                    const int gid = a == 4 ? g4 : (int)m.node(cx, cy, a, t);
#pragma unroll
                    for (int k = 0; k < NF4; ++k)
                        if (U::used(k)) cp_async8(&W.st[sb][U::slot(k) * 5 + a][lane], A.fld[k] + gid);
                }
                const uint8_t* w0 = A.flags + (g0 & ~3);
                // (flag buffers carry 8 bytes of padding: LinearizationState._sync_flags)
                PFF_DCHECK((g0 & ~3) + 8 <= (int)m.n + 8 && (g4 & ~3) + 4 <= (int)m.n + 8);
                cp_async4(&W.fw[sb][0][lane], w0);
                cp_async4(&W.fw[sb][1][lane], w0 + 4);
                cp_async4(&W.fw[sb][2][lane], A.flags + (g4 & ~3));
                W.fo[sb][lane] = (g0 & 3) | ((g4 & 3) << 2);
            }
            cp_async_commit();
        };
        // Dirichlet bits 0..4, active bits 5..9 of staged row sb
        auto bits = [&](int sb) -> unsigned {
            const unsigned lo = W.fw[sb][0][lane], hi = W.fw[sb][1][lane], tip = W.fw[sb][2][lane];
            const unsigned o = W.fo[sb][lane];
            const unsigned long long win = ((unsigned long long)hi << 32) | lo;
            unsigned fl = 0u;
#pragma unroll
            for (int a = 0; a < 5; ++a) {
                const unsigned fb = a == 4 ? (tip >> (8 * (o >> 2))) & 0xffu
                                           : (unsigned)(win >> (8 * ((o & 3) + a))) & 0xffu;
                fl |= (fb & F_DIR ? 1u : 0u) << a;
                fl |= (fb & F_ACT ? 1u : 0u) << (a + 5);
            }
            return fl;
        };
        auto staged = [&](int sb, int f, int a) -> double {
            PFF_DCHECK(U::used(f) && sb >= 0 && sb < 2 && a >= 0 && a < 5);
            return W.st[sb][U::slot(f) * 5 + a][lane];
        };

        stage_row(cstart, 0);
        if (lane == 0) issue_qblock(cstart);
        double carry[3][5];   // lane t = 0: the cell row below's top-row contributions
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int a = 0; a < 5; ++a) carry[k][a] = 0.0;
        for (int cy = cstart; cy < c1; ++cy) {
            const int sb = (cy - cstart) & 1;
            const bool more = cy + 1 < c1;
            if (more) {
                stage_row(cy + 1, sb ^ 1);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            const bool own_row = cy >= c0;
            const int jb = 4 * cy;
            const bool slit_row = m.level >= 1 && cy == half;

            // ---- phase 1: node row b = t of cell c, x-pass per field ---------------
            const unsigned fcur = active ? bits(sb) : 0u;
            if (active) {
                double u[5], xv[5], xd[5];
#pragma unroll
                for (int f = 0; f < NF4; ++f) {
                    if (!U::used(f)) continue;
                    const unsigned mk = fcur >> (f == GP ? 5 : 0);
#pragma unroll
                    for (int a = 0; a < 5; ++a) u[a] = ((mk >> a) & 1u) ? 0.0 : staged(sb, f, a);
                    fwd5<true, true>(K, u, xv, xd);
                    double* B0 = W.bx + cs * BXS + (2 * f) * 25 + t * 5;
#pragma unroll
                    for (int iq = 0; iq < 5; ++iq) {
                        B0[iq] = xv[iq];
                        B0[25 + iq] = xd[iq];
                    }
                }
            }
            mbar_wait(&W.bar, qphase);
            qphase ^= 1u;
            __syncwarp();

            // ---- phase 2: Gauss column iq = t: y-pass, physics, backward y-pass ----
            double T[6][5];
            if (active) {
                auto col = [&](int arr, double (&X)[5]) {
#pragma unroll
                    for (int b = 0; b < 5; ++b) X[b] = W.bx[cs * BXS + arr * 25 + b * 5 + t];
                };
                double d11[5], d22[5], d12[5], pv[5], pgx[5], pgy[5], tmp[5], X[5];
                if (U::ux) {
                    col(1, X);                         // D_x u  -> N_y: e11
                    fwd5<true, false>(K, X, d11, tmp);
                    col(2, X);                         // N_x v  -> D_y: e22
                    fwd5<false, true>(K, X, tmp, d22);
                    col(0, X);                         // N_x u  -> D_y
                    fwd5<false, true>(K, X, tmp, d12);
                    col(3, X);                         // D_x v  -> N_y
                    fwd5<true, false>(K, X, pv, tmp);
                    // d12 = (u_y + v_x) / 2; the Miehe form takes twice that
#pragma unroll
                    for (int q = 0; q < 5; ++q)
                        d12[q] = MIEHE ? d12[q] + pv[q] : 0.5 * (d12[q] + pv[q]);
                }
                if (U::ph) {
                    col(4, X);                         // N_x phi -> value, D_y
                    fwd5<true, true>(K, X, pv, pgy);
                    col(5, X);                         // D_x phi -> N_y
                    fwd5<true, false>(K, X, pgx, tmp);
                }
                const double* qb = W.q;
                auto qv = [&](int arr, int jq) -> double { return qb[arr * QA4 + jq * 30 + lane]; };
                double S11[5], S12[5], S22[5], FV[5], FGX[5], FGY[5];
#pragma unroll
                for (int jq = 0; jq < 5; ++jq) {
                    double s11 = 0.0, s22 = 0.0, s12 = 0.0, fv = 0.0, fgx = 0.0, fgy = 0.0;
                    if (U::DO_PP) fv = qv(U::QPC, jq) * pv[jq];
                    if (MIEHE && U::ux) {
                        // eigen-frame form (pff_sweep.cu): d12[] holds 2 d12 here
                        const double c2 = qv(U::QC2, jq), s2 = qv(U::QC2 + 1, jq);
                        const double pd = d11[jq] + d22[jq], qd = d11[jq] - d22[jq];
                        const double u2 = fma(c2, qd, s2 * d12[jq]);
                        const double e1 = pd + u2, e2 = pd - u2;
                        if (U::DO_COUP)
                            fv = fma(qv(U::QCW, jq), e1, fma(qv(U::QCW + 1, jq), e2, fv));
                        if (U::DO_UU) {
                            const double v2 = fma(c2, d12[jq], -(s2 * qd));
                            const double gs = qv(0, jq), ms = qv(1, jq);
                            const bool ha = __double2hiint(gs) >= 0, hb = __double2hiint(ms) >= 0;
                            const double wq = K.w[jq] * wth2;           // w_jq w_iq h^2
                            const double gw = fabs(gs), gamw = fabs(ms);
                            const double ca = ha ? gw : wq;             // H_tr
                            const double c1 = (ha || hb) ? gw : wq;     // H_1
                            const double cb = (ha && hb) ? gw : wq;     // H_2
                            const double at = (K.lamh * ca) * pd;
                            const double hs1 = fma(K.muh * c1, e1, at);
                            const double hs2 = fma(K.muh * cb, e2, at);
                            const double s3 = (K.mu * gamw) * v2;
                            const double hp = hs1 + hs2, hd = hs1 - hs2;
                            const double tt = fma(c2, hd, -(s2 * s3));
                            s11 = hp + tt;
                            s22 = hp - tt;
                            s12 = fma(s2, hd, c2 * s3);
                        }
                    } else if (U::ux) {
                        if (U::DO_UU) {
                            const double gw = qv(0, jq);
                            const double lt = K.lam * (d11[jq] + d22[jq]);
                            s11 = gw * fma(K.mu2, d11[jq], lt);
                            s22 = gw * fma(K.mu2, d22[jq], lt);
                            s12 = (gw * K.mu2) * d12[jq];
                        }
                        if (U::DO_COUP)
                            fv = fma(qv(U::QCW, jq), d11[jq],
                                     fma(qv(U::QCW + 1, jq), d22[jq], fma(qv(U::QCW + 2, jq), d12[jq], fv)));
                    }
                    S11[jq] = s11;
                    S12[jq] = s12;
                    S22[jq] = s22;
                    if (U::DO_PP) {
                        const double cw = cgl * K.w[jq];
                        fgx = cw * pgx[jq];
                        fgy = cw * pgy[jq];
                    }
                    FV[jq] = fv;
                    FGX[jq] = fgx;
                    FGY[jq] = fgy;
                }
                // backward y-pass: T1 (against N) / T2 (against Dh) per output array
                if (U::DO_UU) {
                    bwd5<true, false>(K, S11, S11, T[0]);   // u: against Dh in x
                    bwd5<false, true>(K, S12, S12, T[1]);   // u: against N in x
                    bwd5<true, false>(K, S12, S12, T[2]);   // v: against Dh in x
                    bwd5<false, true>(K, S22, S22, T[3]);   // v: against N in x
                }
                if (U::DO_PP) {
                    bwd5<true, true>(K, FV, FGY, T[4]);     // phi: against N in x
                    bwd5<true, false>(K, FGX, FGX, T[5]);   // phi: against Dh in x
                }
            }
            __syncwarp();
            // the tangent block is consumed: stage the next cell row's (its latency
            // hides behind the backward x-pass, the stores and the next x-pass)
            if (more && lane == 0) {
                fence_proxy_async();
                issue_qblock(cy + 1);
            }
            if (active) {
#pragma unroll
                for (int A6 = 0; A6 < 6; ++A6) {
                    if ((A6 < 4 && !U::DO_UU) || (A6 >= 4 && !U::DO_PP)) continue;
#pragma unroll
                    for (int b = 0; b < 5; ++b) W.bx[cs * BXS + A6 * 25 + b * 5 + t] = T[A6][b];
                }
            }
            __syncwarp();

            // ---- phase 3: node row b = t, backward x-pass ------------------------------
            double r[3][5];
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
                for (int a = 0; a < 5; ++a) r[k][a] = 0.0;
            if (active) {
                double R1[5], R2[5];
                auto rowv = [&](int arr, double (&Y)[5]) {
#pragma unroll
                    for (int iq = 0; iq < 5; ++iq) Y[iq] = W.bx[cs * BXS + arr * 25 + t * 5 + iq];
                };
                if (U::DO_UU) {
                    rowv(1, R1); rowv(0, R2);
                    bwd5<true, true>(K, R1, R2, r[0]);
                    rowv(3, R1); rowv(2, R2);
                    bwd5<true, true>(K, R1, R2, r[1]);
                }
                if (U::DO_PP) {
                    rowv(4, R1); rowv(5, R2);
                    bwd5<true, true>(K, R1, R2, r[2]);
                }
            }

            // ---- combine: left cell's right column, carried bottom row; store ----------
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double left = __shfl_up_sync(0xffffffffu, r[k][4], N4);
                if (c > 0) r[k][0] += left;
            }
            double up[3][5];   // lane (c, 0) receives lane (c, 4)'s top-row values
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
                for (int a = 0; a < 5; ++a) up[k][a] = __shfl_down_sync(0xffffffffu, r[k][a], 4);
            const int na = cx == ns - 1 ? 5 : 4;
            // identity rows (src/pff_operator.py:262-302) take the raw src value: this
            // lane's own staged node row, or (the slit's lower copies) a global load
            auto store = [&](int gid, const double (&v)[3], bool cdir, bool cact, int a) {
#pragma unroll
                for (int o = 0; o < NC; ++o) {
                    const int pc = U::DO_UU ? o : 2;
                    const int F = pc == 0 ? GX : pc == 1 ? GY : GP;
                    const bool cons = pc < 2 ? cdir : cact;
                    double x = v[pc];
                    if (cons) x = a >= 0 ? staged(sb, F, a) : A.src_out[o][gid];
                    if (FUSED) x = A.rhs[o][gid] - x;
                    A.dst[o][gid] = x;
                }
            };
            if (own_row && owner && (t < 4 || cy == ns - 1)) {   // t = 4: top boundary row
                const int j = jb + t;
#pragma unroll
                for (int a = 0; a < 5; ++a) {
                    if (a >= na) break;
                    const int gc = 4 * cx + a;
                    const bool cdir = (fcur >> a) & 1u, cact = (fcur >> (a + 5)) & 1u;
                    double v[3];
                    if (t == 0 && slit_row && gc < imid) {
                        // lower copy: the cell row below only; upper copy: this row
#pragma unroll
                        for (int k = 0; k < 3; ++k) v[k] = carry[k][a];
                        const uint8_t fl = A.flags[j * np1i + gc];
                        store(j * np1i + gc, v, fl & F_DIR, fl & F_ACT, -1);
#pragma unroll
                        for (int k = 0; k < 3; ++k) v[k] = r[k][a];
                        store(ngrid + gc, v, cdir, cact, a);
                        continue;
                    }
#pragma unroll
                    for (int k = 0; k < 3; ++k) v[k] = r[k][a] + (t == 0 ? carry[k][a] : 0.0);
                    store(j * np1i + gc, v, cdir, cact, a);
                }
            }
#pragma unroll
            for (int k = 0; k < 3; ++k)
#pragma unroll
                for (int a = 0; a < 5; ++a) carry[k][a] = up[k][a];
            __syncwarp();
        }
        __syncwarp();
    }
}

struct LaunchCfg4 {
    bool init = false;
    int blocks_per_sm = 0;
};

template <int MODE, bool MIEHE, bool FUSED>
cudaError_t launch_mode4(Sweep4Args& a, cudaStream_t s) {
    using U = Use4<MODE, MIEHE>;
    const size_t shm = sizeof(Smem4<U::NF, U::NQ>);
    auto k = k_sweep_q4<MODE, MIEHE, FUSED>;
    static LaunchCfg4 cfg;
    static int n_sm = 0;
    if (!cfg.init) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cfg.blocks_per_sm, k, 32, shm);
        if (e != cudaSuccess) return e;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        if (cfg.blocks_per_sm < 1) cfg.blocks_per_sm = 1;
        cfg.init = true;
    }
    const int ns = a.m.nside;
    const int slots = cfg.blocks_per_sm * n_sm;
    int chunks = slots / a.n_strips;   // one full wave
    if (chunks < 1) chunks = 1;
    if (chunks > ns) chunks = ns;
    int rows = (ns + chunks - 1) / chunks;
    if (const char* e = getenv("PFF_SWEEP4_ROWS")) {
        const int r = atoi(e);
        if (r > 0) rows = r < ns ? r : ns;
    }
    a.rows_per_chunk = rows;
    a.n_items = a.n_strips * ((ns + rows - 1) / rows);
    const int grid = a.n_items < slots ? a.n_items : slots;
    k<<<grid, 32, shm, s>>>(a);
    count_launches(1);
    return cudaGetLastError();
}

template <bool MIEHE, bool FUSED>
cudaError_t launch_split4(int mode, Sweep4Args& a, cudaStream_t s) {
    switch (mode) {
        case MODE_FULL: return launch_mode4<MODE_FULL, MIEHE, FUSED>(a, s);
        case MODE_UU: return launch_mode4<MODE_UU, MIEHE, FUSED>(a, s);
        case MODE_PHIPHI: return launch_mode4<MODE_PHIPHI, MIEHE, FUSED>(a, s);
        case MODE_PHIROW: return launch_mode4<MODE_PHIROW, MIEHE, FUSED>(a, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_refresh_tile4(const Level& L, cudaStream_t s) {
    const Mesh& m = L.mesh;
    const int64_t total = (int64_t)L.n_strips4() * m.nside * QA4;
    const unsigned grid = (unsigned)((total + 255) / 256);
    if (L.miehe)
        k_refresh_tile4<true><<<grid, 256, 0, s>>>(m, L.shape, L.mat, L.qcache, L.qtile4(),
                                                   L.n_strips4(), L.tile4_block());
    else
        k_refresh_tile4<false><<<grid, 256, 0, s>>>(m, L.shape, L.mat, L.qcache, L.qtile4(),
                                                    L.n_strips4(), L.tile4_block());
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_sweep4_apply(const Level& L, int mode, const double* src, double* dst,
                                const double* rhs, cudaStream_t s, bool* handled) {
    *handled = false;
    if (!L.sweep4_ok()) return cudaSuccess;
    const Mesh& m = L.mesh;
    const int64_t n = m.n;
    Sweep4Args a;
    a.m = m;
    {
        EO4& K = a.K;
        const Shape& S = L.shape;
        const double ih = 1.0 / m.h;
        double Dh[5][5];
        for (int q = 0; q < 5; ++q)
            for (int b = 0; b < 5; ++b) Dh[q][b] = S.D[q][b] * ih;
        for (int q = 0; q < 2; ++q) {
            for (int b = 0; b < 2; ++b) {
                K.NE[q][b] = 0.5 * (S.N[q][b] + S.N[q][4 - b]);
                K.NO[q][b] = 0.5 * (S.N[q][b] - S.N[q][4 - b]);
                K.DE[q][b] = 0.5 * (Dh[q][b] + Dh[q][4 - b]);
                K.DO[q][b] = 0.5 * (Dh[q][b] - Dh[q][4 - b]);
            }
            K.NM[q] = S.N[q][2];
            K.DM[q] = Dh[q][2];
        }
        for (int b = 0; b < 2; ++b) {
            K.N2E[b] = 0.5 * (S.N[2][b] + S.N[2][4 - b]);
            K.D2O[b] = 0.5 * (Dh[2][b] - Dh[2][4 - b]);
        }
        K.N22 = S.N[2][2];
        for (int q = 0; q < 5; ++q) K.w[q] = S.w[q];
        K.cg = L.mat.gc * L.mat.eps * (m.h * m.h);
        K.lam = L.mat.lam;
        K.mu2 = 2.0 * L.mat.mu;
        K.h2 = m.h * m.h;
        K.lamh = 0.5 * L.mat.lam;
        K.muh = 0.5 * L.mat.mu;
        K.mu = L.mat.mu;
    }
    for (int f = 0; f < NF4; ++f) a.fld[f] = nullptr;
    switch (mode) {
        case MODE_FULL:
        case MODE_PHIROW: a.fld[GX] = src; a.fld[GY] = src + n; a.fld[GP] = src + 2 * n; break;
        case MODE_UU: a.fld[GX] = src; a.fld[GY] = src + n; break;
        case MODE_PHIPHI: a.fld[GP] = src; break;
        default: return cudaErrorInvalidValue;
    }
    a.flags = L.flags;
    a.qtile = L.qtile4();
    a.qblock = L.tile4_block();
    for (int c = 0; c < 3; ++c) { a.dst[c] = nullptr; a.src_out[c] = nullptr; a.rhs[c] = nullptr; }
    if (mode == MODE_FULL || mode == MODE_UU) {
        const int nc = mode == MODE_FULL ? 3 : 2;
        for (int c = 0; c < nc; ++c) {
            a.dst[c] = dst + c * n;
            a.src_out[c] = src + c * n;
            a.rhs[c] = rhs ? rhs + c * n : nullptr;
        }
    } else {
        a.dst[0] = dst;
        a.src_out[0] = mode == MODE_PHIROW ? src + 2 * n : src;
        a.rhs[0] = rhs;
    }
    a.n_strips = L.n_strips4();
    *handled = true;
    if (L.miehe)
        return rhs ? launch_split4<true, true>(mode, a, s) : launch_split4<true, false>(mode, a, s);
    return rhs ? launch_split4<false, true>(mode, a, s) : launch_split4<false, false>(mode, a, s);
}

}  // namespace pff
