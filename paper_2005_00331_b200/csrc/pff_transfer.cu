// pff_transfer.cu -- level transfers and state injection on device.
//
// Prolongation restates src/multigrid.py:44-112 without the CSR: each fine
// scalar row is owned by the first fine cell (ascending cell index) that
// references it, which in closed form is the lowest containing cell in each
// direction -- except the upper slit copies (n_grid + i), owned by the upper
// cell row.  The row is the coarse Lagrange basis of the owner's parent cell
// evaluated through the child embedding; weights with |w| <= 1e-14 are
// dropped exactly as the reference does (multigrid.py:81-83).
// Restriction is the exact transpose (multigrid.py:114-120): one thread per
// coarse cell gathers the fine rows that cell owns and adds the weighted sums
// into the cell's coarse nodes, in four colour passes (cx, cy parities) so
// no two threads touch a coarse node at once -- no atomics, fixed order.
// Injection restates src/mesh_hierarchy.py:316-338 / pff_operator.py:380-400.
#include <cstdlib>

#include "pff_internal.cuh"

namespace pff {

namespace {

// One thread per owned fine node.  The embedding table sits in shared memory
// (runtime-indexed), the owner cell comes from 32-bit index math when the
// level has < 2^31 nodes, and the per-direction weights are read once; the
// sums keep the (my, mx) order and the |w| > 1e-14 filter of the reference's
// CSR rows, so the result is the same bit for bit.
template <int P, bool SMALL, bool WINC = false>
__global__ void __launch_bounds__(256)
k_prolong(Mesh mf, Win wf, Mesh mc, Win wc, Embed E, const double* __restrict__ xc,
          double* __restrict__ yf, const uint8_t* __restrict__ flags_f, int add_masked) {
    constexpr int N1 = P + 1;
    __shared__ double Es[2][N1][N1];
    for (int k = threadIdx.x; k < 2 * N1 * N1; k += blockDim.x) {
        const int c = k / (N1 * N1), r = (k / N1) % N1, m = k % N1;
        Es[c][r][m] = E.E[c][r][m];
    }
    __syncthreads();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= wf.n_owned(mf)) return;
    const int64_t gg = wf.owned_global(mf, t);
    // fine grid position and owner (the lowest containing fine cell; the
    // upper slit copies belong to the upper cell row)
    int64_t i, j;
    const bool dup = gg >= mf.n_grid;
    if (dup) {
        i = gg - mf.n_grid;
        j = mf.i_mid;
    } else if (SMALL) {
        const uint32_t g32 = (uint32_t)gg, w32 = (uint32_t)mf.np1;
        const uint32_t jj = g32 / w32;
        j = jj;
        i = g32 - jj * w32;
    } else {
        j = gg / mf.np1;
        i = gg - j * mf.np1;
    }
    auto lowest = [&](int64_t k) -> int {
        const int64_t c = k > 0 ? (k - 1) / P : 0;
        return (int)(c < mf.nside ? c : mf.nside - 1);
    };
    const int fx = lowest(i);
    const int fy = dup ? (mf.nside >> 1) : lowest(j);
    const int a = (int)(i - (int64_t)P * fx), b = (int)(j - (int64_t)P * fy);
    const int ccx = fx >> 1, ccy = fy >> 1, chx = fx & 1, chy = fy & 1;
    const int64_t g = wf.loc(mf, gg);     // local index of the fine node
    // the add form's flag and z loads first: their latency overlaps the gathers
    uint8_t f = 0;
    double z0 = 0.0, z1 = 0.0, z2 = 0.0;
    if (add_masked) {
        f = flags_f[g];
        z0 = yf[g];
        z1 = yf[wf.n + g];
        z2 = yf[2 * wf.n + g];
    }
    double wx[N1], wy[N1];
#pragma unroll
    for (int m = 0; m < N1; ++m) {
        wx[m] = Es[chx][a][m];
        wy[m] = Es[chy][b][m];
    }
    double acc[3] = {0.0, 0.0, 0.0};
    // WINC: the coarse vector is a slab window's local vector (global id -> local)
    const int64_t cn = WINC ? wc.n : mc.n;
    const double* xk[3] = {xc, xc + cn, xc + 2 * cn};
    // coarse node of (mx, my) in the parent cell (Mesh::node; 32-bit when SMALL:
    // the coarse level is a quarter of the fine one)
    const bool cup = mc.level >= 1 && ccy >= (mc.nside >> 1);
    auto cnode = [&](int mx, int my) -> int64_t {
        int64_t gc;
        if (SMALL) {
            const int jc = P * ccy + my, ic = P * ccx + mx;
            const int imc = (int)mc.i_mid;
            gc = cup && jc == imc && ic < imc ? (int)mc.n_grid + ic : jc * (int)mc.np1 + ic;
        } else {
            gc = mc.node(ccx, ccy, mx, my);
        }
        return WINC ? wc.loc(mc, gc) : gc;
    };
    // branch-free: a dropped weight (|w| <= 1e-14, multigrid.py:81-83) is an exact
    // zero, and fma(0, x, acc) == acc for finite x -- the same sums without the
    // per-lane divergent filter (neighbouring fine nodes have different patterns)
#pragma unroll
    for (int my = 0; my < N1; ++my)
#pragma unroll
        for (int mx = 0; mx < N1; ++mx) {
            const double w0 = wy[my] * wx[mx];
            const double w = fabs(w0) > 1e-14 ? w0 : 0.0;
            const int64_t c = cnode(mx, my);
#pragma unroll
            for (int k = 0; k < 3; ++k) acc[k] = fma(w, xk[k][c], acc[k]);
        }
    if (add_masked) {
        // z += where(cons, 0, P zc)  (src/multigrid.py:340-342)
        if (!(f & F_DIR)) {
            yf[g] = z0 + acc[0];
            yf[wf.n + g] = z1 + acc[1];
        }
        if (!(f & F_ACT)) yf[2 * wf.n + g] = z2 + acc[2];
    } else {
#pragma unroll
        for (int k = 0; k < 3; ++k) yf[k * wf.n + g] = acc[k];
    }
}

struct CellColour {
    int c, hx, hy, cy0;
};

inline CellColour make_colour(int colour, int ns, int row_lo, int row_hi) {
    CellColour k;
    k.c = colour;
    k.hx = (ns - (colour & 1) + 1) >> 1;
    k.cy0 = row_lo + (((row_lo & 1) != (colour >> 1)) ? 1 : 0);
    k.hy = row_hi > k.cy0 ? (row_hi - k.cy0 + 1) >> 1 : 0;
    return k;
}

__device__ __forceinline__ bool owned_fine(const Mesh& mf, const Win& wf, int64_t gg) {
    if (gg >= mf.n_grid) return wf.owns_dup != 0;
    const int64_t j = gg / mf.np1;
    return j >= wf.own_lo && j < wf.own_hi;
}

// ev == nullptr: colour pass (col) adding into xc; otherwise one pass over the
// cells of rows [col.cy0, col.cy0 + col.hy) writing element vectors ev[k][cell][my][mx]
// (ev rows are relative to the coarse level's first q-point row crow0; nce =
// the cells held there -- the whole mesh: 0 and n_cells)
template <int P, bool STAGED = false>
__global__ void __launch_bounds__(128)
k_restrict(Mesh mf, Win wf, Mesh mc, Embed E, const double* __restrict__ yf, double* xc,
           CellColour col, double* __restrict__ ev, int crow0 = 0, int64_t nce = 0) {
    constexpr bool staged = STAGED;
    constexpr int N1 = P + 1, QQ = N1 * N1;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t ntot = (int64_t)col.hx * col.hy;
    const bool valid = t < ntot;
    if (!valid && !(ev && staged)) return;   // the staged form's threads all reach its barriers
    int ccx = 0, ccy = 0;
    if (!valid) {
    } else if (ev) {
        ccx = (int)(t % col.hx);
        ccy = col.cy0 + (int)(t / col.hx);
    } else {
        ccx = (col.c & 1) + 2 * (int)(t % col.hx);
        ccy = col.cy0 + 2 * (int)(t / col.hx);
    }
    double acc[3][N1][N1] = {};
    if (valid) {
    // The fine nodes of the coarse cell's block, each once: rows 0..p of the
    // lower child, then rows 0..p of the upper child, whose row 0 repeats the
    // lower child's row p except where the slit splits it (coarse level 0).
    // First-visit ownership (as k_prolong's owner) in closed form: the cell owns a
    // block node unless it lies on the block's left column (ccx > 0) or
    // bottom row (ccy > 0) -- those belong to the neighbour -- except the
    // upper slit copies, owned by the upper cell row.  The owner's child and
    // local index are the enumeration's own (fcx - 2 ccx, la, fcy - 2 ccy, lb).
#pragma unroll
    for (int fb = 0; fb <= 2 * P + 1; ++fb) {
        const bool up = fb > P;
        const int chy = up ? 1 : 0, lb = up ? fb - P - 1 : fb;
        const int fcy = 2 * ccy + chy;
        const int64_t j = (int64_t)P * fcy + lb;   // fine grid row
#pragma unroll
        for (int fa = 0; fa <= 2 * P; ++fa) {
            const int chx = fa > P ? 1 : 0, la = fa - P * chx;
            const int fcx = 2 * ccx + chx;
            const int64_t i = (int64_t)P * fcx + la;
            const bool dup = mf.level >= 1 && fcy >= (mf.nside >> 1) && j == mf.i_mid && i < mf.i_mid;
            if (up && lb == 0 && !dup) continue;                 // repeats the lower child's row p
            if (fa == 0 && ccx > 0) continue;                    // left neighbour's column
            if (fb == 0 && ccy > 0 && !dup) continue;            // lower neighbour's row
            // window ownership of the fine node
            if (dup ? !wf.owns_dup : (j < wf.own_lo || j >= wf.own_hi)) continue;
            const int64_t gg = dup ? mf.n_grid + i : j * mf.np1 + i;
            const int64_t g = wf.loc(mf, gg);
            const double v0 = yf[g], v1 = yf[wf.n + g], v2 = yf[2 * wf.n + g];
#pragma unroll
            for (int my = 0; my < N1; ++my)
#pragma unroll
                for (int mx = 0; mx < N1; ++mx) {
                    const double w = E.E[chy][lb][my] * E.E[chx][la][mx];
                    if (fabs(w) > 1e-14) {
                        acc[0][my][mx] += w * v0;
                        acc[1][my][mx] += w * v1;
                        acc[2][my][mx] += w * v2;
                    }
                }
        }
    }
    }
    if (ev && !staged) {
        const int64_t nc = nce, cell = (int64_t)(ccy - crow0) * mc.nside + ccx;
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int my = 0; my < N1; ++my)
#pragma unroll
                for (int mx = 0; mx < N1; ++mx)
                    ev[((int64_t)k * nc + cell) * QQ + my * N1 + mx] = acc[k][my][mx];
        return;
    }
    if constexpr (STAGED) {
        // the block's cells are consecutive (t = (ccy - cy0) * nside + ccx over
        // whole cell rows): stage one component's element vectors in shared
        // memory and store them as one contiguous run -- coalesced, instead of
        // every store instruction touching 32 sectors QQ doubles apart
        __shared__ double sh[128 * QQ];
        const int64_t nc = nce, tb = (int64_t)blockIdx.x * blockDim.x;
        const int nb = (int)(ntot - tb < 128 ? ntot - tb : 128);
        const int64_t cell0 = (int64_t)(col.cy0 - crow0) * mc.nside + tb;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            if (valid) {
#pragma unroll
                for (int my = 0; my < N1; ++my)
#pragma unroll
                    for (int mx = 0; mx < N1; ++mx) sh[threadIdx.x * QQ + my * N1 + mx] = acc[k][my][mx];
            }
            __syncthreads();
            double* o = ev + ((int64_t)k * nc + cell0) * QQ;
            for (int e = threadIdx.x; e < nb * QQ; e += 128) o[e] = sh[e];
            __syncthreads();
        }
        return;
    }
#pragma unroll
    for (int my = 0; my < N1; ++my)
#pragma unroll
        for (int mx = 0; mx < N1; ++mx) {
            const int64_t c = mc.node(ccx, ccy, mx, my);
#pragma unroll
            for (int k = 0; k < 3; ++k) xc[k * mc.n + c] += acc[k][my][mx];
        }
}

// Element-vector form of the restriction, one thread per (coarse cell,
// component k, coarse basis row my): the thread accumulates acc[mx] =
// ev[k][cell][my][mx] over the cell's owned fine nodes in the same (fb, fa)
// order as k_restrict's per-cell accumulator, so the element vectors are the
// same bit for bit with 3 (p+1) times the parallelism (the small levels are
// latency-bound on that per-thread chain).  Threads of a warp share (k, my):
// uniform weights and branches.
template <int P>
__global__ void __launch_bounds__(128)
k_restrict_ev(Mesh mf, Win wf, Mesh mc, Embed E, const double* __restrict__ yf, int cy0, int hy,
              double* __restrict__ ev, int crow0, int64_t nce) {
    constexpr int N1 = P + 1, QQ = N1 * N1;
    const int64_t ncw = (int64_t)mc.nside * hy;          // coarse cells of the window rows
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ncw * 3 * N1) return;
    const int km = (int)(t / ncw);                         // k * N1 + my
    const int64_t cw = t - (int64_t)km * ncw;
    const int k = km / N1, my = km % N1;
    const int ccx = (int)(cw % mc.nside), ccy = cy0 + (int)(cw / mc.nside);
    const double* yk = yf + (int64_t)k * wf.n;
    double acc[N1] = {};
#pragma unroll
    for (int fb = 0; fb <= 2 * P + 1; ++fb) {
        const bool up = fb > P;
        const int chy = up ? 1 : 0, lb = up ? fb - P - 1 : fb;
        const int fcy = 2 * ccy + chy;
        const int64_t j = (int64_t)P * fcy + lb;
        const double ey = E.E[chy][lb][my];
#pragma unroll
        for (int fa = 0; fa <= 2 * P; ++fa) {
            const int chx = fa > P ? 1 : 0, la = fa - P * chx;
            const int fcx = 2 * ccx + chx;
            const int64_t i = (int64_t)P * fcx + la;
            const bool dup = mf.level >= 1 && fcy >= (mf.nside >> 1) && j == mf.i_mid && i < mf.i_mid;
            if (up && lb == 0 && !dup) continue;
            if (fa == 0 && ccx > 0) continue;
            if (fb == 0 && ccy > 0 && !dup) continue;
            if (dup ? !wf.owns_dup : (j < wf.own_lo || j >= wf.own_hi)) continue;
            const int64_t gg = dup ? mf.n_grid + i : j * mf.np1 + i;
            const double v = yk[wf.loc(mf, gg)];
#pragma unroll
            for (int mx = 0; mx < N1; ++mx) {
                const double w = ey * E.E[chx][la][mx];
                if (fabs(w) > 1e-14) acc[mx] += w * v;
            }
        }
    }
    const int64_t nc = nce, cell = (int64_t)(ccy - crow0) * mc.nside + ccx;
    double* o = ev + ((int64_t)k * nc + cell) * QQ + my * N1;
#pragma unroll
    for (int mx = 0; mx < N1; ++mx) o[mx] = acc[mx];
}

// coarse node gather of the element vectors (cell rows [lo, hi)), zeroing the
// constrained rows when asked (src/multigrid.py:338)
// (WINC: over the local nodes of a slab window wc -- its ghost rows included;
// the top ghost row receives this rank's partial sums for the neighbour above)
template <int P, bool WINC = false>
__global__ void k_restrict_gather(Mesh mc, Win wc, const double* __restrict__ ev,
                                  double* __restrict__ xc, int lo, int hi,
                                  const uint8_t* __restrict__ flags, int zero_cons) {
    constexpr int N1 = P + 1, QQ = N1 * N1;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nloc = WINC ? wc.n : mc.n;
    if (t >= nloc) return;
    const int64_t c = WINC ? (t < wc.dupl ? t + wc.shift : mc.n_grid + (t - wc.dupl)) : t;
    const int64_t nc = WINC ? wc.ncell : mc.n_cells();
    const int crow0 = WINC ? wc.row0 : 0;
    double acc[3] = {0.0, 0.0, 0.0};
    node_cells_p<P>(mc, c, lo, hi, [&](int cx, int cy, int a, int b) {
        const int64_t cell = (int64_t)(cy - crow0) * mc.nside + cx;
#pragma unroll
        for (int k = 0; k < 3; ++k) acc[k] += ev[((int64_t)k * nc + cell) * QQ + b * N1 + a];
    });
    if (zero_cons) {
        const uint8_t f = flags[t];
        if (f & F_DIR) acc[0] = acc[1] = 0.0;
        if (f & F_ACT) acc[2] = 0.0;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) xc[k * nloc + t] = acc[k];
}

// Q2 restriction as a direct per-coarse-node gather (whole-mesh levels): r_c =
// P^T r_f with the tensor-product weights of the reference's P rows
// (src/multigrid.py:44-120; first-visited-cell owners, |w| > 1e-14 kept) read
// off the 1-D embedding table: coarse even index 2k gathers fine offsets
// -3, -1, 0, +1, +3 (weights E[0][1][2], E[1][1][2], E[1][2][2] -- E[0][0][0]
// at k = 0 --, E[0][1][0], E[1][1][0]), odd index 2k+1 offsets -1, 0, +1
// (E[0][1][1], E[0][2][1], E[1][1][1]).  Every other 1-D weight of a Q2 row is
// at most ~1e-16 and dropped by the reference's filter, so filtering the
// product equals filtering the factors.  The slit: the coarse row i_mid's
// lower copies (grid ids) gather the fine rows below and the fine slit row's
// lower copies, its upper copies the fine rows above and the fine upper copies
// (owned by the upper cell row, weight E[0][0][0]); the tip and the right half
// gather both.  No element vectors, no scratch, write-once; the fine residual
// was just written and is mostly L2-resident.
// the (up to) five 1-D taps of coarse index I: fixed slots, zero weight when
// absent (compile-time indexed: registers, no local memory)
struct W1 {
    int off[5];
    double w[5];
};

__device__ __forceinline__ W1 taps_q2(const Embed& E, int I, int np1) {
    W1 t;
    const bool even = (I & 1) == 0;
    const int o[5] = {-3, -1, 0, 1, 3};
    const double we[5] = {E.E[0][1][2], E.E[1][1][2], I > 0 ? E.E[1][2][2] : E.E[0][0][0],
                          E.E[0][1][0], E.E[1][1][0]};
    const double wo[5] = {0.0, E.E[0][1][1], E.E[0][2][1], E.E[1][1][1], 0.0};
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int i = 2 * I + o[k];
        double w = even ? we[k] : wo[k];
        if (i < 0 || i >= np1 || !(fabs(w) > 1e-14)) w = 0.0;
        t.off[k] = (i < 0 || i >= np1) ? 0 : o[k];   // absent taps read a valid index
        t.w[k] = w;
    }
    return t;
}

__global__ void __launch_bounds__(256)
k_restrict_direct_q2(Mesh mf, Mesh mc, Embed E, const double* __restrict__ yf,
                     double* __restrict__ xc, const uint8_t* __restrict__ flags_c, int zero_cons) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= mc.n) return;
    const int np1c = (int)mc.np1, np1f = (int)mf.np1, imc = (int)mc.i_mid, imf = (int)mf.i_mid;
    int I, J, kind;   // kind 0: grid node, 1: lower copy (row i_mid, left), 2: upper copy
    if (c < mc.n_grid) {
        J = (int)(c / np1c);
        I = (int)(c - (int64_t)J * np1c);
        kind = (mc.level >= 1 && J == imc && I < imc) ? 1 : 0;
    } else {
        I = (int)(c - mc.n_grid);
        J = imc;
        kind = 2;
    }
    const W1 tx = taps_q2(E, I, np1f), ty = taps_q2(E, J, np1f);
    const bool slit = mc.level >= 1 && J == imc;
    double acc[3] = {0.0, 0.0, 0.0};
    const double* y1 = yf + mf.n;
    const double* y2 = yf + 2 * mf.n;
#pragma unroll
    for (int b = 0; b < 5; ++b) {
        const int oy = ty.off[b];
        const double wy = ty.w[b];
        if (wy == 0.0) continue;
        const int j = 2 * J + oy;
        // which copies of fine row j this coarse node sees
        if (slit && kind == 1 && oy > 0) continue;   // lower copy: rows below + the slit row
        if (slit && kind == 2 && oy < 0) continue;   // upper copy: rows above + the slit row
        const bool slit_row = slit && oy == 0;
        double rx[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int a = 0; a < 5; ++a) {
            const double w = tx.w[a];
            if (w == 0.0) continue;
            const int i = 2 * I + tx.off[a];
            if (slit_row && i < imf) {
                // the fine slit row left of the tip: lower copy (grid id, owned by the
                // lower cell: the row's weight wy) and upper copy (n_grid + i, owned by
                // the upper cell at t = 0: weight E[0][0][0])
                const int64_t gl = (int64_t)j * np1f + i, gu = mf.n_grid + i;
                if (kind != 2) {
                    rx[0] = fma(w * wy, yf[gl], rx[0]);
                    rx[1] = fma(w * wy, y1[gl], rx[1]);
                    rx[2] = fma(w * wy, y2[gl], rx[2]);
                }
                if (kind != 1) {
                    const double wu = w * E.E[0][0][0];
                    rx[0] = fma(wu, yf[gu], rx[0]);
                    rx[1] = fma(wu, y1[gu], rx[1]);
                    rx[2] = fma(wu, y2[gu], rx[2]);
                }
                continue;
            }
            const int64_t g = (int64_t)j * np1f + i;
            const double ww = w * wy;
            rx[0] = fma(ww, yf[g], rx[0]);
            rx[1] = fma(ww, y1[g], rx[1]);
            rx[2] = fma(ww, y2[g], rx[2]);
        }
        acc[0] += rx[0];
        acc[1] += rx[1];
        acc[2] += rx[2];
    }
    if (zero_cons) {
        const uint8_t f = flags_c[c];
        if (f & F_DIR) acc[0] = acc[1] = 0.0;
        if (f & F_ACT) acc[2] = 0.0;
    }
    xc[c] = acc[0];
    xc[mc.n + c] = acc[1];
    xc[2 * mc.n + c] = acc[2];
}

// rc[cons_c] = 0 (src/multigrid.py:338)
__global__ void k_zero_cons3(int64_t n, const uint8_t* __restrict__ flags, double* x) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint8_t f = flags[i];
    if (f & F_DIR) {
        x[i] = 0.0;
        x[n + i] = 0.0;
    }
    if (f & F_ACT) x[2 * n + i] = 0.0;
}

__device__ __forceinline__ int64_t inject_src(const Mesh& mf, const Mesh& mc, int64_t c) {
    if (c < mc.n_grid) {
        int64_t I = c % mc.np1, J = c / mc.np1;
        return (2 * J) * mf.np1 + 2 * I;
    }
    return mf.n_grid + 2 * (c - mc.n_grid);
}

__global__ void k_inject_f64(Mesh mf, Mesh mc, const double* __restrict__ src, double* dst,
                             int ncomp) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= mc.n) return;
    int64_t f = inject_src(mf, mc, c);
    for (int k = 0; k < ncomp; ++k) dst[k * mc.n + c] = src[k * mf.n + f];
}

__global__ void k_inject_u8(Mesh mf, Mesh mc, const uint8_t* __restrict__ src, uint8_t* dst) {
    int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= mc.n) return;
    dst[c] = src[inject_src(mf, mc, c)];
}

inline unsigned blocks(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

cudaError_t launch_prolongate(const Level& F, const Level& C, const double* xc, double* yf,
                              int add_masked, cudaStream_t s) {
    if (F.mesh.p != C.mesh.p || F.mesh.level != C.mesh.level + 1) return cudaErrorInvalidValue;
    // a windowed coarse level (slab-to-slab V-cycle) holds the coarse cells of
    // the fine window's owned rows: local coarse indices
    if (C.windowed() && (!F.windowed() || F.cy_begin() != 2 * C.cy_begin() ||
                         F.cy_end() != 2 * C.cy_end()))
        return cudaErrorInvalidValue;
    const Win wf = F.win(), wc = C.win();
    const int64_t nf = wf.n_owned(F.mesh);
    const bool small = F.mesh.n < (int64_t(1) << 31);
#define PFF_PROLONG(PP)                                                                          \
    (C.windowed() ? (small ? k_prolong<PP, true, true> : k_prolong<PP, false, true>)             \
                  : (small ? k_prolong<PP, true> : k_prolong<PP, false>))<<<blocks(nf), 256, 0, s>>>( \
        F.mesh, wf, C.mesh, wc, F.embed, xc, yf, F.flags, add_masked)
    switch (F.mesh.p) {
        case 1: PFF_PROLONG(1); break;
        case 2: PFF_PROLONG(2); break;
        case 3: PFF_PROLONG(3); break;
        case 4: PFF_PROLONG(4); break;
        default: return cudaErrorInvalidValue;
    }
#undef PFF_PROLONG
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_restrict(const Level& F, const Level& C, const double* yf, double* xc,
                            int zero_cons, cudaStream_t s) {
    if (F.mesh.p != C.mesh.p || F.mesh.level != C.mesh.level + 1) return cudaErrorInvalidValue;
    const bool winc = C.windowed();
    if (winc && (!F.windowed() || F.cy_begin() != 2 * C.cy_begin() || F.cy_end() != 2 * C.cy_end() ||
                 !C.qcache))
        return cudaErrorInvalidValue;
    const Win wf = F.win(), wc = C.win();
    // coarse cell rows owning the window's fine rows (fine cell rows cyb-1 .. cye);
    // a coarse window holds exactly rows [q_row0, cy_end) of them
    const int nsc = C.mesh.nside;
    const int cyb = F.cy_begin(), cye = F.cy_end();
    const int lo = cyb > 0 ? (cyb - 1) / 2 : 0;
    const int hi = winc ? C.cy_end() : ((cye / 2 + 1) < nsc ? cye / 2 + 1 : nsc);
    const int crow0 = winc ? C.q_row0() : 0;
    const int64_t nce = winc ? C.local_cells() : C.mesh.n_cells();
    if (zero_cons && !C.flags) return cudaErrorInvalidValue;
    static const bool direct_ok = [] {
        const char* e = getenv("PFF_RESTRICT_DIRECT");
        return !(e && e[0] == '0');
    }();
    if (direct_ok && F.mesh.p == 2 && !F.windowed() && !winc && F.mesh.level >= 2) {
        k_restrict_direct_q2<<<blocks(C.mesh.n), 256, 0, s>>>(F.mesh, C.mesh, F.embed, yf, xc,
                                                             C.flags, zero_cons);
        count_launches(1);
        return cudaGetLastError();
    }
    if (C.qcache) {   // element vectors in the coarse level's scratch + node gather
        CellColour all;
        all.c = 0;
        all.hx = nsc;
        all.cy0 = lo;
        all.hy = hi - lo;
        double* ev = C.ev();
        // measured: the per-(cell, component, row) split wins on the latency-bound
        // small levels, the per-cell kernel on the large ones (fewer loads)
        const bool split = nsc <= 64;
        // element vectors staged through shared memory for coalesced stores:
        // measured faster from 256^2 coarse cells (1024^2 fine: 74 -> 65 us),
        // slower below (the block barriers outweigh the store savings)
        const bool staged = nsc >= 256;
        const int64_t nthr = (int64_t)all.hx * all.hy * (split ? 3 * (F.mesh.p + 1) : 1);
        const unsigned g = (unsigned)((nthr + 127) / 128);
        if (!split) {
            switch (F.mesh.p) {
                case 1: (staged ? k_restrict<1, true> : k_restrict<1, false>)<<<g, 128, 0, s>>>(F.mesh, wf, C.mesh, F.embed, yf, xc, all, ev, crow0, nce); break;
                case 2: (staged ? k_restrict<2, true> : k_restrict<2, false>)<<<g, 128, 0, s>>>(F.mesh, wf, C.mesh, F.embed, yf, xc, all, ev, crow0, nce); break;
                case 3: (staged ? k_restrict<3, true> : k_restrict<3, false>)<<<g, 128, 0, s>>>(F.mesh, wf, C.mesh, F.embed, yf, xc, all, ev, crow0, nce); break;
                case 4: (staged ? k_restrict<4, true> : k_restrict<4, false>)<<<g, 128, 0, s>>>(F.mesh, wf, C.mesh, F.embed, yf, xc, all, ev, crow0, nce); break;
                default: return cudaErrorInvalidValue;
            }
        } else switch (F.mesh.p) {
            case 1: k_restrict_ev<1><<<g, 128, 0, s>>>(F.mesh, wf, C.mesh, F.embed, yf, all.cy0, all.hy, ev, crow0, nce); break;
            case 2: k_restrict_ev<2><<<g, 128, 0, s>>>(F.mesh, wf, C.mesh, F.embed, yf, all.cy0, all.hy, ev, crow0, nce); break;
            case 3: k_restrict_ev<3><<<g, 128, 0, s>>>(F.mesh, wf, C.mesh, F.embed, yf, all.cy0, all.hy, ev, crow0, nce); break;
            case 4: k_restrict_ev<4><<<g, 128, 0, s>>>(F.mesh, wf, C.mesh, F.embed, yf, all.cy0, all.hy, ev, crow0, nce); break;
            default: return cudaErrorInvalidValue;
        }
        const unsigned gn = blocks(winc ? wc.n : C.mesh.n);
#define PFF_GATHER(PP)                                                                           \
    (winc ? k_restrict_gather<PP, true> : k_restrict_gather<PP>)<<<gn, 256, 0, s>>>(             \
        C.mesh, wc, ev, xc, lo, hi, C.flags, zero_cons)
        switch (F.mesh.p) {
            case 1: PFF_GATHER(1); break;
            case 2: PFF_GATHER(2); break;
            case 3: PFF_GATHER(3); break;
            case 4: PFF_GATHER(4); break;
        }
#undef PFF_GATHER
        count_launches(2);
        return cudaGetLastError();
    }
    // no scratch bound to the coarse level: four colour passes into xc
    cudaMemsetAsync(xc, 0, sizeof(double) * 3 * C.mesh.n, s);
    count_launches(1);
    for (int c = 0; c < 4; ++c) {
        const CellColour col = make_colour(c, nsc, lo, hi);
        const int64_t cnt = (int64_t)col.hx * col.hy;
        if (cnt <= 0) continue;
        const unsigned g = (unsigned)((cnt + 127) / 128);
        switch (F.mesh.p) {
            case 1: k_restrict<1><<<g, 128, 0, s>>>(F.mesh, wf, C.mesh, F.embed, yf, xc, col, nullptr); break;
            case 2: k_restrict<2><<<g, 128, 0, s>>>(F.mesh, wf, C.mesh, F.embed, yf, xc, col, nullptr); break;
            case 3: k_restrict<3><<<g, 128, 0, s>>>(F.mesh, wf, C.mesh, F.embed, yf, xc, col, nullptr); break;
            case 4: k_restrict<4><<<g, 128, 0, s>>>(F.mesh, wf, C.mesh, F.embed, yf, xc, col, nullptr); break;
            default: return cudaErrorInvalidValue;
        }
        count_launches(1);
    }
    if (zero_cons) {
        k_zero_cons3<<<blocks(C.mesh.n), 256, 0, s>>>(C.mesh.n, C.flags, xc);
        count_launches(1);
    }
    return cudaGetLastError();
}

cudaError_t launch_inject_f64(const Level& F, const Level& C, const double* src, double* dst,
                              int ncomp, cudaStream_t s) {
    if (F.mesh.p != C.mesh.p || F.mesh.level != C.mesh.level + 1) return cudaErrorInvalidValue;
    k_inject_f64<<<blocks(C.mesh.n), 256, 0, s>>>(F.mesh, C.mesh, src, dst, ncomp);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_inject_u8(const Level& F, const Level& C, const uint8_t* src, uint8_t* dst,
                             cudaStream_t s) {
    if (F.mesh.p != C.mesh.p || F.mesh.level != C.mesh.level + 1) return cudaErrorInvalidValue;
    k_inject_u8<<<blocks(C.mesh.n), 256, 0, s>>>(F.mesh, C.mesh, src, dst);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace pff
