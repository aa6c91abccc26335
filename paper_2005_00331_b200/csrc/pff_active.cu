// pff_active.cu -- device side of the primal-dual active-set loop
// (src/active_set_solver.py:60-163).
//
//  * k_lumped_mass: row sums of the scalar phi mass matrix
//    (src/_kernels.py:828-843).  The reference scatter-adds cell by cell; here
//    every node GATHERS the terms of the cells that contain it, in increasing
//    cell index, with the reference's rounding ((col_a col_b) h) h and no FMA
//    contraction -- so the result is bitwise the reference's, and deterministic.
//  * k_active_set: the complementarity test of determine_active_set
//    (src/active_set_solver.py:72-82), the obstacle reset of freshly activated
//    dofs (lines 113-118) and the counters the loop needs (|A|, moved dofs,
//    changes against the previous set) in one pass.
#include "pff_internal.cuh"

namespace pff {

namespace {

__global__ void k_lumped_mass(Mesh m, Shape S, Win w, double* __restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= w.n) return;
    const int p = m.p, ns = m.nside, q = p + 1;
    // col[a] = sum_iq w_iq N[iq][a], accumulated in the reference's order
    double col[NMAX];
    for (int a = 0; a <= p; ++a) {
        double acc = 0.0;
        for (int iq = 0; iq < q; ++iq) acc = __dadd_rn(acc, __dmul_rn(S.w[iq], S.N[iq][a]));
        col[a] = acc;
    }
    const int64_t cnt = w.dupl;                 // local grid entries
    int64_t i, j;
    int cy_lo = 0, cy_hi = ns;                  // admissible cell rows
    if (t < cnt) {
        const int64_t g = t + w.shift;
        j = g / m.np1;
        i = g - j * m.np1;
        if (m.level >= 1 && j == m.i_mid && i < m.i_mid) cy_hi = ns >> 1;   // lower copy
    } else {
        i = t - cnt;                            // upper slit copy n_grid + i
        j = m.i_mid;
        cy_lo = ns >> 1;
    }
    double acc = 0.0;
    const double h = m.h;
    // cells containing the node, increasing cell index (cy major, cx minor)
    const int cy0 = (int)((j - 1) / p) < 0 ? 0 : (int)((j - 1) / p);
    for (int cy = cy0; cy <= (int)(j / p) && cy < ns; ++cy) {
        const int64_t b = j - (int64_t)cy * p;
        if (cy < cy_lo || cy >= cy_hi || b < 0 || b > p) continue;
        const int cx0 = (int)((i - 1) / p) < 0 ? 0 : (int)((i - 1) / p);
        for (int cx = cx0; cx <= (int)(i / p) && cx < ns; ++cx) {
            const int64_t a = i - (int64_t)cx * p;
            if (a < 0 || a > p) continue;
            acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(__dmul_rn(col[a], col[b]), h), h));
        }
    }
    out[t] = acc;
}

__global__ void k_active_set(int64_t n, const double* __restrict__ rhs_phi,
                             double* __restrict__ phi, const double* __restrict__ phi_old,
                             const double* __restrict__ m_diag, double c,
                             const uint8_t* __restrict__ prev, uint8_t* __restrict__ active,
                             unsigned long long* __restrict__ stats) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned na = 0, nm = 0, nd = 0;
    if (i < n) {
        const double ph = phi[i], po = phi_old[i];
        // (M^-1 b)_i + c (phi - phi_old)_i > 0, numpy's rounding (no contraction)
        const double ind = __dadd_rn(__ddiv_rn(rhs_phi[i], m_diag[i]), __dmul_rn(c, __dsub_rn(ph, po)));
        const bool act = ind > 0.0;
        active[i] = act ? 1 : 0;
        na = act;
        if (act && ph != po) {   // freshly activated: back onto the obstacle
            phi[i] = po;
            nm = 1;
        }
        if (prev) nd = (prev[i] != 0) != act;
    }
    // warp-aggregated counters
    na = __reduce_add_sync(0xffffffffu, na);
    nm = __reduce_add_sync(0xffffffffu, nm);
    nd = __reduce_add_sync(0xffffffffu, nd);
    if ((threadIdx.x & 31) == 0) {
        if (na) atomicAdd(&stats[0], (unsigned long long)na);
        if (nm) atomicAdd(&stats[1], (unsigned long long)nm);
        if (nd) atomicAdd(&stats[2], (unsigned long long)nd);
    }
}

}  // namespace

cudaError_t launch_lumped_mass(const Level& L, double* out, cudaStream_t s) {
    const Win w = L.win();
    const unsigned grid = (unsigned)((w.n + 255) / 256);
    k_lumped_mass<<<grid, 256, 0, s>>>(L.mesh, L.shape, w, out);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_active_set(int64_t n, const double* rhs_phi, double* phi,
                              const double* phi_old, const double* m_diag, double c,
                              const uint8_t* prev, uint8_t* active, unsigned long long* stats,
                              cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(stats, 0, 3 * sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    count_launches(1);
    if (n == 0) return cudaSuccess;
    const unsigned grid = (unsigned)((n + 255) / 256);
    k_active_set<<<grid, 256, 0, s>>>(n, rhs_phi, phi, phi_old, m_diag, c, prev, active, stats);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace pff
