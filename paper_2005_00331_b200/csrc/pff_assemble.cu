// pff_assemble.cu -- dense per-cell Jacobian matrices G_k:
// src/pff_operator.py:328-340 -> src/_kernels.py:754-826.
//
// Used to assemble the CSR Jacobian on the device (assemble_oracle) for the
// assembled-SpMV-versus-matrix-free comparison of the paper.  One thread per
// (cell, column): the q-point responses of the column's basis function are
// computed once (tangent from the generic q-point cache), then every row of
// the column is summed over the q-points in the reference's (jq, iq) order
// and written once.  Layout gk[cell][row][col], rows/cols ordered
// (u_x | u_y | phi) x local nodes b*(p+1)+a, as the reference.
#include "pff_internal.cuh"

namespace pff {

namespace {

template <int P, bool MIEHE>
__global__ void __launch_bounds__(128)
k_cell_matrices(Mesh m, Shape S, Material M, const double* __restrict__ qc, double* __restrict__ gk) {
    constexpr int N1 = P + 1, NL = N1 * N1, NQ = N1 * N1, NC = 3 * NL;
    const int64_t nc = m.n_cells();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nc * NC) return;
    const int64_t cell = t / NC;
    const int col = (int)(t % NC);
    const int comp_j = col / NL, jl = col % NL;
    const int aj = jl % N1, bj = jl / N1;
    const double h = m.h, inv_h = 1.0 / h;
    const int64_t fs = (int64_t)NQ * nc;
    // per q-point responses of basis function j: (ds11, ds22, ds12, coup + pval-factor, pgx, pgy)
    double r11[NQ], r22[NQ], r12[NQ], rv[NQ], rgx[NQ], rgy[NQ], wqs[NQ];
#pragma unroll
    for (int jq = 0; jq < N1; ++jq)
#pragma unroll
        for (int iq = 0; iq < N1; ++iq) {
            const int k = jq * N1 + iq;
            const double wq = S.w[jq] * S.w[iq] * h * h;
            const double gxj = S.D[iq][aj] * S.N[jq][bj] * inv_h;
            const double gyj = S.N[iq][aj] * S.D[jq][bj] * inv_h;
            const double valj = S.N[iq][aj] * S.N[jq][bj];
            const double* q = qc + (int64_t)k * nc + cell;
            double ds11 = 0.0, ds22 = 0.0, ds12 = 0.0, coup = 0.0, pval = 0.0, pgx = 0.0, pgy = 0.0;
            if (comp_j < 2) {
                const double d11 = comp_j == 0 ? gxj : 0.0;
                const double d22 = comp_j == 0 ? 0.0 : gyj;
                const double d12 = comp_j == 0 ? 0.5 * gyj : 0.5 * gxj;
                double spde;
                dsig<MIEHE>(M.lam, M.mu, q[3 * fs], q[0], q[fs], q[2 * fs], d11, d22, d12, ds11,
                            ds22, ds12, spde);
                coup = q[4 * fs] * spde;
            } else {
                pval = q[5 * fs] * valj;
                pgx = M.gc * M.eps * gxj;
                pgy = M.gc * M.eps * gyj;
            }
            r11[k] = ds11;
            r22[k] = ds22;
            r12[k] = ds12;
            rv[k] = coup + pval;
            rgx[k] = pgx;
            rgy[k] = pgy;
            wqs[k] = wq;
        }
    double* out = gk + cell * (int64_t)NC * NC + col;
#pragma unroll 1
    for (int il = 0; il < NL; ++il) {
        const int ai = il % N1, bi = il / N1;
        double gu = 0.0, gv = 0.0, gp = 0.0;
#pragma unroll
        for (int jq = 0; jq < N1; ++jq)
#pragma unroll
            for (int iq = 0; iq < N1; ++iq) {
                const int k = jq * N1 + iq;
                const double gxi = S.D[iq][ai] * S.N[jq][bi] * inv_h;
                const double gyi = S.N[iq][ai] * S.D[jq][bi] * inv_h;
                const double vali = S.N[iq][ai] * S.N[jq][bi];
                gu += (r11[k] * gxi + r12[k] * gyi) * wqs[k];
                gv += (r12[k] * gxi + r22[k] * gyi) * wqs[k];
                gp += (rv[k] * vali + rgx[k] * gxi + rgy[k] * gyi) * wqs[k];
            }
        out[(int64_t)il * NC] = gu;
        out[(int64_t)(NL + il) * NC] = gv;
        out[(int64_t)(2 * NL + il) * NC] = gp;
    }
}

template <int P, bool MIEHE>
cudaError_t run_cm(const Level& L, double* gk, cudaStream_t s) {
    constexpr int NC = 3 * (P + 1) * (P + 1);
    const int64_t total = L.mesh.n_cells() * NC;
    k_cell_matrices<P, MIEHE><<<(unsigned)((total + 127) / 128), 128, 0, s>>>(
        L.mesh, L.shape, L.mat, L.qcache, gk);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_cell_matrices(const Level& L, double* gk, cudaStream_t s) {
    if (L.windowed()) return cudaErrorNotSupported;
    switch (L.mesh.p * 2 + (L.miehe ? 1 : 0)) {
        case 2: return run_cm<1, false>(L, gk, s);
        case 3: return run_cm<1, true>(L, gk, s);
        case 4: return run_cm<2, false>(L, gk, s);
        case 5: return run_cm<2, true>(L, gk, s);
        case 6: return run_cm<3, false>(L, gk, s);
        case 7: return run_cm<3, true>(L, gk, s);
        case 8: return run_cm<4, false>(L, gk, s);
        case 9: return run_cm<4, true>(L, gk, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace pff
