/*
 * pff_oracle.c -- CPU restatement of the reference's matrix-free phase-field
 * fracture cell loops.  TEST INFRASTRUCTURE ONLY: this file is the checker the
 * parity tests, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference arm compare against.  The product path (libpff_b200.so)
 * never links or calls it.
 *
 * Restated from the reference (fracturekit 0.1.0, /root/reference/pkg/src/
 * fracturekit/, cited as src/):
 *   - connectivity          src/mesh_hierarchy.py:156-189 (_scalar_numbering)
 *   - eigen / split helpers src/_kernels.py:26-123
 *   - residual cell loop    src/_kernels.py:319-440
 *   - q-point cache         src/_kernels.py:447-548 (without the optional
 *                           3x3 tangent tensors; the tangent path equals the
 *                           on-the-fly path, src/pff_operator.py:75)
 *   - Jacobian cell loop    src/_kernels.py:555-693 (flags do_uu/do_pp/do_coup)
 *   - block diagonals       src/_kernels.py:700-746
 *   - lumped mass row sums  src/_kernels.py:828-843
 *
 * Arithmetic follows the reference's operation order (separate multiply and
 * add; build with -ffp-contract=off) so the serial oracle reproduces the
 * reference to the last few ulps.  With nthreads > 1 the cells are processed
 * in four colours (cx%2, cy%2); cells of one colour share no node, so the
 * scatter is race-free, and only the summation order per node changes.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define PMAX 4
#define NMAX (PMAX + 1)

typedef struct {
    int p, n1, q, level, nside;
    int64_t np1, n_grid, n_dup, i_mid;
    double h;
    double N[NMAX][NMAX], D[NMAX][NMAX], w[NMAX];
} mesh_t;

static void mesh_init(mesh_t *m, int p, int level, const double *N, const double *D,
                      const double *w) {
    m->p = p;
    m->n1 = p + 1;
    m->q = p + 1;
    m->level = level;
    m->nside = 1 << level;
    m->np1 = (int64_t)p * m->nside + 1;
    m->n_grid = m->np1 * m->np1;
    m->i_mid = (int64_t)p * m->nside / 2;
    m->n_dup = level >= 1 ? m->i_mid : 0;
    m->h = 1.0 / (double)m->nside;
    for (int iq = 0; iq < m->q; ++iq) {
        m->w[iq] = w[iq];
        for (int a = 0; a < m->n1; ++a) {
            m->N[iq][a] = N[iq * m->n1 + a];
            m->D[iq][a] = D[iq * m->n1 + a];
        }
    }
}

/* scalar node id of local node (a, b) of cell (cx, cy): mesh_hierarchy.py:175-188 */
static inline int64_t node_id(const mesh_t *m, int cx, int cy, int a, int b) {
    int64_t j = (int64_t)cy * m->p + b;
    int64_t i = (int64_t)cx * m->p + a;
    if (m->level >= 1 && cy >= m->nside / 2 && j == m->i_mid && i < m->i_mid)
        return m->n_grid + i;
    return j * m->np1 + i;
}

/* ---------------------------------------------------------------- physics */

typedef struct { double ev1, ev2, c, s; } eig_t;

/* closed-form 2x2 eigensystem, ev1 >= ev2, v1 = (c, s): _kernels.py:26-47 */
static inline eig_t eig2(double a11, double a22, double a12) {
    eig_t e;
    double m = 0.5 * (a11 + a22);
    double dh = 0.5 * (a11 - a22);
    double r = sqrt(dh * dh + a12 * a12);
    e.ev1 = m + r;
    e.ev2 = m - r;
    double vx, vy;
    if (dh <= 0.0) { vx = a12; vy = r - dh; }
    else           { vx = r + dh; vy = a12; }
    double nrm = sqrt(vx * vx + vy * vy);
    if (nrm > 0.0) { e.c = vx / nrm; e.s = vy / nrm; }
    else           { e.c = 1.0; e.s = 0.0; }
    return e;
}

static inline double posp(double x) { return x > 0.0 ? x : 0.0; }

/* derivative of A -> A+ in direction dA: _kernels.py:50-74 */
static inline void dpos2(eig_t e, double scale, double d11, double d22, double d12,
                         double *o11, double *o22, double *o12) {
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
    *o11 = dl1p * c * c + dl2p * s * s - 2.0 * rot * s * c;
    *o22 = dl1p * s * s + dl2p * c * c + 2.0 * rot * s * c;
    *o12 = (dl1p - dl2p) * c * s + rot * (c * c - s * s);
}

/* sigma+ from the eigensystem: _kernels.py:77-85 */
static inline void sigplus2(double lam, double mu, double tre, eig_t e,
                            double *p11, double *p22, double *p12) {
    double trp = posp(tre), l1p = posp(e.ev1), l2p = posp(e.ev2);
    double c = e.c, s = e.s;
    *p11 = lam * trp + 2.0 * mu * (l1p * c * c + l2p * s * s);
    *p22 = lam * trp + 2.0 * mu * (l1p * s * s + l2p * c * c);
    *p12 = 2.0 * mu * (l1p - l2p) * c * s;
}

/* tensile energy: _kernels.py:88-93 */
static inline double esplus2(double lam, double mu, double tre, eig_t e) {
    double trp = posp(tre), l1p = posp(e.ev1), l2p = posp(e.ev2);
    return 0.5 * lam * trp * trp + mu * (l1p * l1p + l2p * l2p);
}

/* max(1, |e|_F): _kernels.py:96-99 */
static inline double scale2(double e11, double e22, double e12) {
    double f = sqrt(e11 * e11 + e22 * e22 + 2.0 * e12 * e12);
    return f > 1.0 ? f : 1.0;
}

/* g*dsigma+ + dsigma- and sigma+:de at one point: _kernels.py:102-123 */
static inline void dsig_split(double lam, double mu, double g, double e11, double e22,
                              double e12, double d11, double d22, double d12,
                              double *s11, double *s22, double *s12, double *spde) {
    eig_t e = eig2(e11, e22, e12);
    double tre = e11 + e22;
    double o11, o22, o12;
    dpos2(e, scale2(e11, e22, e12), d11, d22, d12, &o11, &o22, &o12);
    double trde = d11 + d22;
    double tt = tre < 0.0 ? 0.0 : trde;
    double dp11 = lam * tt + 2.0 * mu * o11;
    double dp22 = lam * tt + 2.0 * mu * o22;
    double dp12 = 2.0 * mu * o12;
    double f11 = lam * trde + 2.0 * mu * d11;
    double f22 = lam * trde + 2.0 * mu * d22;
    double f12 = 2.0 * mu * d12;
    double sp11, sp22, sp12;
    sigplus2(lam, mu, tre, e, &sp11, &sp22, &sp12);
    *spde = sp11 * d11 + sp22 * d22 + 2.0 * sp12 * d12;
    *s11 = g * dp11 + (f11 - dp11);
    *s22 = g * dp22 + (f22 - dp22);
    *s12 = g * dp12 + (f12 - dp12);
}

/* ------------------------------------------------- sum factorisation (1-D) */

typedef double nodal_t[NMAX][NMAX]; /* [b][a] = [y][x] */

static inline void gather(const mesh_t *m, const double *v, int cx, int cy, nodal_t out) {
    for (int b = 0; b < m->n1; ++b)
        for (int a = 0; a < m->n1; ++a) out[b][a] = v[node_id(m, cx, cy, a, b)];
}

static inline void scatter_add(const mesh_t *m, double *v, int cx, int cy, nodal_t in) {
    for (int b = 0; b < m->n1; ++b)
        for (int a = 0; a < m->n1; ++a) v[node_id(m, cx, cy, a, b)] += in[b][a];
}

/* t[b][iq] = sum_a M[iq][a] c[b][a] */
static inline void fwd_x(const mesh_t *m, double M[NMAX][NMAX], nodal_t c, nodal_t t) {
    for (int b = 0; b < m->n1; ++b)
        for (int iq = 0; iq < m->q; ++iq) {
            double acc = 0.0;
            for (int a = 0; a < m->n1; ++a) acc += M[iq][a] * c[b][a];
            t[b][iq] = acc;
        }
}

/* o[jq][iq] = sum_b M[jq][b] t[b][iq] */
static inline void fwd_y(const mesh_t *m, double M[NMAX][NMAX], nodal_t t, nodal_t o) {
    for (int jq = 0; jq < m->q; ++jq)
        for (int iq = 0; iq < m->q; ++iq) {
            double acc = 0.0;
            for (int b = 0; b < m->n1; ++b) acc += M[jq][b] * t[b][iq];
            o[jq][iq] = acc;
        }
}

/* t[b][iq] = sum_jq M[jq][b] f[jq][iq] */
static inline void bwd_y(const mesh_t *m, double M[NMAX][NMAX], nodal_t f, nodal_t t) {
    for (int b = 0; b < m->n1; ++b)
        for (int iq = 0; iq < m->q; ++iq) {
            double acc = 0.0;
            for (int jq = 0; jq < m->q; ++jq) acc += M[jq][b] * f[jq][iq];
            t[b][iq] = acc;
        }
}

/* r[b][a] += sum_iq M[iq][a] t[b][iq] */
static inline void bwd_x_add(const mesh_t *m, double M[NMAX][NMAX], nodal_t t, nodal_t r) {
    for (int b = 0; b < m->n1; ++b)
        for (int a = 0; a < m->n1; ++a) {
            double acc = r[b][a];
            for (int iq = 0; iq < m->q; ++iq) acc += M[iq][a] * t[b][iq];
            r[b][a] = acc;
        }
}

static inline void zero_nodal(nodal_t r) { memset(r, 0, sizeof(nodal_t)); }

/* value and reference-cell gradients at the q x q points */
static inline void eval_grad(const mesh_t *m, nodal_t c, nodal_t gx, nodal_t gy) {
    nodal_t tx, td;
    fwd_x(m, (double(*)[NMAX])m->N, c, tx);
    fwd_x(m, (double(*)[NMAX])m->D, c, td);
    fwd_y(m, (double(*)[NMAX])m->D, tx, gy);
    fwd_y(m, (double(*)[NMAX])m->N, td, gx);
}

#define MN ((double(*)[NMAX])m->N)
#define MD ((double(*)[NMAX])m->D)

/* ----------------------------------------------------------- cell drivers */

typedef void (*cell_fn)(const mesh_t *m, int cx, int cy, void *ctx);

/* colour-parallel (or serial, ascending cell order) cell loop */
static void for_all_cells(const mesh_t *m, cell_fn fn, void *ctx, int nthreads) {
    int ns = m->nside;
    if (nthreads <= 1) {
        for (int cy = 0; cy < ns; ++cy)
            for (int cx = 0; cx < ns; ++cx) fn(m, cx, cy, ctx);
        return;
    }
    for (int colour = 0; colour < 4; ++colour) {
        int px = colour & 1, py = colour >> 1;
        int nrows = (ns - py + 1) / 2, ncols = (ns - px + 1) / 2;
        int64_t total = (int64_t)nrows * ncols;
#pragma omp parallel for schedule(static) num_threads(nthreads)
        for (int64_t t = 0; t < total; ++t) {
            int cy = py + 2 * (int)(t / ncols);
            int cx = px + 2 * (int)(t % ncols);
            fn(m, cx, cy, ctx);
        }
    }
}

/* q-point cache layout: arrays (n_cells, q, q), cell = cy * nside + cx */
typedef struct {
    const double *ux, *uy, *ph, *pht;
    double lam, mu, gc, eps, kappa;
    int miehe;
    double *e11, *e22, *e12, *gt, *dg, *esp, *pc;
} cache_ctx;

static void cache_cell(const mesh_t *m, int cx, int cy, void *vctx) {
    cache_ctx *k = (cache_ctx *)vctx;
    nodal_t cu, cv, cp, ct, gxu, gyu, gxv, gyv, vp, vt, tx;
    gather(m, k->ux, cx, cy, cu);
    gather(m, k->uy, cx, cy, cv);
    gather(m, k->ph, cx, cy, cp);
    gather(m, k->pht, cx, cy, ct);
    eval_grad(m, cu, gxu, gyu);
    eval_grad(m, cv, gxv, gyv);
    fwd_x(m, MN, cp, tx);
    fwd_y(m, MN, tx, vp);
    fwd_x(m, MN, ct, tx);
    fwd_y(m, MN, tx, vt);
    double inv_h = 1.0 / m->h, gce = k->gc / k->eps, gdd = 2.0 * (1.0 - k->kappa);
    int64_t base = ((int64_t)cy * m->nside + cx) * m->q * m->q;
    for (int jq = 0; jq < m->q; ++jq)
        for (int iq = 0; iq < m->q; ++iq) {
            double e11 = gxu[jq][iq] * inv_h;
            double e22 = gyv[jq][iq] * inv_h;
            double e12 = 0.5 * (gyu[jq][iq] + gxv[jq][iq]) * inv_h;
            double tre = e11 + e22;
            double g_t = (1.0 - k->kappa) * vt[jq][iq] * vt[jq][iq] + k->kappa;
            double dgv = gdd * vp[jq][iq];
            double esp;
            if (k->miehe) esp = esplus2(k->lam, k->mu, tre, eig2(e11, e22, e12));
            else esp = 0.5 * k->lam * tre * tre + k->mu * (e11 * e11 + e22 * e22 + 2.0 * e12 * e12);
            int64_t o = base + jq * m->q + iq;
            k->e11[o] = e11;
            k->e22[o] = e22;
            k->e12[o] = e12;
            k->gt[o] = g_t;
            k->dg[o] = dgv;
            k->esp[o] = esp;
            k->pc[o] = gdd * esp + gce;
        }
}

int or_cache(int p, int level, const double *N, const double *D, const double *w,
             const double *ux, const double *uy, const double *ph, const double *pht,
             double lam, double mu, double gc, double eps, double kappa, int miehe,
             double *e11, double *e22, double *e12, double *gt, double *dg, double *esp,
             double *pc, int nthreads) {
    if (p < 1 || p > PMAX) return -1;
    mesh_t m;
    mesh_init(&m, p, level, N, D, w);
    cache_ctx k = {ux, uy, ph, pht, lam, mu, gc, eps, kappa, miehe,
                   e11, e22, e12, gt, dg, esp, pc};
    for_all_cells(&m, cache_cell, &k, nthreads);
    return 0;
}

typedef struct {
    const double *dux, *duy, *dph;
    const double *e11, *e22, *e12, *gt, *dg, *pc;
    double lam, mu, gc, eps;
    int miehe, do_uu, do_pp, do_coup;
    double *ox, *oy, *op;
} jac_ctx;

static void jac_cell(const mesh_t *m, int cx, int cy, void *vctx) {
    jac_ctx *k = (jac_ctx *)vctx;
    int q = m->q;
    int need_u = k->do_uu || k->do_coup;
    nodal_t cu, cv, cp, tx, td, t1;
    nodal_t gxu, gyu, gxv, gyv, vp, gxp, gyp;
    nodal_t s11, s22, s12, fv, fgx, fgy, ru, rv, rp;
    if (need_u) {
        gather(m, k->dux, cx, cy, cu);
        gather(m, k->duy, cx, cy, cv);
        eval_grad(m, cu, gxu, gyu);
        eval_grad(m, cv, gxv, gyv);
    }
    if (k->do_pp) {
        gather(m, k->dph, cx, cy, cp);
        fwd_x(m, MN, cp, tx);
        fwd_x(m, MD, cp, td);
        fwd_y(m, MN, tx, vp);
        fwd_y(m, MD, tx, gyp);
        fwd_y(m, MN, td, gxp);
    }
    double h = m->h, inv_h = 1.0 / h;
    int64_t base = ((int64_t)cy * m->nside + cx) * q * q;
    for (int jq = 0; jq < q; ++jq)
        for (int iq = 0; iq < q; ++iq) {
            double wq = m->w[jq] * m->w[iq];
            double wg = wq * h, wv = wq * h * h;
            int64_t o = base + jq * q + iq;
            double coup = 0.0;
            if (need_u) {
                double d11 = gxu[jq][iq] * inv_h;
                double d22 = gyv[jq][iq] * inv_h;
                double d12 = 0.5 * (gyu[jq][iq] + gxv[jq][iq]) * inv_h;
                double e11 = k->e11[o], e22 = k->e22[o], e12 = k->e12[o], g_t = k->gt[o];
                double ds11, ds22, ds12, spde;
                if (k->miehe) {
                    dsig_split(k->lam, k->mu, g_t, e11, e22, e12, d11, d22, d12,
                               &ds11, &ds22, &ds12, &spde);
                } else {
                    double trde = d11 + d22;
                    ds11 = g_t * (k->lam * trde + 2.0 * k->mu * d11);
                    ds22 = g_t * (k->lam * trde + 2.0 * k->mu * d22);
                    ds12 = g_t * 2.0 * k->mu * d12;
                    double tre = e11 + e22;
                    spde = (k->lam * tre + 2.0 * k->mu * e11) * d11 +
                           (k->lam * tre + 2.0 * k->mu * e22) * d22 +
                           2.0 * (2.0 * k->mu * e12) * d12;
                }
                coup = k->dg[o] * spde;
                if (k->do_uu) {
                    s11[jq][iq] = ds11 * wg;
                    s22[jq][iq] = ds22 * wg;
                    s12[jq][iq] = ds12 * wg;
                }
            }
            if (k->do_pp) {
                double pval = k->pc[o] * vp[jq][iq];
                if (k->do_coup) pval += coup;
                fv[jq][iq] = pval * wv;
                fgx[jq][iq] = k->gc * k->eps * gxp[jq][iq] * inv_h * wg;
                fgy[jq][iq] = k->gc * k->eps * gyp[jq][iq] * inv_h * wg;
            } else if (k->do_coup) {
                fv[jq][iq] = coup * wv;
            }
        }
    if (k->do_uu) {
        zero_nodal(ru);
        bwd_y(m, MN, s11, t1); bwd_x_add(m, MD, t1, ru);
        bwd_y(m, MD, s12, t1); bwd_x_add(m, MN, t1, ru);
        zero_nodal(rv);
        bwd_y(m, MN, s12, t1); bwd_x_add(m, MD, t1, rv);
        bwd_y(m, MD, s22, t1); bwd_x_add(m, MN, t1, rv);
        scatter_add(m, k->ox, cx, cy, ru);
        scatter_add(m, k->oy, cx, cy, rv);
    }
    if (k->do_pp || k->do_coup) {
        zero_nodal(rp);
        bwd_y(m, MN, fv, t1); bwd_x_add(m, MN, t1, rp);
        if (k->do_pp) {
            bwd_y(m, MN, fgx, t1); bwd_x_add(m, MD, t1, rp);
            bwd_y(m, MD, fgy, t1); bwd_x_add(m, MN, t1, rp);
        }
        scatter_add(m, k->op, cx, cy, rp);
    }
}

/* out_* are accumulated (+=), as in the reference (_kernels.py:555-560) */
int or_jacobian(int p, int level, const double *N, const double *D, const double *w,
                const double *dux, const double *duy, const double *dph,
                const double *e11, const double *e22, const double *e12, const double *gt,
                const double *dg, const double *pc, double lam, double mu, double gc,
                double eps, int miehe, int do_uu, int do_pp, int do_coup, double *ox,
                double *oy, double *op, int nthreads) {
    if (p < 1 || p > PMAX) return -1;
    mesh_t m;
    mesh_init(&m, p, level, N, D, w);
    jac_ctx k = {dux, duy, dph, e11, e22, e12, gt, dg, pc, lam, mu, gc, eps,
                 miehe, do_uu, do_pp, do_coup, ox, oy, op};
    for_all_cells(&m, jac_cell, &k, nthreads);
    return 0;
}

typedef struct {
    const double *e11, *e22, *e12, *gt, *pc;
    double lam, mu, gc, eps;
    int miehe;
    double *dx, *dy, *dp;
} diag_ctx;

static void diag_cell(const mesh_t *m, int cx, int cy, void *vctx) {
    diag_ctx *k = (diag_ctx *)vctx;
    int q = m->q;
    double h = m->h, inv_h = 1.0 / h;
    int64_t base = ((int64_t)cy * m->nside + cx) * q * q;
    for (int b = 0; b < m->n1; ++b)
        for (int a = 0; a < m->n1; ++a) {
            double ax = 0.0, ay = 0.0, ap = 0.0;
            for (int jq = 0; jq < q; ++jq)
                for (int iq = 0; iq < q; ++iq) {
                    double wq = m->w[jq] * m->w[iq] * h * h;
                    double gx = m->D[iq][a] * m->N[jq][b] * inv_h;
                    double gy = m->N[iq][a] * m->D[jq][b] * inv_h;
                    double val = m->N[iq][a] * m->N[jq][b];
                    int64_t o = base + jq * q + iq;
                    double g_t = k->gt[o];
                    double x11, x22, x12, y11, y22, y12, unused;
                    if (k->miehe) {
                        double e11 = k->e11[o], e22 = k->e22[o], e12 = k->e12[o];
                        dsig_split(k->lam, k->mu, g_t, e11, e22, e12, gx, 0.0, 0.5 * gy,
                                   &x11, &x22, &x12, &unused);
                        dsig_split(k->lam, k->mu, g_t, e11, e22, e12, 0.0, gy, 0.5 * gx,
                                   &y11, &y22, &y12, &unused);
                    } else {
                        x11 = g_t * (k->lam + 2.0 * k->mu) * gx;
                        x22 = g_t * k->lam * gx;
                        x12 = g_t * k->mu * gy;
                        y11 = g_t * k->lam * gy;
                        y22 = g_t * (k->lam + 2.0 * k->mu) * gy;
                        y12 = g_t * k->mu * gx;
                    }
                    (void)x22;
                    (void)y11;
                    ax += (x11 * gx + x12 * gy) * wq;
                    ay += (y12 * gx + y22 * gy) * wq;
                    ap += (k->pc[o] * val * val + k->gc * k->eps * (gx * gx + gy * gy)) * wq;
                }
            int64_t gid = node_id(m, cx, cy, a, b);
            k->dx[gid] += ax;
            k->dy[gid] += ay;
            k->dp[gid] += ap;
        }
}

int or_diagonal(int p, int level, const double *N, const double *D, const double *w,
                const double *e11, const double *e22, const double *e12, const double *gt,
                const double *pc, double lam, double mu, double gc, double eps, int miehe,
                double *dx, double *dy, double *dp, int nthreads) {
    if (p < 1 || p > PMAX) return -1;
    mesh_t m;
    mesh_init(&m, p, level, N, D, w);
    diag_ctx k = {e11, e22, e12, gt, pc, lam, mu, gc, eps, miehe, dx, dy, dp};
    for_all_cells(&m, diag_cell, &k, nthreads);
    return 0;
}

typedef struct {
    const double *ux, *uy, *ph, *pht;
    double lam, mu, gc, eps, kappa;
    int miehe;
    double *ox, *oy, *op;
} res_ctx;

static void res_cell(const mesh_t *m, int cx, int cy, void *vctx) {
    res_ctx *k = (res_ctx *)vctx;
    int q = m->q;
    nodal_t cu, cv, cp, ct, tx, td, t1;
    nodal_t gxu, gyu, gxv, gyv, vp, gxp, gyp, vt;
    nodal_t s11, s22, s12, fv, fgx, fgy, ru, rv, rp;
    gather(m, k->ux, cx, cy, cu);
    gather(m, k->uy, cx, cy, cv);
    gather(m, k->ph, cx, cy, cp);
    gather(m, k->pht, cx, cy, ct);
    eval_grad(m, cu, gxu, gyu);
    eval_grad(m, cv, gxv, gyv);
    fwd_x(m, MN, cp, tx);
    fwd_x(m, MD, cp, td);
    fwd_y(m, MN, tx, vp);
    fwd_y(m, MD, tx, gyp);
    fwd_y(m, MN, td, gxp);
    fwd_x(m, MN, ct, tx);
    fwd_y(m, MN, tx, vt);
    double h = m->h, inv_h = 1.0 / h, gce = k->gc / k->eps;
    for (int jq = 0; jq < q; ++jq)
        for (int iq = 0; iq < q; ++iq) {
            double wq = m->w[jq] * m->w[iq];
            double wg = wq * h, wv = wq * h * h;
            double e11 = gxu[jq][iq] * inv_h;
            double e22 = gyv[jq][iq] * inv_h;
            double e12 = 0.5 * (gyu[jq][iq] + gxv[jq][iq]) * inv_h;
            double tre = e11 + e22;
            double phv = vp[jq][iq], ptv = vt[jq][iq];
            double g_t = (1.0 - k->kappa) * ptv * ptv + k->kappa;
            double sp11, sp22, sp12, sm11, sm22, sm12, esp;
            if (k->miehe) {
                eig_t e = eig2(e11, e22, e12);
                sigplus2(k->lam, k->mu, tre, e, &sp11, &sp22, &sp12);
                sm11 = k->lam * tre + 2.0 * k->mu * e11 - sp11;
                sm22 = k->lam * tre + 2.0 * k->mu * e22 - sp22;
                sm12 = 2.0 * k->mu * e12 - sp12;
                esp = esplus2(k->lam, k->mu, tre, e);
            } else {
                sp11 = k->lam * tre + 2.0 * k->mu * e11;
                sp22 = k->lam * tre + 2.0 * k->mu * e22;
                sp12 = 2.0 * k->mu * e12;
                sm11 = sm22 = sm12 = 0.0;
                esp = 0.5 * k->lam * tre * tre + k->mu * (e11 * e11 + e22 * e22 + 2.0 * e12 * e12);
            }
            s11[jq][iq] = (g_t * sp11 + sm11) * wg;
            s22[jq][iq] = (g_t * sp22 + sm22) * wg;
            s12[jq][iq] = (g_t * sp12 + sm12) * wg;
            double dgv = 2.0 * (1.0 - k->kappa) * phv;
            fv[jq][iq] = (dgv * esp - gce * (1.0 - phv)) * wv;
            fgx[jq][iq] = k->gc * k->eps * gxp[jq][iq] * inv_h * wg;
            fgy[jq][iq] = k->gc * k->eps * gyp[jq][iq] * inv_h * wg;
        }
    zero_nodal(ru);
    bwd_y(m, MN, s11, t1); bwd_x_add(m, MD, t1, ru);
    bwd_y(m, MD, s12, t1); bwd_x_add(m, MN, t1, ru);
    zero_nodal(rv);
    bwd_y(m, MN, s12, t1); bwd_x_add(m, MD, t1, rv);
    bwd_y(m, MD, s22, t1); bwd_x_add(m, MN, t1, rv);
    zero_nodal(rp);
    bwd_y(m, MN, fv, t1); bwd_x_add(m, MN, t1, rp);
    bwd_y(m, MN, fgx, t1); bwd_x_add(m, MD, t1, rp);
    bwd_y(m, MD, fgy, t1); bwd_x_add(m, MN, t1, rp);
    scatter_add(m, k->ox, cx, cy, ru);
    scatter_add(m, k->oy, cx, cy, rv);
    scatter_add(m, k->op, cx, cy, rp);
}

int or_residual(int p, int level, const double *N, const double *D, const double *w,
                const double *ux, const double *uy, const double *ph, const double *pht,
                double lam, double mu, double gc, double eps, double kappa, int miehe,
                double *ox, double *oy, double *op, int nthreads) {
    if (p < 1 || p > PMAX) return -1;
    mesh_t m;
    mesh_init(&m, p, level, N, D, w);
    res_ctx k = {ux, uy, ph, pht, lam, mu, gc, eps, kappa, miehe, ox, oy, op};
    for_all_cells(&m, res_cell, &k, nthreads);
    return 0;
}

typedef struct { double col[NMAX]; double *out; } mass_ctx;

static void mass_cell(const mesh_t *m, int cx, int cy, void *vctx) {
    mass_ctx *k = (mass_ctx *)vctx;
    for (int b = 0; b < m->n1; ++b)
        for (int a = 0; a < m->n1; ++a)
            k->out[node_id(m, cx, cy, a, b)] += k->col[a] * k->col[b] * m->h * m->h;
}

/* lumped phi mass: _kernels.py:828-843 */
int or_mass_rowsum(int p, int level, const double *N, const double *D, const double *w,
                   double *out, int nthreads) {
    if (p < 1 || p > PMAX) return -1;
    mesh_t m;
    mesh_init(&m, p, level, N, D, w);
    mass_ctx k;
    for (int a = 0; a < m.n1; ++a) {
        double acc = 0.0;
        for (int iq = 0; iq < m.q; ++iq) acc += m.w[iq] * m.N[iq][a];
        k.col[a] = acc;
    }
    k.out = out;
    for_all_cells(&m, mass_cell, &k, nthreads);
    return 0;
}

int or_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
