// pff_capi.cu -- extern "C" entry points of libpff_b200.so (include/pff_b200.h).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <vector>
#include <cstdio>
#include <cstring>
#include <new>

#include "../../include/pff_b200.h"
#include "pff_internal.cuh"

using pff::Level;

namespace pff {
std::atomic<long long> g_launch_count{0};
void count_launches(int k) { g_launch_count.fetch_add(k, std::memory_order_relaxed); }
}  // namespace pff

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, const char* what) {
    std::snprintf(g_err, sizeof(g_err), fmt, what);
    return code;
}

int check(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return 0;
    std::snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
    return (int)e;
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

bool bound(const Level* L) { return L && L->U && L->phi_tilde && L->flags && L->qcache; }

}  // namespace

extern "C" {

int pff_abi_version(void) { return PFF_ABI_VERSION; }

const char* pff_last_error(void) { return g_err; }

int64_t pff_launch_counter(void) { return pff::g_launch_count.load(); }

int pff_set_option(int key, int value) {
    switch (key) {
        case PFF_OPT_GENERIC_APPLY: pff::set_generic_apply(value != 0); return 0;
        case PFF_OPT_SWEEP_ROWS: pff::set_sweep_rows_per_chunk(value); return 0;
        case PFF_OPT_SWEEP_MIN_NSIDE: pff::set_sweep_min_nside(value); return 0;
        case PFF_OPT_SWEEP_COLRING: pff::set_sweep_colring(value); return 0;
    }
    return fail(PFF_E_ARG, "%s", "pff_set_option: unknown key");
}

int pff_level_create(pff_level** out, int degree, int level, int split, const pff_material* mat,
                     const double* N, const double* D, const double* w, const double* embed) {
    if (!out || !mat || !N || !D || !w) return fail(PFF_E_ARG, "%s", "pff_level_create: null argument");
    if (degree < 1 || degree > pff::PMAX) return fail(PFF_E_ARG, "%s", "pff_level_create: degree must be in 1..4");
    if (level < 0 || level > 14) return fail(PFF_E_ARG, "%s", "pff_level_create: level out of range");
    if (split != 0 && split != 1) return fail(PFF_E_ARG, "%s", "split must be 'none' or 'miehe'");
    Level* L = new (std::nothrow) Level();
    if (!L) return fail(PFF_E_ARG, "%s", "pff_level_create: out of host memory");
    L->mesh = pff::Mesh::make(degree, level);
    std::memset(&L->shape, 0, sizeof(L->shape));
    std::memset(&L->embed, 0, sizeof(L->embed));
    const int n1 = degree + 1;
    for (int iq = 0; iq < n1; ++iq) {
        L->shape.w[iq] = w[iq];
        for (int a = 0; a < n1; ++a) {
            L->shape.N[iq][a] = N[iq * n1 + a];
            L->shape.D[iq][a] = D[iq * n1 + a];
        }
    }
    if (embed)
        for (int c = 0; c < 2; ++c)
            for (int k = 0; k < n1; ++k)
                for (int m = 0; m < n1; ++m) L->embed.E[c][k][m] = embed[(c * n1 + k) * n1 + m];
    L->mat = pff::Material{mat->lame_lambda, mat->mu, mat->g_c, mat->kappa, mat->eps};
    if (degree == 2) {
        const auto& S = L->shape;
        auto near = [](double a, double b, double tol) { return a - b <= tol && b - a <= tol; };
        bool ok = near(S.N[1][0], 0.0, 1e-14) && near(S.N[1][1], 1.0, 1e-14) &&
                  near(S.N[1][2], 0.0, 1e-14) && near(S.D[1][0], -1.0, 1e-13) &&
                  near(S.D[1][1], 0.0, 1e-13) && near(S.D[1][2], 1.0, 1e-13) &&
                  near(S.w[0], S.w[2], 1e-15);
        for (int a = 0; a < 3; ++a)   // mirror symmetry of the outer Gauss points
            ok = ok && near(S.N[2][a], S.N[0][2 - a], 1e-14) && near(S.D[2][a], -S.D[0][2 - a], 1e-13);
        L->q2_struct = ok;
    }
    if (degree == 4) {   // mirror symmetry of the 5-point Gauss basis (even-odd form)
        const auto& S = L->shape;
        auto near = [](double a, double b, double tol) { return a - b <= tol && b - a <= tol; };
        bool ok = near(S.D[2][2], 0.0, 1e-12);
        for (int q = 0; q < 5; ++q) {
            ok = ok && near(S.w[q], S.w[4 - q], 1e-15);
            for (int a = 0; a < 5; ++a)
                ok = ok && near(S.N[4 - q][4 - a], S.N[q][a], 1e-13) &&
                     near(S.D[4 - q][4 - a], -S.D[q][a], 1e-12);
        }
        L->q4_struct = ok;
    }
    L->min_nside = pff::sweep_min_nside();
    L->miehe = split;
    *out = reinterpret_cast<pff_level*>(L);
    return 0;
}

int pff_level_destroy(pff_level* L) {
    delete reinterpret_cast<Level*>(L);
    return 0;
}

int64_t pff_level_n_scalar(const pff_level* L) {
    return L ? reinterpret_cast<const Level*>(L)->local_n() : -1;
}

int pff_level_set_window(pff_level* h, int cy_begin, int cy_end) {
    Level* L = reinterpret_cast<Level*>(h);
    if (!L) return fail(PFF_E_ARG, "%s", "pff_level_set_window: null level");
    if (cy_begin == 0 && cy_end == L->mesh.nside) {   // whole mesh
        L->win_begin = 0;
        L->win_end = -1;
        return 0;
    }
    if (cy_begin < 0 || cy_end > L->mesh.nside || cy_begin >= cy_end)
        return fail(PFF_E_ARG, "%s", "pff_level_set_window: bad cell-row range");
    if (!L->sweep_ok())
        return fail(PFF_E_ARG, "%s", "pff_level_set_window: slab windows need Q2 and >= 64x64 cells");
    L->win_begin = cy_begin;
    L->win_end = cy_end;
    return 0;
}

int pff_level_window(const pff_level* h, int64_t* rows) {
    const Level* L = reinterpret_cast<const Level*>(h);
    if (!L || !rows) return fail(PFF_E_ARG, "%s", "pff_level_window: null argument");
    rows[0] = L->j_lo();
    rows[1] = L->j_hi();
    rows[2] = L->local_dup() ? 1 : 0;
    rows[3] = L->dupoff() - L->row_shift();   // local index of the first slit copy
    rows[4] = L->cy_begin();
    rows[5] = L->cy_end();
    return 0;
}

int64_t pff_level_n_cells(const pff_level* L) {
    return L ? reinterpret_cast<const Level*>(L)->mesh.n_cells() : -1;
}

int64_t pff_level_qcache_len(const pff_level* L) {
    return L ? reinterpret_cast<const Level*>(L)->qcache_len() : -1;
}

int pff_level_uses_sweep(const pff_level* L) {
    if (!L) return -1;
    const Level* V = reinterpret_cast<const Level*>(L);
    return (V->sweep_ok() || V->sweep4_ok()) ? 1 : 0;
}

int pff_level_bind(pff_level* h, const double* U, const double* phi_tilde, const uint8_t* flags,
                   double* qcache) {
    Level* L = reinterpret_cast<Level*>(h);
    if (!L) return fail(PFF_E_ARG, "%s", "pff_level_bind: null level");
    L->U = U;
    L->phi_tilde = phi_tilde;
    L->flags = flags;
    L->qcache = qcache;
    return 0;
}

int pff_level_refresh(pff_level* h, void* stream) {
    Level* L = reinterpret_cast<Level*>(h);
    if (!bound(L)) return fail(PFF_E_UNBOUND, "%s", "pff_level_refresh: state not bound");
    return check(pff::launch_refresh(*L, S(stream)), "pff_level_refresh");
}

int pff_apply(const pff_level* h, int mode, const double* src, double* dst, const double* rhs,
              void* stream) {
    const Level* L = reinterpret_cast<const Level*>(h);
    if (!bound(L) && !(L && L->windowed() && L->U && L->phi_tilde && L->flags && L->qcache))
        return fail(PFF_E_UNBOUND, "%s", "pff_apply: state not bound");
    if (mode < 0 || mode > 3 || !src || !dst) return fail(PFF_E_ARG, "%s", "pff_apply: bad mode or null vector");
    return check(pff::launch_apply(*L, mode, src, dst, rhs, S(stream)), "pff_apply");
}

int pff_apply_cheb(const pff_level* h, int mode, const double* d, double* d_out,
                   const double* rhs, double* cr, const double* invd, double* acc, double c1,
                   double c2, void* stream) {
    const Level* L = reinterpret_cast<const Level*>(h);
    if (!bound(L) && !(L && L->windowed() && L->U && L->phi_tilde && L->flags && L->qcache))
        return fail(PFF_E_UNBOUND, "%s", "pff_apply_cheb: state not bound");
    if ((mode != 1 && mode != 2) || !d || !d_out || !rhs || !cr || !invd || !acc || d_out == d)
        return fail(PFF_E_ARG, "%s", "pff_apply_cheb: mode must be UU or PHIPHI, d_out != d");
    const pff::ChebArgs cb{invd, d_out, acc, c1, c2};
    return check(pff::launch_apply(*L, mode, d, cr, rhs, S(stream), &cb), "pff_apply_cheb");
}

int pff_apply_cheb_ex(const pff_level* h, int mode, const double* d, double* d_out,
                      const double* rhs, double* cr, const double* invd, double* acc, double c1,
                      double c2, int flags, void* stream) {
    const Level* L = reinterpret_cast<const Level*>(h);
    if (!bound(L) && !(L && L->windowed() && L->U && L->phi_tilde && L->flags && L->qcache))
        return fail(PFF_E_UNBOUND, "%s", "pff_apply_cheb_ex: state not bound");
    if ((mode != 1 && mode != 2) || !d || !d_out || !rhs || !cr || !invd || !acc || d_out == d ||
        (flags & ~(PFF_CHEB_FIRST | PFF_CHEB_LAST | PFF_CHEB_NOACC)) ||
        ((flags & PFF_CHEB_NOACC) && (flags & (PFF_CHEB_FIRST | PFF_CHEB_LAST))))
        return fail(PFF_E_ARG, "%s", "pff_apply_cheb_ex: mode must be UU or PHIPHI, d_out != d, known flags (NOACC alone)");
    pff::ChebArgs cb{invd, d_out, acc, c1, c2};
    cb.acc_src = (flags & PFF_CHEB_FIRST) ? 1 : 0;
    cb.last = (flags & PFF_CHEB_LAST) ? 1 : 0;
    cb.noacc = (flags & PFF_CHEB_NOACC) ? 1 : 0;
    return check(pff::launch_apply(*L, mode, d, cr, rhs, S(stream), &cb), "pff_apply_cheb_ex");
}

int pff_apply_cheb_first(const pff_level* h, int mode, const double* d, double* d_out,
                         const double* rhs, double* cr, const double* invd, double* acc,
                         double c1, double c2, void* stream) {
    return pff_apply_cheb_ex(h, mode, d, d_out, rhs, cr, invd, acc, c1, c2, PFF_CHEB_FIRST, stream);
}

int pff_apply_emit(const pff_level* h, int mode, const double* src, double* dst,
                   const double* rhs, const double* invd, double* d0, double theta,
                   void* stream) {
    const Level* L = reinterpret_cast<const Level*>(h);
    if (!bound(L) && !(L && L->windowed() && L->U && L->phi_tilde && L->flags && L->qcache))
        return fail(PFF_E_UNBOUND, "%s", "pff_apply_emit: state not bound");
    if ((mode != 0 && mode != 1 && mode != 3) || !src || !dst || !rhs || !invd || !d0 || !(theta != 0.0))
        return fail(PFF_E_ARG, "%s", "pff_apply_emit: mode must be FULL, UU or PHIROW, fused, theta != 0");
    pff::ChebArgs cb{invd, nullptr, nullptr, 0.0, 0.0};
    cb.emit = d0;
    cb.theta = theta;
    cb.emit_nc = mode == 3 ? 1 : 2;
    return check(pff::launch_apply(*L, mode, src, dst, rhs, S(stream), &cb), "pff_apply_emit");
}

int pff_smooth_init(const pff_level* h, const double* r, double* z, double* res_u,
                    const double* invd_u, double* d_u, double theta, void* stream) {
    return pff_smooth_init_ex(h, r, z, res_u, invd_u, d_u, theta, 0, stream);
}

int pff_smooth_init_ex(const pff_level* h, const double* r, double* z, double* res_u,
                       const double* invd_u, double* d_u, double theta, int flags, void* stream) {
    const Level* L = reinterpret_cast<const Level*>(h);
    if (!L || !L->flags) return fail(PFF_E_UNBOUND, "%s", "pff_smooth_init: flags not bound");
    if (!r || !z || !res_u || !invd_u || !d_u || !(theta != 0.0) || (flags & ~PFF_SMOOTH_ADD_D0))
        return fail(PFF_E_ARG, "%s", "pff_smooth_init: bad argument");
    return check(pff::launch_smooth_init(*L, r, z, res_u, invd_u, d_u, theta,
                                         (flags & PFF_SMOOTH_ADD_D0) != 0, S(stream)),
                 "pff_smooth_init");
}

int pff_apply_rows(const pff_level* h, int mode, const double* src, double* dst,
                   const double* rhs, int cy_begin, int cy_end, void* stream) {
    const Level* L = reinterpret_cast<const Level*>(h);
    if (!bound(L)) return fail(PFF_E_UNBOUND, "%s", "pff_apply_rows: state not bound");
    if (mode < 0 || mode > 3 || !src || !dst) return fail(PFF_E_ARG, "%s", "pff_apply_rows: bad mode or null vector");
    bool handled = false;
    cudaError_t e = pff::launch_sweep_apply_rows(*L, mode, src, dst, rhs, cy_begin, cy_end,
                                                 S(stream), &handled);
    if (!handled && e == cudaSuccess)
        return fail(PFF_E_ARG, "%s", "pff_apply_rows: needs the Q2 sweep kernel (p = 2, >= 64x64 cells)");
    return check(e, "pff_apply_rows");
}

namespace {

// Copy streams and events of pff_apply_host: created once per process (the
// pipeline is enqueue-bound when they are made per call), one pipeline at a
// time (the mutex), events recycled from a fixed pool.
struct HostPipe {
    std::mutex mu;
    bool ready = false;
    int device = -1;
    cudaStream_t s_in = nullptr, s_out = nullptr;
    static constexpr int NEV = 3 * 64 + 2;
    cudaEvent_t ev[NEV] = {};
    cudaError_t init() {
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        if (ready && dev == device) return cudaSuccess;
        if (ready) return cudaErrorNotSupported;   // one device per process
        if ((e = cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking)) != cudaSuccess) return e;
        if ((e = cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking)) != cudaSuccess) return e;
        for (auto& x : ev)
            if ((e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming)) != cudaSuccess) return e;
        device = dev;
        ready = true;
        return cudaSuccess;
    }
};
HostPipe g_pipe;

// chunk weights: small first and last chunks shorten the fill (the first
// chunk's H2D runs alone) and the drain (the last chunk's D2H);
// PFF_PIPE_RAMP="w0,w1,..." overrides (measurement knob)
std::vector<int> pipe_ramp() {
    std::vector<int> w;
    if (const char* env = std::getenv("PFF_PIPE_RAMP")) {
        for (const char* c = env; *c;) {
            char* end = nullptr;
            const long v = std::strtol(c, &end, 10);
            if (end == c) break;
            if (v > 0) w.push_back((int)v);
            c = *end ? end + 1 : end;
        }
    }
    if (w.empty()) w = {1, 2, 4, 4, 4, 4, 4, 4, 2, 1};
    return w;
}

}  // namespace

int pff_apply_host(const pff_level* h, int mode, const double* xh, double* yh, double* xd, double* yd,
                   int nchunks, void* stream) {
    const Level* L = reinterpret_cast<const Level*>(h);
    if (!bound(L)) return fail(PFF_E_UNBOUND, "%s", "pff_apply_host: state not bound");
    if (mode < 0 || mode > 3 || !xh || !yh || !xd || !yd || nchunks < 0 || nchunks > 64)
        return fail(PFF_E_ARG, "%s", "pff_apply_host: bad mode, null buffer or nchunks outside 0..64");
    if (L->windowed() || !L->sweep_ok())
        return fail(PFF_E_ARG, "%s", "pff_apply_host: needs a whole-mesh level on the Q2 sweep kernel (p = 2, >= 64x64 cells)");
    static const int NC_IN[4] = {3, 2, 1, 3}, NC_OUT[4] = {3, 2, 1, 1};
    const int cin = NC_IN[mode], cout = NC_OUT[mode];
    const pff::Mesh& m = L->mesh;
    const int64_t n = m.n, np1 = m.np1, ng = m.n_grid, nd = m.n_dup, im = m.i_mid;
    const int ns = m.nside, p = m.p;
    // chunk boundaries in cell rows
    std::vector<int> w = nchunks > 0 ? std::vector<int>(nchunks, 1) : pipe_ramp();
    if ((int)w.size() > ns) w.assign(ns < 8 ? ns : 8, 1);
    if ((int)w.size() > 64) return fail(PFF_E_ARG, "%s", "pff_apply_host: more than 64 chunks");
    double tot = 0.0;
    for (int x : w) tot += x;
    std::vector<int> cuts{0};
    double acc = 0.0;
    for (int x : w) {
        acc += x;
        const int c = (int)std::lround(acc / tot * ns);
        if (c > cuts.back()) cuts.push_back(c);
    }
    const int K = (int)cuts.size() - 1;
    std::lock_guard<std::mutex> lock(g_pipe.mu);
    cudaError_t e = g_pipe.init();
    if (e != cudaSuccess) return check(e, "pff_apply_host: streams");
    cudaStream_t main = S(stream), s_in = g_pipe.s_in, s_out = g_pipe.s_out;
    cudaEvent_t* ev_in = g_pipe.ev;            // [K]: chunk k's inputs on the device
    cudaEvent_t* ev_done = g_pipe.ev + 64;     // [K]: chunk k's sweep done
    cudaEvent_t ev_start = g_pipe.ev[192], ev_end = g_pipe.ev[193];
    // PFF_PIPE_1D=1: one 1-D copy per component instead of one 2-D copy (measurement knob)
    static const bool one_d = [] {
        const char* e = std::getenv("PFF_PIPE_1D");
        return e && e[0] == '1';
    }();
    auto copy = [&](double* dst, const double* src, int64_t a, int64_t cnt, int nc, cudaStream_t s) {
        const size_t pitch = (size_t)n * sizeof(double);
        if (one_d) {
            for (int c = 0; c < nc; ++c) {
                const cudaError_t ce = cudaMemcpyAsync(dst + a + c * n, src + a + c * n,
                                                       (size_t)cnt * sizeof(double), cudaMemcpyDefault, s);
                if (ce != cudaSuccess) return ce;
            }
            return cudaSuccess;
        }
        return cudaMemcpy2DAsync(dst + a, pitch, src + a, pitch, (size_t)cnt * sizeof(double),
                                 (size_t)nc, cudaMemcpyDefault, s);
    };
    // on a failure part-way, copies already queued on s_in / s_out still read xh /
    // write yh and the device buffers: drain both copy streams before returning,
    // so the caller may free or reuse every buffer once the error is reported
    auto drain = [&]() {
        cudaStreamSynchronize(s_in);
        cudaStreamSynchronize(s_out);
    };
#define PFF_TRY(x) do { if ((e = (x)) != cudaSuccess) { drain(); return check(e, "pff_apply_host"); } } while (0)
    // the caller's earlier work on xd / yd / xh / yh comes first
    PFF_TRY(cudaEventRecord(ev_start, main));
    PFF_TRY(cudaStreamWaitEvent(s_in, ev_start, 0));
    PFF_TRY(cudaStreamWaitEvent(s_out, ev_start, 0));
    // every H2D first: the copy engine's queue never waits on the host
    int64_t loaded = -1;   // last node row on the device
    bool dups_in = nd == 0;
    for (int k = 0; k < K; ++k) {
        const int c1 = cuts[k + 1];
        const int64_t hi = std::min<int64_t>((int64_t)p * c1 + (c1 < ns ? 1 : 0), np1 - 1);
        if (hi > loaded) {   // all components of the new node rows: one strided copy
            PFF_TRY(copy(xd, xh, (loaded + 1) * np1, (hi - loaded) * np1, cin, s_in));
            loaded = hi;
        }
        if (!dups_in && c1 > ns / 2) {
            PFF_TRY(copy(xd, xh, ng, nd, cin, s_in));
            dups_in = true;
        }
        PFF_TRY(cudaEventRecord(ev_in[k], s_in));
    }
    for (int k = 0; k < K; ++k) {
        const int c0 = cuts[k], c1 = cuts[k + 1];
        PFF_TRY(cudaStreamWaitEvent(main, ev_in[k], 0));
        bool handled = false;
        PFF_TRY(pff::launch_sweep_apply_rows(*L, mode, xd, yd, nullptr, c0, c1, main, &handled));
        if (!handled) {
            drain();
            return fail(PFF_E_ARG, "%s", "pff_apply_host: sweep kernel refused the rows");
        }
        PFF_TRY(cudaEventRecord(ev_done[k], main));
        PFF_TRY(cudaStreamWaitEvent(s_out, ev_done[k], 0));
        const int64_t top = (int64_t)p * c1 + (c1 == ns ? 1 : 0);
        PFF_TRY(copy(yh, yd, (int64_t)p * c0 * np1, (top - (int64_t)p * c0) * np1, cout, s_out));
        if (nd && (int64_t)p * c0 <= im && im < top) PFF_TRY(copy(yh, yd, ng, nd, cout, s_out));
    }
    // the caller's stream resumes after the last D2H (and the last H2D)
    PFF_TRY(cudaEventRecord(ev_end, s_out));
    PFF_TRY(cudaStreamWaitEvent(main, ev_end, 0));
    PFF_TRY(cudaEventRecord(ev_start, s_in));
    PFF_TRY(cudaStreamWaitEvent(main, ev_start, 0));
#undef PFF_TRY
    return 0;
}

int pff_diagonal(const pff_level* h, double* duu, double* dpp, int invert, void* stream) {
    const Level* L = reinterpret_cast<const Level*>(h);
    if (!bound(L)) return fail(PFF_E_UNBOUND, "%s", "pff_diagonal: state not bound");
    if (!duu || !dpp) return fail(PFF_E_ARG, "%s", "pff_diagonal: null output");
    return check(pff::launch_diagonal(*L, duu, duu + L->local_n(), dpp, invert, S(stream)),
                 "pff_diagonal");
}

int pff_residual(const pff_level* h, double* out, int md, int ma, void* stream) {
    const Level* L = reinterpret_cast<const Level*>(h);
    if (!bound(L)) return fail(PFF_E_UNBOUND, "%s", "pff_residual: state not bound");
    if (!out) return fail(PFF_E_ARG, "%s", "pff_residual: null output");
    return check(pff::launch_residual(*L, out, md, ma, S(stream)), "pff_residual");
}

int pff_cell_matrices(const pff_level* h, double* gk, void* stream) {
    const Level* L = reinterpret_cast<const Level*>(h);
    if (!bound(L)) return fail(PFF_E_UNBOUND, "%s", "pff_cell_matrices: state not bound");
    if (!gk) return fail(PFF_E_ARG, "%s", "pff_cell_matrices: null output");
    return check(pff::launch_cell_matrices(*L, gk, S(stream)), "pff_cell_matrices");
}

int pff_dense_jacobian(const pff_level* h, const double* gk, double* G, void* stream) {
    const Level* L = reinterpret_cast<const Level*>(h);
    if (!bound(L)) return fail(PFF_E_UNBOUND, "%s", "pff_dense_jacobian: state not bound");
    if (!gk || !G) return fail(PFF_E_ARG, "%s", "pff_dense_jacobian: null argument");
    if (L->windowed() || 3 * L->mesh.n > 8192)
        return fail(PFF_E_ARG, "%s", "pff_dense_jacobian: whole-mesh levels with 3n <= 8192 only");
    return check(pff::launch_dense_jacobian(*L, gk, G, S(stream)), "pff_dense_jacobian");
}

int pff_dgemm(int m, int n, int k, double alpha, const double* A, int lda, const double* B, int ldb,
              double beta, double* C, int ldc, void* stream) {
    if (m < 0 || n < 0 || k < 0 || (m > 0 && n > 0 && (!C || (k > 0 && (!A || !B)))) ||
        lda < k || ldb < n || ldc < n)
        return fail(PFF_E_ARG, "%s", "pff_dgemm: bad sizes, leading dimensions or null matrix");
    return check(pff::launch_dgemm(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, S(stream)),
                 "pff_dgemm");
}

int pff_dmat_axpby(int m, int n, double a, double* Y, int ldy, double b, const double* s,
                   const double* X, int ldx, void* stream) {
    if (m < 0 || n < 0 || (m > 0 && n > 0 && (!Y || !X)) || ldy < n || ldx < n)
        return fail(PFF_E_ARG, "%s", "pff_dmat_axpby: bad sizes or null matrix");
    return check(pff::launch_dmat_axpby(m, n, a, Y, ldy, b, s, X, ldx, S(stream)), "pff_dmat_axpby");
}

int pff_dmat_diag(int n, const double* s, double* Y, int ldy, void* stream) {
    if (n < 0 || (n > 0 && !Y) || ldy < n)
        return fail(PFF_E_ARG, "%s", "pff_dmat_diag: bad size or null matrix");
    return check(pff::launch_dmat_diag(n, s, Y, ldy, S(stream)), "pff_dmat_diag");
}

int pff_recip(int64_t n, const double* x, double* y, int mode, void* stream) {
    if (n < 0 || (n > 0 && (!x || !y)) || (mode != 0 && mode != 1))
        return fail(PFF_E_ARG, "%s", "pff_recip: bad size, null vector or mode");
    return check(pff::launch_recip(n, x, y, mode, S(stream)), "pff_recip");
}

int pff_flags(int64_t n, uint8_t* dir, uint8_t* act, uint8_t* flags, int mode, void* stream) {
    if (n < 0 || (n > 0 && (!dir || !act || !flags)) || (mode != 0 && mode != 1))
        return fail(PFF_E_ARG, "%s", "pff_flags: bad size, null mask or mode");
    return check(pff::launch_flags(n, dir, act, flags, mode, S(stream)), "pff_flags");
}

int pff_lumped_mass(const pff_level* h, double* out, void* stream) {
    const Level* L = reinterpret_cast<const Level*>(h);
    if (!L || !out) return fail(PFF_E_ARG, "%s", "pff_lumped_mass: null argument");
    return check(pff::launch_lumped_mass(*L, out, S(stream)), "pff_lumped_mass");
}

int pff_active_set(int64_t n, const double* rhs_phi, double* phi, const double* phi_old,
                   const double* m_diag, double c, const uint8_t* prev, uint8_t* active,
                   uint64_t* stats, void* stream) {
    if (n < 0 || (n > 0 && (!rhs_phi || !phi || !phi_old || !m_diag || !active)) || !stats)
        return fail(PFF_E_ARG, "%s", "pff_active_set: bad argument");
    if (!(c > 0.0)) return fail(PFF_E_ARG, "%s", "pff_active_set: complementarity constant must be positive");
    return check(pff::launch_active_set(n, rhs_phi, phi, phi_old, m_diag, c, prev, active,
                                        reinterpret_cast<unsigned long long*>(stats), S(stream)),
                 "pff_active_set");
}

int pff_prolongate(const pff_level* f, const pff_level* c, const double* xc, double* yf,
                   int add_masked, void* stream) {
    const Level* F = reinterpret_cast<const Level*>(f);
    const Level* C = reinterpret_cast<const Level*>(c);
    if (!F || !C || !xc || !yf) return fail(PFF_E_ARG, "%s", "pff_prolongate: null argument");
    if (add_masked && !F->flags) return fail(PFF_E_UNBOUND, "%s", "pff_prolongate: fine flags not bound");
    return check(pff::launch_prolongate(*F, *C, xc, yf, add_masked, S(stream)), "pff_prolongate");
}

int pff_restrict(const pff_level* f, const pff_level* c, const double* yf, double* xc,
                 int zero_cons, void* stream) {
    const Level* F = reinterpret_cast<const Level*>(f);
    const Level* C = reinterpret_cast<const Level*>(c);
    if (!F || !C || !xc || !yf) return fail(PFF_E_ARG, "%s", "pff_restrict: null argument");
    if (zero_cons && !C->flags) return fail(PFF_E_UNBOUND, "%s", "pff_restrict: coarse flags not bound");
    return check(pff::launch_restrict(*F, *C, yf, xc, zero_cons, S(stream)), "pff_restrict");
}

int pff_inject_f64(const pff_level* f, const pff_level* c, const double* src, double* dst,
                   int ncomp, void* stream) {
    const Level* F = reinterpret_cast<const Level*>(f);
    const Level* C = reinterpret_cast<const Level*>(c);
    if (!F || !C || !src || !dst || ncomp < 1) return fail(PFF_E_ARG, "%s", "pff_inject_f64: bad argument");
    return check(pff::launch_inject_f64(*F, *C, src, dst, ncomp, S(stream)), "pff_inject_f64");
}

int pff_inject_u8(const pff_level* f, const pff_level* c, const uint8_t* src, uint8_t* dst,
                  void* stream) {
    const Level* F = reinterpret_cast<const Level*>(f);
    const Level* C = reinterpret_cast<const Level*>(c);
    if (!F || !C || !src || !dst) return fail(PFF_E_ARG, "%s", "pff_inject_u8: bad argument");
    return check(pff::launch_inject_u8(*F, *C, src, dst, S(stream)), "pff_inject_u8");
}

int pff_cons(const pff_level* h, int layout, int op, const double* r, double* z, void* stream) {
    const Level* L = reinterpret_cast<const Level*>(h);
    if (!L || !L->flags) return fail(PFF_E_UNBOUND, "%s", "pff_cons: flags not bound");
    if (layout < 0 || layout > 2 || op < 0 || op > 3 || !z || (op != 1 && !r))
        return fail(PFF_E_ARG, "%s", "pff_cons: bad argument");
    return check(pff::launch_cons(*L, layout, op, r, z, S(stream)), "pff_cons");
}

int pff_cheb_init(int64_t n, const double* invd, const double* rhs, double theta, double* d,
                  double* acc, int acc_mode, void* stream) {
    if (n < 0 || !invd || !rhs || !d || (acc_mode != 2 && !acc)) return fail(PFF_E_ARG, "%s", "pff_cheb_init: bad argument");
    return check(pff::launch_cheb_init(n, invd, rhs, theta, d, acc, acc_mode, S(stream)), "pff_cheb_init");
}

int pff_cheb_step(int64_t n, const double* invd, const double* r, double c1, double c2,
                  double* d, double* acc, void* stream) {
    if (n < 0 || !invd || !r || !d || !acc) return fail(PFF_E_ARG, "%s", "pff_cheb_step: bad argument");
    return check(pff::launch_cheb_step(n, invd, r, c1, c2, d, acc, S(stream)), "pff_cheb_step");
}

int pff_axpby(int64_t n, double a, const double* x, double b, double* y, void* stream) {
    if (n < 0 || !x || !y) return fail(PFF_E_ARG, "%s", "pff_axpby: bad argument");
    return check(pff::launch_axpby(n, a, x, b, y, S(stream)), "pff_axpby");
}

int pff_div(int64_t n, const double* x, const double* sdev, double sval, double* y, void* stream) {
    if (n < 0 || !x || !y) return fail(PFF_E_ARG, "%s", "pff_div: bad argument");
    return check(pff::launch_div(n, x, sdev, sval, y, S(stream)), "pff_div");
}

int pff_mul(int64_t n, const double* a, const double* x, double* y, void* stream) {
    if (n < 0 || !a || !x || !y) return fail(PFF_E_ARG, "%s", "pff_mul: bad argument");
    return check(pff::launch_lanczos_scale(n, a, x, y, S(stream)), "pff_mul");
}

int pff_lanczos_ranges(int nruns, const pff_level* const* levels, const int* modes,
                       const int64_t* ns, const double* const* dhalf, double* const* work,
                       int max_iterations, double* lo_hi, double* partials, double* dots,
                       void* stream) {
    if (nruns < 0 || (nruns > 0 && (!levels || !modes || !ns || !dhalf || !work || !lo_hi ||
                                    !partials || !dots)))
        return fail(PFF_E_ARG, "%s", "pff_lanczos_ranges: bad argument");
    for (int r = 0; r < nruns; ++r) {
        const Level* L = reinterpret_cast<const Level*>(levels[r]);
        if (!bound(L)) return fail(PFF_E_UNBOUND, "%s", "pff_lanczos_ranges: state not bound");
        if ((modes[r] != 1 && modes[r] != 2) || !dhalf[r] || !work[r] || ns[r] <= 0)
            return fail(PFF_E_ARG, "%s", "pff_lanczos_ranges: bad run");
    }
    return check(pff::lanczos_ranges(nruns, reinterpret_cast<const Level* const*>(levels), modes,
                                     ns, dhalf, work, max_iterations, lo_hi, partials, dots,
                                     S(stream)),
                 "pff_lanczos_ranges");
}

int pff_copy_components(double* dst, const double* src, int64_t count, int ncomp,
                        int64_t stride, void* stream) {
    if (!dst || !src || count < 0 || ncomp < 1 || stride < count)
        return fail(PFF_E_ARG, "%s", "pff_copy_components: bad argument");
    if (count == 0) return 0;
    const size_t pitch = (size_t)stride * sizeof(double);
    return check(cudaMemcpy2DAsync(dst, pitch, src, pitch, (size_t)count * sizeof(double),
                                   (size_t)ncomp, cudaMemcpyDefault, S(stream)),
                 "pff_copy_components");
}

int64_t pff_reduce_scratch_len(void) { return 2 * pff::RED_BLOCKS; }

int pff_dot(int64_t n, const double* x, const double* y, double* partials, double* out,
            void* stream) {
    if (n < 0 || !x || !y || !partials) return fail(PFF_E_ARG, "%s", "pff_dot: bad argument");
    return check(pff::launch_dot(n, x, y, partials, out, S(stream)), "pff_dot");
}

int pff_mgs(int64_t n, int j, const double* V, int64_t ldv, double* w, double* partials, double* h,
            void* stream) {
    if (n < 0 || j < 0 || !V || !w || !partials || !h || ldv < n) return fail(PFF_E_ARG, "%s", "pff_mgs: bad argument");
    return check(pff::launch_mgs(n, j, V, ldv, w, partials, h, S(stream)), "pff_mgs");
}

int pff_mgs_lowsync(int64_t n, int j, const double* V, int64_t ldv, double* w, double* gram,
                    int64_t ldg, double* partials, double* h, void* stream) {
    if (n < 0 || j < 0 || j > 1023 || !V || !w || !gram || ldg <= j || !partials || !h || ldv < n)
        return fail(PFF_E_ARG, "%s", "pff_mgs_lowsync: bad argument");
    return check(pff::launch_lsmgs(n, j, V, ldv, w, gram, ldg, partials, h, S(stream)),
                 "pff_mgs_lowsync");
}

int pff_mdot(int64_t n, int k, const double* V, int64_t ldv, const double* w, double* partials,
             double* out, void* stream) {
    if (n < 0 || k < 0 || k > 4096 || !V || !w || !partials || !out || ldv < n)
        return fail(PFF_E_ARG, "%s", "pff_mdot: bad argument");
    return check(pff::launch_mdot(n, k, V, ldv, w, partials, out, S(stream)), "pff_mdot");
}

int pff_combine(int64_t n, int k, const double* V, int64_t ldv, const double* y, double* out,
                int accumulate, void* stream) {
    if (n < 0 || k < 0 || !V || !y || !out) return fail(PFF_E_ARG, "%s", "pff_combine: bad argument");
    return check(pff::launch_combine(n, k, V, ldv, y, out, accumulate, S(stream)), "pff_combine");
}

int pff_dense_matvec(int64_t rows, int64_t cols, const double* M, const double* x, double* y,
                     void* stream) {
    if (rows < 1 || cols < 1 || rows > (1 << 24) || cols > (1 << 24) || !M || !x || !y || x == y)
        return fail(PFF_E_ARG, "%s", "pff_dense_matvec: bad argument");
    return check(pff::launch_dense_matvec((int)rows, (int)cols, M, x, y, S(stream)), "pff_dense_matvec");
}

int pff_coarse_dense(int64_t n, const double* Cu, const double* Gpu, const double* Cp,
                     const uint8_t* cmask, const double* r, double* z, void* stream) {
    if (n < 1 || n > pff::coarse_dense_nmax() || !Cu || !Gpu || !Cp || !cmask || !r || !z)
        return fail(PFF_E_ARG, "%s", "pff_coarse_dense: bad argument (n must be in 1..256)");
    return check(pff::launch_coarse_dense((int)n, Cu, Gpu, Cp, cmask, r, z, S(stream)),
                 "pff_coarse_dense");
}

}  // extern "C"
