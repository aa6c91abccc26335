// pff_lanczos.cu -- batched Lanczos range estimates for the GMG setup
// (src/multigrid.py:123-162 estimate_lambda_range, run for every level and
// block as in GmgPreconditioner._estimate_ranges, 259-275).
//
// The runs are independent; they advance in lockstep, the scalars of the
// recurrence stay on the device, and the host (Ritz values, stopping tests)
// trails the GPU by one round, so no round waits on the host; the loop, the
// launches and the tridiagonal Ritz values stay in C++ instead of ~150
// Python/ctypes calls per round.  Per run and iteration, exactly the
// reference's recurrence on the Jacobi-scaled operator D^-1/2 A D^-1/2:
//   w = D^-1/2 A D^-1/2 v - beta v_prev;  alpha = v.w;  w -= alpha v;
//   Ritz values of T_k;  beta = |w|;  stop on beta < 1e-12 max(1, |hi|), on
//   |hi - hi_prev| <= 1e-4 |hi|, or after max_it;  v_prev, v = v, w / beta.
// Extreme Ritz values by Sturm-sequence bisection to full precision.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "pff_internal.cuh"

namespace pff {

namespace {

// number of eigenvalues of the symmetric tridiagonal (a, b) below x
int sturm_count(const std::vector<double>& a, const std::vector<double>& b, double x) {
    int cnt = 0;
    double q = a[0] - x;
    if (q < 0.0) ++cnt;
    for (size_t i = 1; i < a.size(); ++i) {
        const double qq = q != 0.0 ? q : DBL_MIN;
        q = (a[i] - x) - b[i - 1] * b[i - 1] / qq;
        if (q < 0.0) ++cnt;
    }
    return cnt;
}

// eigenvalue number k (0 = smallest) by bisection on the Gershgorin interval
double tridiag_eig(const std::vector<double>& a, const std::vector<double>& b, int k) {
    const size_t m = a.size();
    double lo = a[0], hi = a[0];
    for (size_t i = 0; i < m; ++i) {
        const double r = (i > 0 ? std::fabs(b[i - 1]) : 0.0) + (i + 1 < m ? std::fabs(b[i]) : 0.0);
        lo = std::min(lo, a[i] - r);
        hi = std::max(hi, a[i] + r);
    }
    for (int it = 0; it < 400; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (mid <= lo || mid >= hi) break;   // interval at machine resolution
        if (sturm_count(a, b, mid) > k) hi = mid;
        else lo = mid;
    }
    return 0.5 * (lo + hi);
}

// ---- batched vector kernels: one launch per phase for all active runs ----------
// Each run keeps the exact per-run arithmetic and reduction structure of the
// single-run kernels (k_mul, k_div, k_axpby, k_dot_partials / k_reduce_final:
// RED_BLOCKS x RED_THREADS grid-stride partials, fixed-order final sum), so a
// run's alphas and betas do not depend on how many runs share a launch.
constexpr int LZ_MAX = 32;
struct LzBatch {
    int nr;
    int slot[LZ_MAX];            // run index: partials / dots slot
    int64_t n[LZ_MAX];
    const double* dhalf[LZ_MAX];
    double* v[LZ_MAX];
    double* vp[LZ_MAX];
    double* w[LZ_MAX];
    double* tmp[LZ_MAX];
    int first;                   // round 0: no v / beta scaling, beta_prev = 0
    const double* sc;            // device scalars: sc[2 run] = alpha, sc[2 run + 1] = beta^2
};

__device__ __forceinline__ double lz_block_sum(double v) {
    __shared__ double sh[RED_THREADS / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double t = 0.0;
    if (wid == 0) {
        t = lane < RED_THREADS / 32 ? sh[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    }
    return t;
}

// (v = v / beta;) tmp = dhalf v -- beta = sqrt of the previous round's w.w,
// read on the device (IEEE sqrt: the same double the host's std::sqrt gives)
__global__ void __launch_bounds__(RED_THREADS) k_lz_pre(const LzBatch B) {
    const int r = blockIdx.y;
    const int64_t n = B.n[r];
    const double* dh = B.dhalf[r];
    double* v = B.v[r];
    double* t = B.tmp[r];
    const bool dv = !B.first;
    const double sv = dv ? sqrt(B.sc[2 * B.slot[r] + 1]) : 1.0;
    for (int64_t i = (int64_t)blockIdx.x * RED_THREADS + threadIdx.x; i < n;
         i += (int64_t)RED_BLOCKS * RED_THREADS) {
        double x = v[i];
        if (dv) {
            x = x / sv;
            v[i] = x;
        }
        t[i] = dh[i] * x;
    }
}

// post-apply: w = dhalf w; w = (-beta) vp + w; partials of v.w
// alpha step: w = (-alpha) v + w; partials of w.w
template <bool POST>
__global__ void __launch_bounds__(RED_THREADS) k_lz_update(const LzBatch B, double* part) {
    const int r = blockIdx.y;
    const int64_t n = B.n[r];
    // POST: -beta_prev (-0 in round 0, as the host's beta = 0 gave);  alpha step: -alpha
    const double a = POST ? (B.first ? -0.0 : -sqrt(B.sc[2 * B.slot[r] + 1])) : -B.sc[2 * B.slot[r]];
    const double* dh = B.dhalf[r];
    const double* v = B.v[r];
    const double* x = POST ? B.vp[r] : B.v[r];
    double* w = B.w[r];
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * RED_THREADS + threadIdx.x; i < n;
         i += (int64_t)RED_BLOCKS * RED_THREADS) {
        double wi = w[i];
        if (POST) wi = dh[i] * wi;
        wi = fma(a, x[i], wi);
        w[i] = wi;
        acc = POST ? fma(v[i], wi, acc) : fma(wi, wi, acc);
    }
    const double t = lz_block_sum(acc);
    if (threadIdx.x == 0) part[(int64_t)B.slot[r] * 2 * RED_BLOCKS + blockIdx.x] = t;
}

// dots[2 slot + which] = fixed-order sum of the run's RED_BLOCKS partials
__global__ void __launch_bounds__(RED_THREADS) k_lz_final(const LzBatch B, const double* part,
                                                          double* dots, int which) {
    const int slot = B.slot[blockIdx.x];
    const double* p = part + (int64_t)slot * 2 * RED_BLOCKS;
    double v = 0.0;
    for (int k = threadIdx.x; k < RED_BLOCKS; k += RED_THREADS) v += p[k];
    const double t = lz_block_sum(v);
    if (threadIdx.x == 0) dots[2 * slot + which] = t;
}

// pinned history of the per-round scalars (grown on demand, one driver at a time)
struct LzHost {
    std::mutex mu;
    double* hist = nullptr;
    size_t cap = 0;
    cudaEvent_t ev[4] = {};
    int device = -1;
};
LzHost g_lz;

struct Run {
    const Level* L;
    int mode;
    int64_t n;
    const double* dhalf;
    double *v, *vp, *w, *tmp;
    std::vector<double> alphas, betas;
    double beta = 0.0, lo = 1.0, hi = 1.0, prev = 0.0;
    bool has_prev = false, done = false;
    int left = 0;
};

}  // namespace

cudaError_t lanczos_ranges(int nruns, const Level* const* levels, const int* modes,
                           const int64_t* ns, const double* const* dhalf, double* const* work,
                           int max_it, double* lo_hi, double* partials, double* dots,
                           cudaStream_t s) {
    std::vector<Run> runs(nruns);
    for (int r = 0; r < nruns; ++r) {
        Run& R = runs[r];
        R.L = levels[r];
        R.mode = modes[r];
        R.n = ns[r];
        R.dhalf = dhalf[r];
        R.v = work[r];                 // holds the start vector on entry
        R.vp = work[r] + R.n;
        R.w = work[r] + 2 * R.n;
        R.tmp = work[r] + 3 * R.n;
        R.left = (int)std::min<int64_t>(max_it, R.n);
        R.done = R.left <= 0;
        cudaError_t e = cudaMemsetAsync(R.vp, 0, sizeof(double) * R.n, s);
        if (e != cudaSuccess) return e;
    }
    // The scalars never leave the device inside a round: alpha and beta^2 land in
    // dots[2 r], dots[2 r + 1] and the kernels read them from there.  Each round
    // ends with an async copy of dots into a pinned history slot; the host
    // processes round k (Ritz values, stopping tests) while the GPU already runs
    // round k + 1.  A run that stops at round k has done one extra round on its
    // own scratch vectors, which nothing reads: its alphas / betas, hence its
    // range, are those of the synchronous recurrence, bit for bit.
    std::lock_guard<std::mutex> lock(g_lz.mu);
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (g_lz.device != dev) {
        if (g_lz.device >= 0) return cudaErrorNotSupported;   // one device per process
        for (auto& x : g_lz.ev)
            if ((e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming)) != cudaSuccess) return e;
        g_lz.device = dev;
    }
    const int max_rounds = std::max(1, max_it) + 2;
    const size_t need = (size_t)max_rounds * 2 * nruns;
    if (g_lz.cap < need) {
        if (g_lz.hist) cudaFreeHost(g_lz.hist);
        g_lz.hist = nullptr;
        g_lz.cap = 0;
        if ((e = cudaHostAlloc(&g_lz.hist, need * sizeof(double), cudaHostAllocDefault)) != cudaSuccess) return e;
        g_lz.cap = need;
    }
    // the active runs in batches of LZ_MAX; per phase one launch per batch
    std::vector<char> live(nruns);   // in the round being enqueued
    auto batches = [&](int first, auto&& launch) -> cudaError_t {
        LzBatch B;
        B.nr = 0;
        B.first = first;
        B.sc = dots;
        for (int r = 0; r < nruns; ++r) {
            if (!live[r]) continue;
            const Run& R = runs[r];
            const int k = B.nr;
            B.n[k] = R.n;
            B.dhalf[k] = R.dhalf;
            B.v[k] = R.v;
            B.vp[k] = R.vp;
            B.w[k] = R.w;
            B.tmp[k] = R.tmp;
            B.slot[k] = r;
            if (++B.nr == LZ_MAX) {
                cudaError_t x = launch(B);
                if (x != cudaSuccess) return x;
                B.nr = 0;
            }
        }
        return B.nr ? launch(B) : cudaSuccess;
    };
    auto final_dots = [&](const LzBatch& B, int which) -> cudaError_t {
        k_lz_final<<<B.nr, RED_THREADS, 0, s>>>(B, partials, dots, which);
        count_launches(1);
        return cudaGetLastError();
    };
    // one round for the runs in `live`: device work, then the scalars to hist[round]
    auto enqueue = [&](int round) -> cudaError_t {
        cudaError_t x = batches(round == 0, [&](const LzBatch& B) -> cudaError_t {
            // (v = w_prev / beta;) tmp = D^-1/2 v
            k_lz_pre<<<dim3(RED_BLOCKS, B.nr), RED_THREADS, 0, s>>>(B);
            count_launches(1);
            return cudaGetLastError();
        });
        if (x != cudaSuccess) return x;
        for (int r = 0; r < nruns; ++r)
            if (live[r] && (x = launch_apply(*runs[r].L, runs[r].mode, runs[r].tmp, runs[r].w, nullptr, s)) != cudaSuccess)
                return x;
        // w = D^-1/2 w - beta v_prev;  alpha = v.w
        x = batches(round == 0, [&](const LzBatch& B) -> cudaError_t {
            k_lz_update<true><<<dim3(RED_BLOCKS, B.nr), RED_THREADS, 0, s>>>(B, partials);
            count_launches(1);
            cudaError_t y = cudaGetLastError();
            return y != cudaSuccess ? y : final_dots(B, 0);
        });
        if (x != cudaSuccess) return x;
        // w -= alpha v;  beta^2 = w.w
        x = batches(round == 0, [&](const LzBatch& B) -> cudaError_t {
            k_lz_update<false><<<dim3(RED_BLOCKS, B.nr), RED_THREADS, 0, s>>>(B, partials);
            count_launches(1);
            cudaError_t y = cudaGetLastError();
            return y != cudaSuccess ? y : final_dots(B, 1);
        });
        if (x != cudaSuccess) return x;
        x = cudaMemcpyAsync(g_lz.hist + (size_t)round * 2 * nruns, dots, sizeof(double) * 2 * nruns,
                            cudaMemcpyDeviceToHost, s);
        if (x != cudaSuccess) return x;
        // v_prev, v, w = v, w, v_prev for the next round (the swap the recurrence does
        // after a non-stopping round; a stopped run's later rounds are never read)
        for (int r = 0; r < nruns; ++r)
            if (live[r]) {
                Run& R = runs[r];
                double* old_vp = R.vp;
                R.vp = R.v;
                R.v = R.w;
                R.w = old_vp;
            }
        return cudaEventRecord(g_lz.ev[round & 3], s);
    };
    std::vector<std::vector<char>> members;   // runs in each enqueued round
    auto any_live = [&]() {
        for (int r = 0; r < nruns; ++r) live[r] = !runs[r].done;
        for (int r = 0; r < nruns; ++r)
            if (live[r]) return true;
        return false;
    };
    int enq = 0;
    if (any_live()) {
        members.push_back(live);
        if ((e = enqueue(enq++)) != cudaSuccess) return e;
    }
    for (int k = 0; k < enq; ++k) {
        // keep the GPU one round ahead: round k + 1 for every run not known to be done
        if (k + 1 == enq && enq < max_rounds && any_live()) {
            members.push_back(live);
            if ((e = enqueue(enq++)) != cudaSuccess) return e;
        }
        if ((e = cudaEventSynchronize(g_lz.ev[k & 3])) != cudaSuccess) return e;
        const double* h = g_lz.hist + (size_t)k * 2 * nruns;
        const std::vector<char>& in = members[k];
        for (int r = 0; r < nruns; ++r)
            if (in[r] && !runs[r].done) runs[r].alphas.push_back(h[2 * r]);
        // largest Ritz value of every active run (it drives the stopping test;
        // the smallest is needed only once a run stops): independent
        // bisections, spread over the host cores
#pragma omp parallel for schedule(dynamic, 1)
        for (int r = 0; r < nruns; ++r) {
            Run& R = runs[r];
            if (!in[r] || R.done) continue;
            if (R.betas.empty()) R.lo = R.hi = R.alphas.back();
            else R.hi = tridiag_eig(R.alphas, R.betas, (int)R.alphas.size() - 1);
        }
        for (int r = 0; r < nruns; ++r) {
            Run& R = runs[r];
            if (!in[r] || R.done) continue;
            const double beta = std::sqrt(h[2 * r + 1]);
            R.beta = beta;
            R.left -= 1;
            if (beta < 1e-12 * std::max(1.0, std::fabs(R.hi))) { R.done = true; continue; }
            if (R.has_prev && std::fabs(R.hi - R.prev) <= 1e-4 * std::fabs(R.hi)) {
                R.done = true;
                continue;
            }
            // (the stopping run's smallest Ritz value is taken after the loop)
            R.prev = R.hi;
            R.has_prev = true;
            R.betas.push_back(beta);
            if (R.left <= 0) R.done = true;
        }
    }
    // the speculative last round has finished before the caller reuses dots / work
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
#pragma omp parallel for schedule(dynamic, 1)
    for (int r = 0; r < nruns; ++r) {
        Run& R = runs[r];
        if (!R.betas.empty() || R.alphas.size() > 1) {
            // T of the final Ritz values: alphas[0..m), betas[0..m-1)
            std::vector<double> b(R.betas.begin(), R.betas.begin() + (R.alphas.size() - 1));
            R.lo = tridiag_eig(R.alphas, b, 0);
        }
    }
    for (int r = 0; r < nruns; ++r) {
        lo_hi[2 * r] = runs[r].lo;
        lo_hi[2 * r + 1] = runs[r].hi;
    }
    if (getenv("PFF_LANCZOS_DEBUG"))
        for (int r = 0; r < nruns; ++r)
            fprintf(stderr, "lanczos run %d: n %lld mode %d, %zu iterations, [%.6g, %.6g]\n", r,
                    (long long)runs[r].n, runs[r].mode, runs[r].alphas.size(), runs[r].lo, runs[r].hi);
    return cudaSuccess;
}

}  // namespace pff
