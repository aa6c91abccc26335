// pff_lanczos.cu -- batched Lanczos range estimates for the GMG setup
// (src/multigrid.py:123-162 estimate_lambda_range, run for every level and
// block as in GmgPreconditioner._estimate_ranges, 259-275).
//
// The runs are independent; they advance in lockstep so each round costs two
// host synchronisations for all of them (alpha = v.w, then |w|), and the loop,
// the launches and the tridiagonal Ritz values stay in C++ instead of ~150
// Python/ctypes calls per round.  Per run and iteration, exactly the
// reference's recurrence on the Jacobi-scaled operator D^-1/2 A D^-1/2:
//   w = D^-1/2 A D^-1/2 v - beta v_prev;  alpha = v.w;  w -= alpha v;
//   Ritz values of T_k;  beta = |w|;  stop on beta < 1e-12 max(1, |hi|), on
//   |hi - hi_prev| <= 1e-4 |hi|, or after max_it;  v_prev, v = v, w / beta.
// Extreme Ritz values by Sturm-sequence bisection to full precision.
#include <algorithm>
#include <cfloat>
#include <cmath>
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
    std::vector<double> host(nruns);
    auto fetch = [&]() -> cudaError_t {
        cudaError_t e = cudaMemcpyAsync(host.data(), dots, sizeof(double) * nruns,
                                        cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        return e;
    };
    cudaError_t e = cudaSuccess;
    for (;;) {
        bool any = false;
        for (int r = 0; r < nruns; ++r) {
            Run& R = runs[r];
            if (R.done) continue;
            any = true;
            if ((e = launch_lanczos_scale(R.n, R.dhalf, R.v, R.tmp, s)) != cudaSuccess) return e;
            if ((e = launch_apply(*R.L, R.mode, R.tmp, R.w, nullptr, s)) != cudaSuccess) return e;
            if ((e = launch_lanczos_scale(R.n, R.dhalf, R.w, R.w, s)) != cudaSuccess) return e;
            if ((e = launch_axpby(R.n, -R.beta, R.vp, 1.0, R.w, s)) != cudaSuccess) return e;
            if ((e = launch_dot(R.n, R.v, R.w, partials + (int64_t)r * 2 * RED_BLOCKS, dots + r, s)) !=
                cudaSuccess)
                return e;
        }
        if (!any) break;
        if ((e = fetch()) != cudaSuccess) return e;
        for (int r = 0; r < nruns; ++r) {
            Run& R = runs[r];
            if (R.done) continue;
            const double alpha = host[r];
            if ((e = launch_axpby(R.n, -alpha, R.v, 1.0, R.w, s)) != cudaSuccess) return e;
            R.alphas.push_back(alpha);
            if (R.betas.empty()) {
                R.lo = R.hi = alpha;
            } else {
                R.lo = tridiag_eig(R.alphas, R.betas, 0);
                R.hi = tridiag_eig(R.alphas, R.betas, (int)R.alphas.size() - 1);
            }
            if ((e = launch_dot(R.n, R.w, R.w, partials + (int64_t)r * 2 * RED_BLOCKS, dots + r, s)) !=
                cudaSuccess)
                return e;
        }
        if ((e = fetch()) != cudaSuccess) return e;
        for (int r = 0; r < nruns; ++r) {
            Run& R = runs[r];
            if (R.done) continue;
            const double beta = std::sqrt(host[r]);
            R.beta = beta;
            R.left -= 1;
            if (beta < 1e-12 * std::max(1.0, std::fabs(R.hi))) { R.done = true; continue; }
            if (R.has_prev && std::fabs(R.hi - R.prev) <= 1e-4 * std::fabs(R.hi)) {
                R.done = true;
                continue;
            }
            R.prev = R.hi;
            R.has_prev = true;
            R.betas.push_back(beta);
            double* old_vp = R.vp;
            R.vp = R.v;
            R.v = R.w;
            R.w = old_vp;
            if ((e = launch_div(R.n, R.v, nullptr, beta, R.v, s)) != cudaSuccess) return e;
            if (R.left <= 0) R.done = true;
        }
    }
    for (int r = 0; r < nruns; ++r) {
        lo_hi[2 * r] = runs[r].lo;
        lo_hi[2 * r + 1] = runs[r].hi;
    }
    return cudaSuccess;
}

}  // namespace pff
