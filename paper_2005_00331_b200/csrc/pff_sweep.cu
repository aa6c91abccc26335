// pff_sweep.cu -- write-once Q2 operator kernel (placeholder until tuned).
#include "pff_internal.cuh"

namespace pff {

cudaError_t launch_sweep_apply(const Level& L, int mode, const double* src, double* dst,
                               const double* rhs, cudaStream_t s, bool* handled) {
    *handled = false;
    return cudaSuccess;
}

}  // namespace pff
