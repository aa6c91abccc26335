# Debug build with device-side staging checks (PFF_DEBUG_CHECKS: TMA alignment and
# sizes, staged-row / flag-row / tangent-block index bounds, bounded mbarrier waits)
# and the GPU suite on it.  compute-sanitizer is closed on the GPU pool; these are
# the checks of our own it asks for.  Build in the container, run on the box:
#   PFF_BUILD_TAG=debug PFF_NVCC_EXTRA=-DPFF_DEBUG_CHECKS python -c \
#       "from paper_2005_00331_b200 import _build; _build.build(force=True)"
#   gpurun -- bash tools/debug_checks.sh
mkdir -p gpurun_out
PFF_LIB=$PWD/paper_2005_00331_b200/libpff_b200_debug.so timeout 1500 python -m pytest tests -m gpu -q \
    -k "not level10 and not level11 and not level12" > gpurun_out/debug_checks.log 2>&1
echo "rc=$?" >> gpurun_out/debug_checks.log
PFF_LIB=$PWD/paper_2005_00331_b200/libpff_b200_debug.so timeout 600 python tools/sanitize_sweep.py >> gpurun_out/debug_checks.log 2>&1
echo "sanitize_sweep rc=$?" >> gpurun_out/debug_checks.log
