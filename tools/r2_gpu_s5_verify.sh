# session-5 verification after the eigen-frame tile / column ring: debug-checks build, GPU suite,
# functional N=2 run (two ranks on one GPU over gloo), the full bench incl. configs[4]
mkdir -p gpurun_out
bash tools/debug_checks.sh
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/s5_gputest_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s5_gputest_full.log
PFF_BENCH_ONE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --newton-level 10 --level 10 > gpurun_out/s5_n2_onegpu_l10.log 2>&1; echo "rc=$?" >> gpurun_out/s5_n2_onegpu_l10.log
timeout 1200 python bench.py > gpurun_out/s5_bench_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/s5_bench_full.log
