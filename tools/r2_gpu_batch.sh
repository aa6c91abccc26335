# round-2 GPU batch: full GPU suite, the reference suite through the drop-in,
# the bench line, per-level V-cycle costs at configs[4], a bounded oracle pin
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rs > gpurun_out/gputest_b1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_b1.log
PFF_REFSUITE=1 timeout 900 python -m pytest tests/ref_suite -q -rA > gpurun_out/refsuite_b1.log 2>&1; echo "refsuite rc=$?" >> gpurun_out/refsuite_b1.log
timeout 900 python bench.py > gpurun_out/bench_b1.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_b1.log
timeout 600 python tools/prof_vcycle_levels.py 12 > gpurun_out/vcycle_levels_l12.json 2> gpurun_out/vcycle_levels.err
timeout 1500 python tools/pin_newton_oracle.py --level 12 --split miehe --max-iterations 8 --out gpurun_out/pin_oracle_l12_miehe_it8.json > gpurun_out/pin12_it8.log 2>&1; echo "pin rc=$?" >> gpurun_out/pin12_it8.log
