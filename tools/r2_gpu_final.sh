# full evidence run: GPU suite, smoke, bench, ncu launch list + full captures of the hot kernels
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/gputest_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_final.log
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_final.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --steps 20 --warmup 3 --no-newton --no-cpu-baseline --no-configs4 > gpurun_out/bench_launches.csv 2> gpurun_out/bench_launches.err
for cfg in "--degree 2 --level 10 --split miehe" "--degree 2 --level 10 --split none"; do
  tag=$(echo $cfg | tr -d ' -')
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sweep -c 1 -o gpurun_out/ncu_final_$tag python tools/prof_apply.py $cfg --reps 1 > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/ncu_final_$tag.ncu-rep > gpurun_out/ncu_final_$tag.txt 2>&1
done
