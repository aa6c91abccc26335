# session-5 final evidence: GPU suite, smoke, bench, launch list, FP64/DRAM metric pass (Q2 + Q4),
# full ncu captures of the Q2 Miehe / none and Q4 Miehe sweeps
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/gputest_s5_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_s5_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s5_final.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_s5_final.log
timeout 1200 python bench.py > gpurun_out/bench_s5_final.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_s5_final.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_s5_reference.log 2>&1; echo "rc=$?" >> gpurun_out/bench_s5_reference.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --steps 20 --warmup 3 --no-newton --no-cpu-baseline --no-configs4 > gpurun_out/bench_launches_s5.csv 2> gpurun_out/bench_launches_s5.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum
rm -f gpurun_out/fp64_times_s5.txt
for cfg in "--degree 2 --level 10 --split miehe" "--degree 2 --level 10 --split none" "--degree 4 --level 9 --split miehe" "--degree 4 --level 9 --split none"; do
  tag=$(echo $cfg | tr -d ' -')
  timeout 300 python tools/prof_apply.py $cfg --reps 50 >> gpurun_out/fp64_times_s5.txt 2>&1
  timeout 600 ncu --metrics $M --clock-control none -k regex:"k_sweep|k_apply" --csv python tools/prof_apply.py $cfg --reps 1 > gpurun_out/fp64_ncu_$tag.csv 2>&1
done
for cfg in "--degree 2 --level 10 --split miehe" "--degree 2 --level 10 --split none" "--degree 4 --level 9 --split miehe"; do
  tag=$(echo $cfg | tr -d ' -')
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sweep -c 1 -o gpurun_out/ncu_s5_$tag python tools/prof_apply.py $cfg --reps 1 > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/ncu_s5_$tag.ncu-rep > gpurun_out/ncu_s5_$tag.txt 2>&1
done
