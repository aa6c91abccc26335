# session-5 evidence: FP64 / DRAM metric pass and full ncu captures of the Q2 sweeps (both splits)
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum
for cfg in "--degree 2 --level 10 --split miehe" "--degree 2 --level 10 --split none"; do
  tag=$(echo $cfg | tr -d ' -')
  timeout 300 python tools/prof_apply.py $cfg --reps 50 >> gpurun_out/fp64_times_s5.txt 2>&1
  timeout 600 ncu --metrics $M --clock-control none -k regex:"k_sweep|k_apply" --csv python tools/prof_apply.py $cfg --reps 1 > gpurun_out/fp64_ncu_$tag.csv 2>&1
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sweep -c 1 -o gpurun_out/ncu_s5_$tag python tools/prof_apply.py $cfg --reps 1 > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/ncu_s5_$tag.ncu-rep > gpurun_out/ncu_s5_$tag.txt 2>&1
done
