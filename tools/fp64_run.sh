set -x
mkdir -p gpurun_out
tools/micro/dfma_peak > gpurun_out/fp64_peak.json
for cfg in "--degree 2 --level 10 --split miehe" "--degree 2 --level 10 --split none" "--degree 4 --level 9 --split miehe" "--degree 4 --level 9 --split none"; do
  python tools/prof_apply.py $cfg --reps 50 >> gpurun_out/fp64_times.txt 2>&1
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum
for cfg in "--degree 2 --level 10 --split miehe" "--degree 2 --level 10 --split none" "--degree 4 --level 9 --split miehe" "--degree 4 --level 9 --split none"; do
  tag=$(echo $cfg | tr -d ' -')
  ncu --metrics $M --clock-control none -k regex:"k_sweep|k_apply" --csv python tools/prof_apply.py $cfg --reps 1 > gpurun_out/fp64_ncu_$tag.csv 2>&1
done
