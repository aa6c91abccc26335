# compute-sanitizer over every Q2 sweep-kernel form (tools/sanitize_sweep.py)
mkdir -p gpurun_out
for t in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_sweep.py > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$?" >> gpurun_out/sanitize_$t.log
done
