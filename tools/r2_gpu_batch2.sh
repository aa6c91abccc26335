# round-2 GPU batch 2: reference suite (6 files), distributed tests, smoke launch list, setup phases
mkdir -p gpurun_out
PFF_REFSUITE=1 timeout 1200 python -m pytest tests/ref_suite -q -rA > gpurun_out/refsuite_b2.log 2>&1; echo "refsuite rc=$?" >> gpurun_out/refsuite_b2.log
timeout 600 python -m pytest tests/test_distributed.py -q > gpurun_out/dist_b2.log 2>&1; echo "rc=$?" >> gpurun_out/dist_b2.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_launches.csv 2> gpurun_out/smoke_ncu.err
timeout 300 python tools/prof_setup2.py > gpurun_out/setup_phases.txt 2>&1
