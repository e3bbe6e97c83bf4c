T=$1
timeout 600 python -m pytest tests/test_gpu_lms.py -x -q > gpurun_out/${T}_lmstest.log 2>&1
python scripts/bench_lms.py > gpurun_out/${T}_lms.json 2>&1
ncu --set full --import-source on --clock-control none -k regex:fused_tc_kernel --launch-skip 2 --launch-count 2 -o gpurun_out/${T}_lmsf python scripts/prof_lms.py > gpurun_out/${T}_ncu.log 2>&1
