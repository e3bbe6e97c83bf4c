#!/bin/bash
# One GPU: the bench line, the ncu launch list of one timed bench step (cold, serialised) and one
# `ncu --set full` capture of the path's kernels, into gpurun_out/<tag>_*.  Usage: capture_profiles.sh TAG
tag=${1:-r01}
out=gpurun_out
timeout 900 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $out/${tag}_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu \
  > $out/${tag}_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"init_seg|cut_pass|sample_cluster|seg_pass|radix_round|exact_cluster" -c 12 \
  -o $out/${tag}_full python scripts/prof_kernels.py select > $out/${tag}_full.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"residual_tc|batched_select|pack_rows|lts_reduce" -c 5 \
  -o $out/${tag}_lms python scripts/prof_kernels.py lms > $out/${tag}_lms.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fused_tc|lms_cuts|batched_select" -c 4 \
  -o $out/${tag}_lmsf python scripts/prof_kernels.py lms_fused > $out/${tag}_lmsf.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:"exact_cluster" -c 2 \
  -o $out/${tag}_small python scripts/time_small.py 100000 > $out/${tag}_small.log 2>&1
tail -c 400 $out/${tag}_bench.json
