#!/bin/bash
# Round 2 captures on one GPU, into gpurun_out/r02_*: the bench line, the launch list of one timed
# bench step (ncu, cold, serialised), ncu --set full of the headline kernels (sample, init, radix),
# of the paper's-method Kelley passes (pass_kernel / seg_pass_kernel) and of the fused LMS pass.
out=gpurun_out
timeout 900 python bench.py > $out/r02_bench.json 2> $out/r02_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $out/r02_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-lms --no-side \
  > $out/r02_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"init_seg|sample_grid|sample_cluster|pool_gather|radix_coop|vbin" -c 8 \
  -o $out/r02_full python scripts/prof_kernels.py select > $out/r02_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"seg_pass|pass_kernel" -c 4 \
  -o $out/r02_kelley python scripts/time_kelley.py 30 uniform --reps 1 > $out/r02_kelley_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_tc -s 1 -c 1 \
  -o $out/r02_lmsf python scripts/prof_kernels.py lms_fused > $out/r02_lmsf.log 2>&1
python scripts/launch_table.py $out/r02_launches.csv --sel 4 > $out/r02_launch_table.md 2>&1
tail -c 300 $out/r02_bench.json
