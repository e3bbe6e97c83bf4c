# Round-1 final profiles, part b: the fused LMS kernels and the one-launch small-array path.
tag=r01f; out=gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active \
  --clock-control none --csv --log-file $out/${tag}_lmsf_launches.csv python scripts/prof_kernels.py lms_fused > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"fused_tc|lms_cuts|batched_select" -c 4 \
  -o $out/${tag}_lmsf python scripts/prof_kernels.py lms_fused > $out/${tag}_lmsf.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:"exact_cluster" -c 1 \
  -o $out/${tag}_small python scripts/time_small.py 100000 > $out/${tag}_small.log 2>&1
python scripts/time_small.py 100000 > $out/${tag}_small_time.txt 2>&1
python scripts/bench_lms.py --cmp > $out/${tag}_lms.json 2>/dev/null
ls -la $out
