tag=r01f; out=gpurun_out
timeout 900 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $out/${tag}_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-lms \
  > $out/${tag}_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none \
  -k regex:"init_seg|sample_cluster|radix_round" -c 5 \
  -o $out/${tag}_full python scripts/prof_kernels.py select > $out/${tag}_full.log 2>&1
ls -la $out
