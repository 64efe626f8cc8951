set -x
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/r2_c4_launches.csv python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2_c4_ncu.log 2>&1
echo done
