# C4 bench line + its launch list (same command under ncu, timing-only metric)
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 > gpurun_out/r02b_bench_c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_c4_launches.csv python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
tail -1 gpurun_out/r02b_bench_c4.log
