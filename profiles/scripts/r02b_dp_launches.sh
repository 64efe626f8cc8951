# launch list of the W=8 union-compacted DP step (rank 0 on one GPU, C5)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dp8_launches.csv \
  python tests/dp_projection.py --config c5 --worlds 8 --steps 2 --warmup 1 > gpurun_out/dp8_ncu.log 2>&1
