# launch list of the W=8 union-compacted DP step at C2 (rank 0 on one GPU)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dpc2w8_launches.csv \
  python tests/dp_projection.py --config c2 --worlds 8 --steps 2 --warmup 1 > gpurun_out/dpc2w8_ncu.log 2>&1
