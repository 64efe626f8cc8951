# launch lists: the single-GPU U2 step and the W=1 / W=8 union steps (C2)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dpc2_launches.csv \
  python tests/dp_projection.py --config c2 --worlds 1,8 --steps 2 --warmup 1 > gpurun_out/dpc2_ncu.log 2>&1
