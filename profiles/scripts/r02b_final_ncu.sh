# The round's committed profiles (round 2, final code): one U2 step (C2) with --set full plus the
# utilisation metrics, and the launch list of a default bench run.
set -x
M=lts__t_bytes.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed
timeout 900 ncu --set full --metrics $M --import-source on --clock-control none \
  -k regex:"k_(filter|decide|raster_fwd|raster_bwd|ssim_fwd|chain|adam|gather)" --launch-skip 9 --launch-count 9 \
  -o gpurun_out/r2b_final_full python tests/profile_train.py 3 plain > gpurun_out/r2b_final_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r2b_final_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-batched > gpurun_out/r2b_final_launch_run.log 2>&1
timeout 900 ncu --set full --metrics $M --import-source on --clock-control none \
  -k regex:"k_(filter|decide|raster_fwd|raster_bwd|ssim_fwd|chain|adam|sort_pass|pair_records|super_scan)" --launch-skip 13 --launch-count 13 \
  -o gpurun_out/r2b_final_c5 python tests/profile_train.py 3 plain c5 > gpurun_out/r2b_final_c5.log 2>&1
echo done
