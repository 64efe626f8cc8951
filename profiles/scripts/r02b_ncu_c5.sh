# source-level capture of the C5 (2048^2, 8M) slice kernels: one U2 step
set -x
timeout 900 ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none \
  -k regex:"k_(decide|raster_fwd|raster_bwd|ssim_fwd|chain|filter|sort_pass|pair_records|super_scan|gather)" --launch-skip 12 --launch-count 12 \
  -o gpurun_out/r3_c5 python tests/profile_train.py 3 plain c5 > gpurun_out/r3_c5.log 2>&1
echo done
