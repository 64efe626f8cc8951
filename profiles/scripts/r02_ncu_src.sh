# source-level stall sampling of the slice kernels (one U2 step, C2)
set -x
timeout 600 ncu --set full --import-source on --sampling-interval 0 --clock-control none \
  -k regex:"k_(decide|raster_fwd|raster_bwd|ssim_fwd|chain)$" --launch-skip 5 --launch-count 5 \
  -o gpurun_out/r2_src python tests/profile_train.py 3 plain > gpurun_out/r2_ncu_src.log 2>&1
echo done
