set -x
timeout 600 ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none \
  -k regex:"k_(decide|raster_fwd|raster_bwd|ssim_fwd|chain|filter)" --launch-skip 6 --launch-count 6 \
  -o gpurun_out/r3_src python tests/profile_train.py 3 plain > gpurun_out/r3_src.log 2>&1
echo done
