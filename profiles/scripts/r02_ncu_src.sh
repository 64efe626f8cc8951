# source-level stall sampling of the slice kernels (one U2 step, C2)
set -x
timeout 600 ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none \
  -k regex:"k_(decide|raster_fwd|raster_bwd|ssim_fwd|chain)$" --launch-skip 5 --launch-count 5 \
  -o gpurun_out/r2_src python tests/profile_train.py 3 plain > gpurun_out/r2_ncu_src.log 2>&1
echo done
timeout 300 python bench.py --config c4 --steps 6 --warmup 2 --no-cpu-baseline > gpurun_out/r2_bench_c4b.log 2>&1
timeout 300 python -m pytest tests/test_voxel_gpu.py tests/test_configs_gpu.py -k "voxel or c4" -q -p no:cacheprovider > gpurun_out/r2_vox_tests.log 2>&1
