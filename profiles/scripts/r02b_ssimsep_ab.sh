# A/B at C5: the SSIM backward fused into the raster backward's prologue vs k_ssim_bwd (32 x 32 tiles) + dL/dI in HBM
for v in "" 4096 "" 4096; do
  GPK_SSIM_FUSE_MAX_TILES=$v timeout 300 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu-baseline --no-batched > gpurun_out/sep_$v.log 2>&1
  echo "max_tiles=${v:-inf} $(python tests/_stages.py gpurun_out/sep_$v.log)"
done
GPK_SSIM_FUSE_MAX_TILES=0 timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-batched > gpurun_out/sep_c2.log 2>&1
echo "C2 separate: $(python tests/_stages.py gpurun_out/sep_c2.log)"
