# the stand-alone photometric_loss (k_ssim_fwd + k_ssim_bwd) at C5 through the API, and the GPU tests
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
GPK_SSIM_FUSE_MAX_TILES=0 timeout 300 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu-baseline --no-batched > gpurun_out/apiloss_c5.log 2>&1
echo "$(python tests/_stages.py gpurun_out/apiloss_c5.log)"
