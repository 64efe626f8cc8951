# A/B: SSIM tiles started as their raster tiles finish (GPK_SSIM_OVERLAP=1) vs at the kernel boundary
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
for v in 1 0 1 0; do
  GPK_SSIM_OVERLAP=$v timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-batched > gpurun_out/ssim_$v.log 2>&1
  echo "overlap=$v $(python tests/_stages.py gpurun_out/ssim_$v.log)"
done
GPK_SSIM_OVERLAP=1 timeout 300 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu-baseline --no-batched > gpurun_out/ssim_c5.log 2>&1
echo "c5 $(python tests/_stages.py gpurun_out/ssim_c5.log)"
