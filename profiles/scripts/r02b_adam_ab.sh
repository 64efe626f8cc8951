# A/B: k_adam plain vs software-pipelined (5 / 4 CTAs per SM)
for v in 0 1 2 0 1 2; do
  GPK_ADAM_PIPE=$v timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-batched > gpurun_out/adam_$v.log 2>&1
  echo "pipe=$v $(python tests/_stages.py gpurun_out/adam_$v.log)"
done
