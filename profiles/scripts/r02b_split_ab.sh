# A/B: Adam split around the render (GPK_ADAM_SPLIT) on the current slice kernels
for cfg in "0 0" "1 0" "1 592" "1 1184"; do
  set -- $cfg
  GPK_ADAM_SPLIT=$1 GPK_ADAM_REST_CTAS=$2 timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-batched > gpurun_out/split_$1_$2.log 2>&1
  echo "split=$1 ctas=$2 $(python tests/_stages.py gpurun_out/split_$1_$2.log)"
done
