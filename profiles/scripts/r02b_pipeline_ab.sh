# A/B: Adam fused with the next slice's cull (bench --pipeline, k_adam_cull, pipelined planes) vs separate kernels
for v in plain pipe3 pipe2 plain pipe3 pipe2; do
  case $v in plain) P=; M=3;; pipe3) P=--pipeline; M=3;; pipe2) P=--pipeline; M=2;; esac
  GPK_ADAM_CULL_MINB=$M timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-batched $P > gpurun_out/pipe_$v.log 2>&1
  echo "$v $(python tests/_stages.py gpurun_out/pipe_$v.log)"
done
