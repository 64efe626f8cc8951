# A/B: k_chain's early trigger + Adam's first-plane prefetch before its PDL wait
for v in 1 0 1 0; do
  GPK_CHAIN_EARLY_TRIGGER=$v timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-batched > gpurun_out/early_$v.log 2>&1
  echo "early=$v $(python tests/_stages.py gpurun_out/early_$v.log)"
done
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
