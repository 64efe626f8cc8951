# A/B of the L2 warm-up of Adam's moments (GPK_L2_PREFETCH=0 off, 1 m, 2 m+v) at C2 and C5
for r in 1 2; do for v in 0 1 2; do
  GPK_L2_PREFETCH=$v timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-batched > gpurun_out/pf2_$v.log 2>&1
  GPK_L2_PREFETCH=$v timeout 300 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu-baseline --no-batched > gpurun_out/pf5_$v.log 2>&1
  echo "pf=$v C2 $(python tests/_stages.py gpurun_out/pf2_$v.log | cut -d' ' -f2-) | C5 $(python tests/_stages.py gpurun_out/pf5_$v.log | cut -d' ' -f2-)"
done; done
