# A/B of backward variants (prebuilt libraries swapped in): base (scalar x loop), packed x pairs at 5 / 6 CTAs per SM
L=paper_2603_20611_b200/_lib
cp $L/libgpile_b200.so /tmp/lib_keep.so
for v in base mb5 mb6 base mb5 mb6; do
  cp $L/alts/lib_$v.so $L/libgpile_b200.so
  timeout 300 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu-baseline --no-batched > gpurun_out/bwd_$v.log 2>&1
  timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-batched > gpurun_out/bwdc2_$v.log 2>&1
  echo "$v $(python tests/_stages.py gpurun_out/bwd_$v.log) | $(python tests/_stages.py gpurun_out/bwdc2_$v.log)"
done
cp /tmp/lib_keep.so $L/libgpile_b200.so
