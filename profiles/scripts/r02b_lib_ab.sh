# A/B of prebuilt library variants (paper_2603_20611_b200/_lib/alts/lib_<v>.so) at C2 and C5
L=paper_2603_20611_b200/_lib
cp $L/libgpile_b200.so /tmp/lib_keep.so
for v in $VARIANTS; do
  cp $L/alts/lib_$v.so $L/libgpile_b200.so
  timeout 300 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu-baseline --no-batched > gpurun_out/ab5_$v.log 2>&1
  timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-batched > gpurun_out/ab2_$v.log 2>&1
  echo "$v C5 $(python tests/_stages.py gpurun_out/ab5_$v.log | cut -d' ' -f2-) | C2 $(python tests/_stages.py gpurun_out/ab2_$v.log | cut -d' ' -f2-)"
done
cp /tmp/lib_keep.so $L/libgpile_b200.so
