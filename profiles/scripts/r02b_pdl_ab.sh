# A/B: PDL with an explicit early trigger (griddepcontrol.launch_dependents at kernel entry) vs the implicit one
cp paper_2603_20611_b200/_lib/libgpile_b200.so /tmp/lib_base.so
for v in base early base early; do
  if [ $v = early ]; then cp paper_2603_20611_b200/_lib/alt/libgpile_b200.so paper_2603_20611_b200/_lib/libgpile_b200.so; else cp /tmp/lib_base.so paper_2603_20611_b200/_lib/libgpile_b200.so; fi
  timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-batched > gpurun_out/pdl_$v.log 2>&1
  echo "$v $(python tests/_stages.py gpurun_out/pdl_$v.log)"
done
cp /tmp/lib_base.so paper_2603_20611_b200/_lib/libgpile_b200.so
