# A/B of prebuilt library variants at C4 (voxelizer) + voxel parity tests on the last variant
L=paper_2603_20611_b200/_lib
cp $L/libgpile_b200.so /tmp/lib_keep.so
for v in $VARIANTS; do
  cp $L/alts/lib_$v.so $L/libgpile_b200.so
  timeout 300 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab4_$v.log 2>&1
  echo "$v C4 $(tail -1 gpurun_out/ab4_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d.get("e2e",{}).get("value"))')"
done
cp /tmp/lib_keep.so $L/libgpile_b200.so
timeout 900 python -m pytest tests -m gpu -q -x -k "vox or c4" 2>&1 | tail -3
