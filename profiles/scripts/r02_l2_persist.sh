# A/B: an L2 set-aside for the cull's evict-last parameter lines (read again by Adam)
set -x
for mb in 0 48 80; do
  GPK_L2_PERSIST_MB=$mb timeout 200 python tests/batch_probe.py c2 40 > gpurun_out/r2_l2p_$mb.log 2>&1
done
GPK_L2_PERSIST_MB=48 timeout 200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_l2p_ncu48.csv python tests/profile_train.py 4 plain > /dev/null 2>&1
echo done
timeout 600 python bench.py --no-cpu-baseline --steps 200 > gpurun_out/r2_e2e_check.log 2>&1
timeout 600 python -m pytest tests/test_configs_gpu.py -k "voxelize_backward" -q -s -p no:cacheprovider > gpurun_out/r2_vbwd.log 2>&1
