set -x
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/r2_batch_launches2.csv python tests/profile_batch.py 3 8 > gpurun_out/r2_ncu_batch2.log 2>&1
timeout 600 ncu --set full --metrics lts__t_bytes.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --import-source on --clock-control none -k regex:"k_(filter|decide|raster_fwd|raster_bwd|ssim_fwd|chain|adam)" --launch-skip 9 --launch-count 9 -o gpurun_out/r2_train_full2 python tests/profile_train.py 3 plain > gpurun_out/r2_ncu_full2.log 2>&1
timeout 300 ncu --set full --metrics lts__t_bytes.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --import-source on --clock-control none -k regex:"k_adam_batch|k_filter_multi" --launch-skip 2 --launch-count 2 -o gpurun_out/r2_batch_full python tests/profile_batch.py 3 8 > gpurun_out/r2_ncu_batchfull.log 2>&1
echo done
