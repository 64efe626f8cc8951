set -x
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_lazy_launches.csv python tests/profile_train.py 24 plain > gpurun_out/r2_lazy_launches.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_(filter|lazy_survivors|lazy_window)" --launch-skip 60 --launch-count 3 -o gpurun_out/r2_lazy_full python tests/profile_train.py 24 plain > gpurun_out/r2_lazy_full.log 2>&1
echo done
