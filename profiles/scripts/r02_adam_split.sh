# A/B of the Adam split (k_adam_rest beside the render) on the C2 probe
set -x
timeout 300 python -m pytest tests/test_train_gpu.py tests/test_configs_gpu.py -k "train or c2_u2" -q -x -p no:cacheprovider > gpurun_out/r2_split_tests.log 2>&1
for cfg in "GPK_ADAM_SPLIT=0" "GPK_ADAM_REST_CTAS=-1" "GPK_ADAM_REST_CTAS=148" "GPK_ADAM_REST_CTAS=296" "GPK_ADAM_REST_CTAS=592"; do
  env $cfg timeout 200 python tests/batch_probe.py c2 40 > gpurun_out/r2_split_$(echo $cfg | tr '=' '_').log 2>&1
done
echo done
