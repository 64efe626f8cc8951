# A/B: the fused loss finished in k_ssim_fwd (ticket) vs the raster backward's CTA 0
for v in 0 1 0 1; do
  GPK_LOSS_IN_FWD=$v GPK_BENCH_E2E_DEBUG=1 timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-batched > gpurun_out/ab_$v.log 2>&1
  python -c "
import json
L=[l for l in open('gpurun_out/ab_$v.log').read().splitlines() if l.startswith('{')]
d=json.loads(L[-1]); print('loss_in_fwd=$v', d['ms_per_step'], d['e2e']['ms_median'])
"; grep 'e2e debug' gpurun_out/ab_$v.log
done
