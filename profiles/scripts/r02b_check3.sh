# gpu tests + C2 / C3 / C5 quick bench lines (stage times)
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-batched > gpurun_out/bench_c2.log 2>&1
timeout 300 python bench.py --config c3 --steps 100 --warmup 10 --no-cpu-baseline --no-batched > gpurun_out/bench_c3.log 2>&1
timeout 300 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu-baseline --no-batched > gpurun_out/bench_c5.log 2>&1
