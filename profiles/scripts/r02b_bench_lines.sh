# round-2 final bench lines on one B200 (each a separate process)
set -x
timeout 900 python bench.py > gpurun_out/r02b_bench_c2.log 2>&1
timeout 600 python bench.py --unit u1 --no-cpu-baseline > gpurun_out/r02b_bench_u1.log 2>&1
timeout 600 python bench.py --batch 8 --no-cpu-baseline > gpurun_out/r02b_bench_b8.log 2>&1
timeout 900 python bench.py --config c3 > gpurun_out/r02b_bench_c3.log 2>&1
timeout 900 python bench.py --config c5 --steps 50 > gpurun_out/r02b_bench_c5.log 2>&1
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 > gpurun_out/r02b_bench_c4.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02b_bench_ref.log 2>&1
echo done
