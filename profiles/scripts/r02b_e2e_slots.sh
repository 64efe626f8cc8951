# gpu tests, then the C2 bench three times (e2e with alternating target slots)
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
for r in 1 2 3; do
  timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-batched > gpurun_out/slots_$r.log 2>&1
  python tests/_stages.py gpurun_out/slots_$r.log
done
