"""Probe: pinned H2D bandwidth on the box, with and without GPU-local CPU affinity (not a test)."""
import os
import subprocess
import sys

import torch


def sweep(tag):
    cs = torch.cuda.Stream()
    for mb in (0.25, 1, 4, 16, 64):
        n = int(mb * (1 << 20)) // 4
        h = torch.ones(n).pin_memory()
        d = torch.empty(n, device="cuda")
        for _ in range(3):
            d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(cs):
                e0.record(cs)
                d.copy_(h, non_blocking=True)
                e1.record(cs)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        med = ts[len(ts) // 2]
        print(f"{tag:10s} {mb:6.2f} MB  median {med * 1e3:8.1f} us  {mb * 1.048576e-3 / med:6.1f} GB/s  "
              f"min {ts[0] * 1e3:8.1f} us", flush=True)


print("affinity before:", sorted(os.sched_getaffinity(0))[:8], "... n =", len(os.sched_getaffinity(0)))
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
print(subprocess.run(["lscpu"], capture_output=True, text=True).stdout[:1500])
torch.cuda.init()
sweep("default")
import pynvml  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(int(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0] or 0))
try:
    pynvml.nvmlDeviceSetCpuAffinity(h)
    print("affinity after:", sorted(os.sched_getaffinity(0))[:8], "... n =", len(os.sched_getaffinity(0)))
except Exception as e:  # noqa: BLE001
    print("set affinity failed:", e)
sweep("gpu-local")
sys.stdout.flush()
