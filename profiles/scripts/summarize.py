"""Summaries committed under profiles/ from ncu captures in gpurun_out/.

    python profiles/scripts/summarize.py full  <rep.ncu-rep> <config> <out.json>
    python profiles/scripts/summarize.py launches <launches.csv> <out.json>

`full`: per-kernel duration, DRAM/L2 bytes, shared wavefronts, utilisation
(% of peak), warp instructions, launch shape, occupancy, IPC and the top four
stall reasons of a `--set full` capture (cold caches, serialised). `launches`:
per-kernel launch counts and times of a `--metrics gpu__time_duration.sum`
launch list, our kernels (namespace gpk) apart from library ones."""
import csv
import io
import json
import re
import subprocess
import sys
from collections import OrderedDict, defaultdict

HBM_PEAK = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6543.4) if __import__("os").path.exists(
    "MEASURED_PEAKS.json") else 6543.4
PCT = ["dram__throughput", "lts__t_sectors", "l1tex__data_pipe_lsu_wavefronts_mem_shared",
       "sm__pipe_fma_cycles_active", "sm__inst_executed_pipe_xu", "sm__throughput"]


def short(name):
    name = re.sub(r"^(void )?(gpk::)?(\(anonymous namespace\)::|<unnamed>::|unnamed>::)?", "", name)
    return name.split("(")[0]


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def full(rep, config, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    ks = []
    for x in rows[2:]:
        d = dict(zip(h, x))
        g = lambda k: num(d.get(k, ""))  # noqa: E731
        dur = g("gpu__time_duration.sum")  # ns or us per the unit row
        unit = dict(zip(h, rows[1])).get("gpu__time_duration.sum", "ns")
        dur_us = dur / 1000.0 if unit == "ns" else (dur * 1000.0 if unit == "ms" else dur)
        rd, wr = g("dram__bytes_read.sum") or 0.0, g("dram__bytes_write.sum") or 0.0
        units = dict(zip(h, rows[1]))

        def nbytes(k):
            v, u = g(k) or 0.0, units.get(k, "byte")
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)

        rd, wr, l2 = nbytes("dram__bytes_read.sum"), nbytes("dram__bytes_write.sum"), nbytes("lts__t_bytes.sum")
        stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): num(v)
                  for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_")
                  and k.endswith("_per_issue_active.ratio") and num(v) is not None}
        top = OrderedDict(sorted(((k, v) for k, v in stalls.items() if k not in ("selected",)),
                                 key=lambda kv: -kv[1])[:4])
        ks.append(OrderedDict(
            kernel=short(d["Kernel Name"]), duration_us=dur_us, dram_read_bytes=rd, dram_write_bytes=wr,
            l2_bytes=l2, smem_wavefronts=g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
            dram_gbs=(rd + wr) / (dur_us * 1e3), dram_frac_of_measured_peak=(rd + wr) / (dur_us * 1e3) / HBM_PEAK,
            l2_gbs=l2 / (dur_us * 1e3),
            pct_of_peak={p: g(p + (".avg.pct_of_peak_sustained_active" if p.startswith("sm__pipe") or "pipe_xu" in p
                                   else ".avg.pct_of_peak_sustained_elapsed")) for p in PCT},
            warp_instructions=g("smsp__inst_executed.sum"), registers=g("launch__registers_per_thread"),
            grid=g("launch__grid_size"), block=g("launch__block_size"),
            achieved_occupancy_pct=g("sm__warps_active.avg.pct_of_peak_sustained_active"),
            ipc_per_sm=g("sm__inst_executed.avg.per_cycle_active"), top_stalls=top))
    tot = sum(k["duration_us"] for k in ks)
    for k in ks:
        k["share_of_step"] = round(k["duration_us"] / tot, 4)
    json.dump(OrderedDict(capture=rep.split("/")[-1], config=config,
                          note="ncu --set full --clock-control none, cold caches, serialised",
                          sum_us=tot, kernels=ks), open(out, "w"), indent=1)


def launches(path, out):
    rows = list(csv.reader(open(path)))
    h = None
    ours, other = defaultdict(list), defaultdict(list)
    for r in rows:
        if r and r[0] == "ID":
            h = r
            continue
        if h and len(r) == len(h):
            d = dict(zip(h, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            us = num(d["Metric Value"]) / (1000.0 if d.get("Metric Unit", "ns") in ("ns", "nsecond") else 1.0)
            name = d["Kernel Name"]
            (ours if "gpk::" in name or "unnamed>::k_" in name else other)[short(name)[:48]].append(us)
    tot = sum(sum(v) for v in ours.values())
    res = OrderedDict(source=path.split("/")[-1],
                      note="ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised per launch)",
                      our_kernels=OrderedDict(sorted(((k, dict(launches=len(v), total_us=sum(v), mean_us=sum(v) / len(v),
                                                                share_of_our_kernels=sum(v) / tot))
                                                      for k, v in ours.items()), key=lambda kv: -kv[1]["total_us"])),
                      other_kernels={k: dict(launches=len(v), total_us=sum(v)) for k, v in other.items()})
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        launches(sys.argv[2], sys.argv[3])
