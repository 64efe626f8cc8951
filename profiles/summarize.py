"""Summarize ncu captures into the tracked files under profiles/.

    python profiles/summarize.py full  <capture.ncu-rep> <out.json> [--config c2]
    python profiles/summarize.py launches <launches.csv> <out.json>

`full`: one `ncu --set full` capture of one training step (tests/profile_train.py)
-> per kernel: duration, DRAM bytes read/written, instructions, registers,
achieved occupancy, IPC, top warp-stall reasons. Also merges the kernel's
DRAM bytes into profiles/ncu_summary.json (read by bench.py for the
roofline `traffic` field).
`launches`: the `--metrics gpu__time_duration.sum` launch list of a bench run
-> per kernel name: launch count, total / mean duration (cold, serialised:
shares, not absolute step times).
"""
from __future__ import annotations

import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

HERE = Path(__file__).resolve().parent
try:
    HBM_GBS = float(json.loads((HERE.parent / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
except Exception:  # the profiling recipe's fallback
    HBM_GBS = 6650.0
PCT = ["dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors.avg.pct_of_peak_sustained_elapsed",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum", *PCT,
           "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__grid_size", "launch__block_size", "sm__inst_executed.avg.per_cycle_active"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3,
        "us": 1.0, "ns": 1e-3, "ms": 1e3}


def short(name: str) -> str:
    m = re.search(r"(k_[a-z_]+)(<[^>]*>)?\(", name)
    return m.group(1) + (m.group(2) or "") if m else name[:60]


def ncu_raw(rep: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[head.index("Kernel Name")])}
        for m in METRICS:
            if m not in head:
                d[m] = None
                continue
            i = head.index(m)
            v = float(r[i].replace(",", "")) if r[i] not in ("", "n/a") else None
            if v is not None and units[i] in UNIT:
                v *= UNIT[units[i]]
            d[m] = v
        res.append(d)
    return res


def stalls(rep: str, kernel: str, top: int = 4) -> dict:
    out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:(^|::){kernel}(<|$)", "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    head, r = rows[0], rows[2]
    items = {}
    for i, h in enumerate(head):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                items[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(r[i].replace(",", ""))
            except ValueError:
                pass
    tot = sum(items.values()) or 1.0
    return {k: round(v / tot, 3) for k, v in sorted(items.items(), key=lambda x: -x[1])[:top]}


def full(rep: str, out: str, config: str) -> None:
    rows = ncu_raw(rep)
    kernels = []
    for d in rows:
        kernels.append({
            "kernel": d["kernel"],
            "duration_us": d["gpu__time_duration.sum"],
            "dram_read_bytes": d["dram__bytes_read.sum"],
            "dram_write_bytes": d["dram__bytes_write.sum"],
            "l2_bytes": d["lts__t_bytes.sum"],
            "smem_wavefronts": d["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"],
            # achieved DRAM bandwidth against MEASURED_PEAKS.json's copy peak, and
            # ncu's own utilisation of the DRAM, L2, shared-memory, FMA and
            # MUFU (XU) pipes (percent of peak)
            "dram_gbs": (((d["dram__bytes_read.sum"] or 0) + (d["dram__bytes_write.sum"] or 0)) /
                         (d["gpu__time_duration.sum"] * 1e3)) if d["gpu__time_duration.sum"] else None,
            "dram_frac_of_measured_peak": (((d["dram__bytes_read.sum"] or 0) + (d["dram__bytes_write.sum"] or 0)) /
                                           (d["gpu__time_duration.sum"] * 1e3) / HBM_GBS)
            if d["gpu__time_duration.sum"] else None,
            "l2_gbs": ((d["lts__t_bytes.sum"] or 0) / (d["gpu__time_duration.sum"] * 1e3))
            if d["gpu__time_duration.sum"] else None,
            "pct_of_peak": {m.split(".")[0]: d[m] for m in PCT},
            "warp_instructions": d["smsp__inst_executed.sum"],
            "registers": d["launch__registers_per_thread"],
            "grid": d["launch__grid_size"], "block": d["launch__block_size"],
            "achieved_occupancy_pct": d["sm__warps_active.avg.pct_of_peak_sustained_active"],
            "ipc_per_sm": d["sm__inst_executed.avg.per_cycle_active"],
            "top_stalls": stalls(rep, d["kernel"].split("<")[0]),
        })
    total = sum(k["duration_us"] or 0 for k in kernels)
    for k in kernels:
        k["share_of_step"] = round((k["duration_us"] or 0) / total, 4) if total else None
    Path(out).write_text(json.dumps({"capture": Path(rep).name, "config": config,
                                     "note": "ncu --set full --clock-control none, cold caches, serialised "
                                             "(one U2 training step of tests/profile_train.py, the third)",
                                     "sum_us": total, "kernels": kernels}, indent=1))
    # traffic per launch for bench.py's roofline field
    summ = HERE / "ncu_summary.json"
    s = json.loads(summ.read_text()) if summ.exists() else {}
    cfg = s.setdefault(config, {})
    for k in kernels:
        name = k["kernel"].split("<")[0]
        cfg[name] = {"dram_bytes_per_launch": (k["dram_read_bytes"] or 0) + (k["dram_write_bytes"] or 0),
                     "duration_us_cold": k["duration_us"], "ipc_per_sm": k.get("ipc_per_sm"),
                     "issue_frac": (k["ipc_per_sm"] / 4.0) if k.get("ipc_per_sm") is not None else None,
                     "source": Path(out).name}
    summ.write_text(json.dumps(s, indent=1))


def launches(csv_path: str, out: str) -> None:
    text = Path(csv_path).read_text()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    agg = defaultdict(lambda: {"launches": 0, "total_us": 0.0})
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", "")) * UNIT.get(r.get("Metric Unit", "usecond"), 1.0)
        a = agg[short(r["Kernel Name"])]
        a["launches"] += 1
        a["total_us"] += v
    ours = {k: v for k, v in agg.items() if k.startswith("k_")}
    tot = sum(v["total_us"] for v in ours.values()) or 1.0
    res = {k: {**v, "mean_us": v["total_us"] / v["launches"], "share_of_our_kernels": v["total_us"] / tot}
           for k, v in sorted(ours.items(), key=lambda x: -x[1]["total_us"])}
    others = {k: v for k, v in agg.items() if not k.startswith("k_")}
    Path(out).write_text(json.dumps({"source": Path(csv_path).name,
                                     "note": "ncu --metrics gpu__time_duration.sum --clock-control none "
                                             "(cold, serialised per launch)",
                                     "our_kernels": res,
                                     "other_kernels": {k[:50]: v for k, v in others.items()}}, indent=1))


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    cfg = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "c2"
    (full(src, dst, cfg) if mode == "full" else launches(src, dst))
