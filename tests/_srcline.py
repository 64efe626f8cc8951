"""Per-CUDA-source-line stall samples of a kernel from an ncu report (SASS
samples mapped to lines through the cubin's line table).
python tests/_srcline.py <rep> <kernel> <object.o> [top] [inst]   (inst: weigh by warp
instructions executed instead of stall samples)"""
import csv
import re
import subprocess
import sys
from collections import defaultdict

rep, kern, obj = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
col = "Instructions Executed" if len(sys.argv) > 5 and sys.argv[5] == "inst" else "Warp Stall Sampling (All Samples)"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:(^|::){kern}(<|$|\\()",
                      "--print-source", "sass"], capture_output=True, text=True).stdout.splitlines()
r = csv.reader(out)
next(r)
h = next(r)
rows = [dict(zip(h, x)) for x in r]
rows = [x for x in rows if x.get("Address", "").startswith("0x")]
seen, first = set(), []
for x in rows:
    if x["Address"] in seen:
        break
    seen.add(x["Address"])
    first.append(x)
base = int(first[0]["Address"], 16)
samp = {int(x["Address"], 16) - base: int(x[col] or 0) for x in first}
# line table of the kernel's function in the object's cubin
cub = subprocess.run(["cuobjdump", "-xelf", "all", __import__("os").path.abspath(obj)], capture_output=True, text=True, cwd="/tmp")
dis = subprocess.run(f"nvdisasm --print-line-info /tmp/{obj.split('/')[-1].replace('.o','')}*.cubin",
                     shell=True, capture_output=True, text=True).stdout
lines_by_off = {}
cur_fn, cur_line, in_fn = None, None, False
for ln in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        in_fn = re.search(re.escape(kern) + r"[IE]", m.group(1)) is not None  # (not k_filter_multi for k_filter)
        continue
    m = re.search(r"//## File \"([^\"]+)\", line (\d+)", ln)
    if m:
        cur_line = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and in_fn:
        lines_by_off[int(m.group(1), 16)] = cur_line
agg = defaultdict(int)
for off, v in samp.items():
    agg[lines_by_off.get(off, "?")] += v
tot = sum(agg.values()) or 1
print("samples", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{v:7d} {100 * v / tot:5.1f}%  {k}")
