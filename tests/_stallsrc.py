"""Top stalled SASS lines of a kernel in an ncu report: python tests/_stallsrc.py rep kernel [n]"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:(^|::){kern}(<|$)",
                      "--print-source", "sass"], capture_output=True, text=True).stdout.splitlines()
r = csv.reader(out); next(r); h = next(r)
rows = [dict(zip(h, x)) for x in r]
rows = [x for x in rows if x.get('Instructions Executed', '').isdigit()]
seen = set(); first = []
for x in rows:
    if x['Address'] in seen:
        break
    seen.add(x['Address']); first.append(x)
rows = first
tot = sum(int(x['Warp Stall Sampling (All Samples)'] or 0) for x in rows)
print('total stall samples', tot, 'instructions', sum(int(x['Instructions Executed']) for x in rows))
top = sorted(range(len(rows)), key=lambda i: -int(rows[i]['Warp Stall Sampling (All Samples)'] or 0))[:n]
for i in sorted(top):
    x = rows[i]
    print(i, x['Warp Stall Sampling (All Samples)'], x['Instructions Executed'], x['Source'].strip()[:90])
