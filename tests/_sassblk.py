"""Group a kernel's SASS (ncu source page) into runs of equal execution count."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern, "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
r = csv.reader(out)
next(r)
h = next(r)
rows = [dict(zip(h, x)) for x in r]
rows = [x for x in rows if x.get('Instructions Executed', '').isdigit()]
# the page may list the function twice; keep the first copy
seen = set(); first = []
for x in rows:
    if x['Address'] in seen:
        break
    seen.add(x['Address']); first.append(x)
rows = first
tot = sum(int(x['Instructions Executed']) for x in rows)
print('total', tot, 'instructions', len(rows))
runs = []; cur = None
for i, x in enumerate(rows):
    c = int(x['Instructions Executed'])
    st = int(x['Warp Stall Sampling (All Samples)'] or 0)
    if cur and cur[0] == c:
        cur[2] = i; cur[3] += c; cur[4] += st
    else:
        cur = [c, i, i, c, st]; runs.append(cur)
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
for c, a, b, t, st in sorted(runs, key=lambda z: -z[3])[:n]:
    print(f'{a:5d}-{b:5d} per={c:8d} total={t:9d} ({100*t/tot:4.1f}%) stalls={st:5d}',
          rows[a]['Source'].strip()[:46], '...', rows[b]['Source'].strip()[:40])
if len(sys.argv) > 4:
    lo, hi = map(int, sys.argv[4].split(':'))
    for i in range(lo, hi):
        print(i, rows[i]['Instructions Executed'], rows[i]['Warp Stall Sampling (All Samples)'], rows[i]['Source'].strip())
