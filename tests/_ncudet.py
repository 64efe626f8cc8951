"""Print selected ncu details metrics per kernel: python tests/_ncudet.py rep.ncu-rep [regex]"""
import csv, subprocess, sys
rep = sys.argv[1]
cmd = ["ncu", "-i", rep, "--page", "details", "--csv"]
if len(sys.argv) > 2:
    cmd += ["-k", "regex:" + sys.argv[2]]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
want = {'Duration', 'Registers Per Thread', 'Achieved Occupancy', 'DRAM Throughput', 'Executed Ipc Active',
        'Warp Cycles Per Issued Instruction', 'Compute (SM) Throughput', 'Block Limit Registers', 'L2 Hit Rate'}
r = csv.reader(out.splitlines())
h = next(r)
for row in r:
    d = dict(zip(h, row))
    if d.get('Metric Name') in want:
        print(d['ID'], d['Kernel Name'][:40], d['Metric Name'], d['Metric Value'], d['Metric Unit'])
