import json, sys
for f in sys.argv[1:]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f.split('/')[-1], round(d['ms_per_step'], 4), round(d['value']), 'e2e', round(d['e2e']['value']),
          {k: round(v * 1e3, 1) for k, v in d['stage_ms_per_step'].items()}, d['roofline']['kernel'],
          round(d['roofline']['frac'], 3))
