"""Print ms/step and stage times of bench JSON lines: python tests/_stages.py log..."""
import json, sys
for f in sys.argv[1:]:
    L = [l for l in open(f).read().splitlines() if l.startswith("{")]
    if not L:
        print(f, "no JSON line"); continue
    d = json.loads(L[-1])
    print(f, round(d["ms_per_step"], 4), "steady", round(d.get("steady_state", {}).get("ms_per_step", 0), 4),
          "e2e", round(d["e2e"].get("ms_median", 0), 4), {k: round(v * 1000, 1) for k, v in d.get("stage_ms_per_step", {}).items()})
