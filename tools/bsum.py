"""Summarise a bench.py JSON line: headline, roofline, per-window us per layout."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("value", d["value"], "ms/step", d["ms_per_step"], "frac", d["roofline"]["frac"],
      "e2e", (d.get("e2e") or {}).get("value"))
for k, v in d["layouts"].items():
    print(f"  {k:10s} {v['gcodes_s']:8.1f} Gcodes/s  frac {v.get('frac')}  us:",
          [round(x["us"], 1) for x in v["windows"].values()])
