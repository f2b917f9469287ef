"""Print the headline and per-window µs of a bench.py JSON line read from stdin."""
import json
import sys

d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print(d["value"], {k: [w["us"] for w in v["windows"].values()] for k, v in d["layouts"].items()})
