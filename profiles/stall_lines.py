"""Stall samples of one reason by CUDA source line (with the top SASS rows).
    python profiles/stall_lines.py REPORT [stall_column] [n]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
col = sys.argv[2] if len(sys.argv) > 2 else "stall_long_sb"
nl = int(sys.argv[3]) if len(sys.argv) > 3 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
fname, src, ci = "?", "?", None
agg, sass = collections.Counter(), collections.defaultdict(list)
for r in csv.reader(out.splitlines()):
    if not r or r[0] == "Function Name":
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        ci = r.index(col)
        continue
    if r[0]:
        src = f"{fname}:{r[0]} {r[1].strip()[:70]}"
        continue
    try:
        v = int(r[ci] or 0)
    except (ValueError, TypeError):
        continue
    agg[src] += v
    if v:
        sass[src].append((v, r[3].strip()[:60]))
print(col, "total", sum(agg.values()))
for s, n in agg.most_common(nl):
    print(f"{n:6d} {s}")
    for v, t in sorted(sass[s], reverse=True)[:2]:
        print(f"         {v:5d} {t}")
