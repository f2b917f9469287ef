"""Per-kernel SASS breakdown of an ncu report: warp instructions per 1024-row
tile by opcode and by CUDA source line (the SASS rows are attributed to the
source line printed before them).
  python profiles/sass_lines.py REPORT [TILES] [NLINES] [KERNEL_INDEX]"""
import collections
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
tiles = float(sys.argv[2]) if len(sys.argv) > 2 else 262144
nl = int(sys.argv[3]) if len(sys.argv) > 3 else 40
kidx = int(sys.argv[4]) if len(sys.argv) > 4 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
rows_all = list(csv.reader(out.splitlines()))
first_file = next(r[1] for r in rows_all if r and r[0] == "File Path")
kernels, cur = [], None
for r in rows_all:
    if r and r[0] == "File Path" and r[1] == first_file:
        cur = []
        kernels.append(cur)
    cur.append(r)
rows = kernels[kidx]
ops, lines = collections.Counter(), collections.Counter()
fname, src = "?", "?"
ie = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        ie = r.index("Instructions Executed")
        continue
    if r[0]:  # cuda source row
        src = f"{fname}:{r[0]:>4} {r[1].strip()[:80]}"
        continue
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[3].strip())
    try:
        n = int(r[ie] or 0)
    except (ValueError, TypeError):
        continue
    if m:
        ops[m.group(2)] += n
        lines[src] += n
print(f"kernel {kidx} of {len(kernels)}")
tot = sum(ops.values())
print(f"warp-instr per tile {tot / tiles:.1f}")
print(" ".join(f"{o}:{n / tiles:.1f}" for o, n in ops.most_common(24)))
for s, n in lines.most_common(nl):
    print(f"{n / tiles:7.1f} {s}")
