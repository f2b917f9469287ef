"""L2 sectors requested per CUDA source line of one kernel of an ncu report
(column "L2 Theoretical Sectors Global"), to find which loads move the bytes.
  python profiles/sectors_lines.py REPORT KERNEL_INDEX [NLINES]"""
import collections
import csv
import subprocess
import sys

rep, kidx = sys.argv[1], int(sys.argv[2])
nl = int(sys.argv[3]) if len(sys.argv) > 3 else 20
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
hdr = next(r for r in rows if r and r[0] == "Line No")
ci = hdr.index("L2 Theoretical Sectors Global")
lines = collections.Counter()
fname, src = "?", "?"
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 2 and r[0] and r[0] != "Line No" and r[2] == "-":
        src = f"{fname}:{r[0]:>4} {r[1].strip()[:90]}"
        continue
    if r[0] == "" and len(r) > ci:
        try:
            lines[src] += int(float(r[ci] or 0))
        except ValueError:
            pass
tot = sum(lines.values())
print(f"kernel {kidx}: {tot} sectors = {tot * 32 / 1e6:.1f} MB")
for s, n in lines.most_common(nl):
    print(f"{n * 32 / 1e6:9.1f} MB  {s}")
