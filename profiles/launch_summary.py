"""Per-kernel totals of an ncu launch list (--csv --metrics gpu__time_duration.sum,dram__bytes_*):
kernel | launches | total us | mean us | DRAM rd MB | DRAM wr MB (means per launch).
    python profiles/launch_summary.py LAUNCHES.csv [OUT.txt]"""
import collections
import csv
import re
import sys

path = sys.argv[1]
with open(path) as f:
    lines = [l for l in f if l.startswith('"')]
cur = collections.OrderedDict()
for x in csv.DictReader(lines):
    cur.setdefault((int(x["ID"]), x["Kernel Name"]), {})[x["Metric Name"]] = float(
        x["Metric Value"].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for (_, name), m in cur.items():
    k = re.sub(r"\(.*$", "", name.replace("bsb::", "").replace("void ", ""))
    a = agg[k]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0) / 1e3
    a[2] += m.get("dram__bytes_read.sum", 0.0) / 1e6
    a[3] += m.get("dram__bytes_write.sum", 0.0) / 1e6
out = ["kernel | launches | total us | mean us | DRAM rd MB | DRAM wr MB"]
for k, (n, us, rd, wr) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    out.append(f"{k} | {n} | {us:.0f} | {us / n:.1f} | {rd / n:.1f} | {wr / n:.1f}")
text = "\n".join(out) + "\n"
if len(sys.argv) > 2:
    open(sys.argv[2], "w").write(text)
else:
    sys.stdout.write(text)
