"""Summaries of a round-2 cfg5 ncu capture (tools/cfg5_probe.py on one
2^29-row segment per column, profiles/run_ncu_cfg5.sh): per kernel launch
the duration, DRAM bytes, instruction and pipe counters, and the per-query
DRAM traffic file the bench's roofline reads (profiles/ncu_traffic_cfg5.json).
  python profiles/summarize_r2.py REPORT OUT_TXT OUT_JSON"""
import csv
import json
import subprocess
import sys

rep, out_txt, out_json = sys.argv[1:4]
metrics = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(metrics)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
ki = h.index("Kernel Name")
idx = {m: h.index(m) for m in metrics}
units = {m: rows[1][idx[m]] for m in metrics}
lines = ["kernel | us | DRAM rd MB | DRAM wr MB | Minst | issue% | warps% | alu% | fma% | dram% | regs"]
recs = []
for r in rows[2:]:
    def f(m):
        v = float(r[idx[m]].replace(",", ""))
        u = units[m]
        if m.startswith("dram__bytes"):
            v = v * {"Gbyte": 1e3, "Mbyte": 1.0, "Kbyte": 1e-3, "byte": 1e-6}.get(u, 1.0)
        if m == "gpu__time_duration.sum":
            v = v * {"ms": 1e3, "us": 1.0, "usecond": 1.0, "ns": 1e-3, "nsecond": 1e-3}.get(u, 1.0)
        return v
    rec = {"kernel": r[ki][:60], **{m: f(m) for m in metrics}}
    recs.append(rec)
    lines.append(f"{rec['kernel']} | {rec['gpu__time_duration.sum']:.1f} | "
                 f"{rec['dram__bytes_read.sum']:.0f} | {rec['dram__bytes_write.sum']:.0f} | "
                 f"{rec['smsp__inst_executed.sum'] / 1e6:.0f} | "
                 f"{rec['smsp__issue_active.avg.pct_of_peak_sustained_active']:.0f} | "
                 f"{rec['sm__warps_active.avg.pct_of_peak_sustained_active']:.0f} | "
                 f"{rec['sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active']:.0f} | "
                 f"{rec['sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active']:.0f} | "
                 f"{rec['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']:.0f} | "
                 f"{rec['launch__registers_per_thread']:.0f}")
open(out_txt, "w").write("\n".join(lines) + "\n")
# probe order (tools/cfg5_probe.py --reps=1: 2 warm-ups + 1 timed launch per
# query): u0 x3, u1 x3, z0 x3, z1 x3, then 3 AND chains (bs_conj_kernel + the
# two epilogue-masked vbs_ds_kernel legs); the last launch of each group
traffic = {}
for nm, k in (("u0", 2), ("u1", 5), ("z0", 8), ("z1", 11)):
    if k < len(recs):
        traffic[nm] = int((recs[k]["dram__bytes_read.sum"] + recs[k]["dram__bytes_write.sum"]) * 1e6)
conj = [i for i, r in enumerate(recs) if "bs_conj_kernel" in r["kernel"]]
if conj and conj[-1] + 3 <= len(recs):
    traffic["and4"] = int(sum(r["dram__bytes_read.sum"] + r["dram__bytes_write.sum"]
                              for r in recs[conj[-1]:conj[-1] + 3]) * 1e6)
json.dump({"source": rep, "unit": "bytes per launch (dram read + write, ncu, one 2^29-row "
                                  "segment per column)", **traffic}, open(out_json, "w"), indent=1)
print(open(out_txt).read())
print(json.load(open(out_json)))
