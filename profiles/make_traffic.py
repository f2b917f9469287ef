"""Write profiles/ncu_traffic.json from the `ncu --set full` captures of
profiles/run_ncu.sh (four BETWEEN windows per layout, first warm-up step of
`bench.py --profile`) and the algorithmic bytes of a bench.py JSON line.

    python profiles/make_traffic.py PROF_VBS.ncu-rep PROF_BS.ncu-rep BENCH.json TAG
"""
import csv
import json
import subprocess
import sys

WINDOWS = ("0.001", "0.01", "0.1", "0.5")
TILES = (1 << 28) // 1024
METRICS = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
           "smsp__inst_executed.sum", "sm__inst_issued.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread")


def kernels(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          ",".join(METRICS)], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        v = {}
        for m in METRICS:
            i = h.index(m)
            x = float(r[i].replace(",", ""))
            u = units[i]
            scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}.get(u, 1.0)
            v[m] = x * scale if "bytes" in m else x
        res.append(v)
    return res


def main(rep_v, rep_b, bench_json, tag):
    line = json.loads(open(bench_json).read().strip().splitlines()[-1])
    n = line["config"]["rows_per_gpu"]
    out = {"source": f"ncu --set full --clock-control none, profiles/run_ncu.sh (first warm-up "
                     f"step of bench.py --profile), capture {tag}",
           "note": "traffic = dram__bytes_read.sum + dram__bytes_write.sum per launch; mean over "
                   "the four BETWEEN windows (bench.py's roofline.traffic). alg_bytes = the "
                   "reference-stats algorithmic bytes of SURVEY.md 8(d) (bench.py)."}
    for layout, rep in (("ppvbs", rep_v), ("byteslice", rep_b)):
        ks = kernels(rep)
        assert len(ks) == 4, (rep, len(ks))
        per = {}
        for w, k in zip(WINDOWS, ks):
            abpc = line["layouts"][layout]["windows"][w]["alg_bytes_per_code"]
            rd, wr = k["dram__bytes_read.sum"], k["dram__bytes_write.sum"]
            per[w] = {"dram_bytes": int(rd + wr), "alg_bytes": int(round(abpc * n)),
                      "dram_read": int(rd), "dram_write": int(wr),
                      "ncu_us": round(k["gpu__time_duration.sum"] / 1e3
                                      if k["gpu__time_duration.sum"] > 1e4
                                      else k["gpu__time_duration.sum"], 2),
                      "warp_instr_per_tile": round(k["smsp__inst_executed.sum"] / TILES, 1),
                      "issue_active_pct": round(k["sm__inst_issued.avg.pct_of_peak_sustained_active"], 1),
                      "warps_active_pct": round(k["sm__warps_active.avg.pct_of_peak_sustained_active"], 1),
                      "regs": int(k["launch__registers_per_thread"])}
        out[layout] = int(sum(p["dram_bytes"] for p in per.values()) / 4)
        out[layout + "_per_window"] = per
    json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if not k.endswith("window")}))


if __name__ == "__main__":
    main(*sys.argv[1:5])
