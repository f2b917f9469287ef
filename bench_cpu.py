"""CPU baselines beside the GPU numbers (SURVEY.md §8(d) "CPU baseline"):
the oracle port of the reference algorithms (oracle/, the checker -- never
the product) timed on the GPU box's host cores for the lookup, execute and
advisor paths, at threads=1 (the paper's one-core methodology) and with all
cores where the reference partitions work (scans; ThreadPoolExecutor,
SPEC.md:613).  Each entry states its sample; every sample is a bounded slice
of the BASELINE config's own generator so the run stays within seconds.
"""

from __future__ import annotations

import os
import platform
import statistics
import time

import numpy as np


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def _timed(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def lookup_baseline(m: int = 1 << 22, n_ids: int = 1 << 18) -> dict:
    """cfg3 lookups on the first m rows of the cfg3 columns: ByteSlice
    (uniform 24-bit, identity codes) and PP-VBS (Zipf 1.0 / 2^20, decoded
    through the padded-code dictionary): random ids (unsorted, with
    replacement) and a 20% bitvector; Mrows/s."""
    import oracle as O
    codes = np.random.default_rng(3).integers(0, 1 << 24, m)
    planes = O.bs_build(codes, 24)
    vals = O.gen_zipf(1.0, 20, m, 4)
    d = O.OracleDict.from_values(vals, "prefix_preserving")
    col = O.vbs_build(*d.row_codes(d.encode_rows(vals)))
    ids = np.random.default_rng(5).integers(0, m, n_ids)
    sel = np.flatnonzero(np.random.default_rng(6).random(m) < 0.20)
    out = {}
    for name, rows in (("ids_unsorted", ids), ("bits_20pct", sel)):
        tb = _timed(lambda rows=rows: O.bs_lookup(planes, 24, rows))
        tv = _timed(lambda rows=rows: d.decode_padded(O.vbs_lookup(col, rows)[0]))
        out[f"byteslice/{name}"] = round(len(rows) / tb / 1e6, 3)
        out[f"ppvbs/{name}"] = round(len(rows) / tv / 1e6, 3)
    got = d.decode_padded(O.vbs_lookup(col, ids)[0])
    assert np.array_equal(got, vals[ids]), "oracle lookup self-check"
    return {"unit": "Mrows/s", "cores": 1, "kind": "port", "values": out,
            "sample": f"first {m} rows of the cfg3 columns; {n_ids} random ids and a 20% "
                      f"bitvector; numpy oracle (vectorised gathers, one thread)"}


def execute_baseline(m: int = 1 << 21, threads: int = 1) -> dict:
    """The cfg4 query (4-predicate AND, ByteSlice first as engine.conj_order,
    then 3 projections decoded + SUM) on the first m rows of the cfg4 columns
    with the oracle; rows/s of the query (codes scanned / s as well)."""
    import oracle as O
    rng = {nm: np.random.default_rng(100 + i) for i, nm in enumerate(
        ("u16", "u24", "u20", "u32"))}
    raw = {"u16": rng["u16"].integers(0, 1 << 16, m), "u24": rng["u24"].integers(0, 1 << 24, m),
           "u20": rng["u20"].integers(0, 1 << 20, m),
           "u32": rng["u32"].integers(-(1 << 31), 1 << 31, m),
           "z12": O.gen_zipf(1.0, 12, m, 109), "z16": O.gen_zipf(1.5, 16, m, 110),
           "z24": O.gen_zipf(1.0, 24, m, 112)}
    lay = {"u16": "bs", "u24": "bs", "u20": "bs", "u32": "bs", "z12": "vbs", "z16": "vbs",
           "z24": "vbs"}
    cols = {}
    for nm, v in raw.items():
        if lay[nm] == "bs":
            d = O.OracleDict.from_values(v, "fixed")
            cols[nm] = ("bs", d, O.bs_build(d.encode_rows(v), d.width_bits))
        else:
            d = O.OracleDict.from_values(v, "prefix_preserving")
            cols[nm] = ("vbs", d, O.vbs_build(*d.row_codes(d.encode_rows(v))))

    def q(nm, x):
        s = np.sort(raw[nm])
        return int(s[min(m - 1, int(x * m))])
    preds = [("u16", "LT", 32768, None), ("u24", "GE", q("u24", 0.6), None),
             ("z12", "BETWEEN", q("z12", 0.2), q("z12", 0.9)), ("z16", "LE", q("z16", 0.7), None)]
    enc = [(nm, cols[nm][1].encode_literal(op, lo, hi)) for nm, op, lo, hi in preds]

    def run():
        run_m = None
        for nm, p in enc:
            kind, d, c = cols[nm]
            run_m = (O.bs_scan(c, d.width_bits, m, p, run_m, threads=threads)[0] if kind == "bs"
                     else O.vbs_scan(c, p, run_m, threads=threads)[0])
        rows = O.words_to_rows(run_m, m)
        res = {}
        for nm in ("u32", "z24", "u20"):
            kind, d, c = cols[nm]
            if kind == "bs":
                res[nm] = d.decode_ranks(O.bs_lookup(c, d.width_bits, rows)[0].astype(np.int64))
            else:
                res[nm] = d.decode_padded(O.vbs_lookup(c, rows)[0])
        return rows, res
    rows, res = run()
    flags = ((raw["u16"] < 32768) & (raw["u24"] >= preds[1][2]) & (raw["z12"] >= preds[2][2])
             & (raw["z12"] <= preds[2][3]) & (raw["z16"] <= preds[3][2]))
    assert np.array_equal(rows, np.flatnonzero(flags)), "oracle execute self-check"
    assert int(res["u32"].sum()) == int(raw["u32"][flags].sum())
    t = _timed(run, reps=2)
    return {"value": round(m / t / 1e6, 3), "unit": "Mrows/s (query over the sample)",
            "gcodes_s": round(4 * m / t / 1e9, 5), "cores": threads, "kind": "port",
            "sample": f"first {m} rows of the cfg4 predicate / projection columns (7 of 16); "
                      f"AND of 4 predicates pipelined + 3 projections decoded + SUM(u32); "
                      f"numpy oracle, {threads} thread(s)"}


def advisor_baseline(m: int = 1 << 20) -> dict:
    """advise_column(cost='bytes', count=100) (advisor.py:119-150) with the
    oracle on the first m rows of the cfg4 z16 column (Zipf 1.5 / 2^16):
    seconds per column, 1 thread."""
    import oracle as O
    v = O.gen_zipf(1.5, 16, m, 110)
    t0 = time.perf_counter()
    r = O.advise_column(v, count=100, cost="bytes")
    t = time.perf_counter() - t0
    return {"value": round(t, 3), "unit": "s per column", "cores": 1, "kind": "port",
            "chosen": r["chosen"],
            "sample": f"first {m} rows of cfg4's z16 column; 100 literals x 2 layouts, bytes "
                      f"cost; numpy oracle, one thread"}


def cpu_extras() -> dict:
    out = {"cpu_model": cpu_model(), "os_cpu_count": os.cpu_count()}
    for name, fn in (("lookup", lookup_baseline), ("execute", execute_baseline),
                     ("advisor", advisor_baseline)):
        t0 = time.perf_counter()
        try:
            out[name] = fn()
        except Exception as exc:  # noqa: BLE001 - recorded, not swallowed
            out[name] = {"error": f"{type(exc).__name__}: {exc}"}
        out[name]["wall_s"] = round(time.perf_counter() - t0, 1)
    try:
        thr = os.cpu_count() or 1
        t0 = time.perf_counter()
        out["execute_all_cores"] = execute_baseline(threads=thr)
        out["execute_all_cores"]["wall_s"] = round(time.perf_counter() - t0, 1)
    except Exception as exc:  # noqa: BLE001
        out["execute_all_cores"] = {"error": f"{type(exc).__name__}: {exc}"}
    return out


if __name__ == "__main__":
    import json
    print(json.dumps(cpu_extras(), indent=1))
