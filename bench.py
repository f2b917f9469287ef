#!/usr/bin/env python
"""ByteStore hot-path benchmark on B200.

Default workload (BASELINE.json configs[4], the config its metric is quoted
on at 1/2/4/8 B200): cfg5 -- a 4-column x 2^32-row table (2 uniform int32
columns as ByteSlice, 2 Zipf(1.1)/2^24 columns as PP-VBS), stored as 8 fixed
2^29-row segments per column and row-range sharded over the GPUs (strong
scaling: total work fixed).  One step = u0 < q(.1), u1 >= q(.5), z0 BETWEEN
q(.8) AND q(.95), z1 <= q(.6) and their 4-way AND over the rank's segments,
plus the AND's global row-id compaction, then one NCCL all_gather of the
per-rank counts.  Metric: codes scanned per second, whole job.  See
bench_cfg5.py; every segment's result words are checked against a device
filter of the raw values before timing.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--workload cfg5|cfg2]

At N = 1 the line also carries configs.cfg2 (2^28-row Zipf(1.2) column, the
four BETWEEN windows on PP-VBS and ByteSlice -- the round-1 headline),
configs.cfg3 (lookups), configs.cfg1 and configs.cfg4.  `--impl reference`
times the CPU oracle port of the reference algorithm on the host cores on a
bounded sample of the same workload (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ZIPF_S, DOMAIN_BITS, SEED = 1.2, 20, 42
WINDOWS = (0.001, 0.01, 0.1, 0.5)
METRIC = "scan Gcodes/s (PP-VBS + ByteSlice BETWEEN scans, cfg2)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="default: 30 (cfg5) / 400 (cfg2)")
    ap.add_argument("--warmup", type=int, default=None, help="default: 5 (cfg5) / 20 (cfg2)")
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--workload", choices=("cfg5", "cfg2"), default="cfg5",
                    help="cfg5 (default): 4 x 2^32-row table row-range sharded over the "
                         "GPUs; cfg2: the 2^28-row Zipf column, 8 BETWEEN scans per GPU")
    ap.add_argument("--seg-log2", type=int, default=29,
                    help="cfg5 segment rows (8 segments per column; 29 = 2^32 rows)")
    ap.add_argument("--cfg5-streams", type=int, default=5, choices=(1, 2, 3, 4, 5))
    ap.add_argument("--rows-log2", type=int, default=28)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-lookup", action="store_true")
    ap.add_argument("--lookup-steps", type=int, default=10)
    ap.add_argument("--no-extra", action="store_true", help="skip cfg1/cfg4/cfg5")
    ap.add_argument("--streams", type=int, default=8, choices=(1, 2, 4, 8),
                    help="graph step: the 8 scans on this many forked streams")
    ap.add_argument("--no-graph", action="store_true",
                    help="time the step as eager launches instead of a CUDA graph replay")
    ap.add_argument("--deep-mode", default="auto",
                    help="PP-VBS deep layout: auto|packed|sliced")
    ap.add_argument("--profile", action="store_true",
                    help="short run for ncu: no clocks/e2e/cpu baseline")
    return ap.parse_args()


def window_bounds(uniq: np.ndarray, counts: np.ndarray, n: int):
    """BETWEEN q(1-p-m) AND q(1-m), m = min(p, .25), q = nearest rank."""
    cum = np.cumsum(counts)

    def q(x):
        return int(uniq[np.searchsorted(cum, min(n - 1, int(x * n)), side="right")])

    out = []
    for p in WINDOWS:
        m = min(p, 0.25)
        out.append((p, q(1 - p - m), q(1 - m)))
    return out


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join("/tmp", f"bsb_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu)], stdout=self.fh, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, flag in zip(names, parts[5:9]):
                if flag.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------- column build
def build_cfg2(n: int, deep_mode: str = "auto"):
    """Generate + encode the cfg2 column on the device (untimed)."""
    import torch

    from paper_2209_00220_b200 import ColumnKind, Dictionary, FrequencyTable, ZipfSpec
    from paper_2209_00220_b200.byteslice import build_byteslice
    from paper_2209_00220_b200.datagen import gen_zipf_device
    from paper_2209_00220_b200.dictionary import freq_table_and_ranks
    from paper_2209_00220_b200.vbs import build_vbs

    t0 = time.perf_counter()
    vals = gen_zipf_device(ZipfSpec(ZIPF_S, DOMAIN_BITS, n, SEED))
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    u, c, ranks = freq_table_and_ranks(vals)
    table = FrequencyTable(u.cpu().numpy(), c.cpu().numpy(), ColumnKind.NUMERIC)
    d_ppe = Dictionary.build(table, "prefix_preserving")
    d_fix = Dictionary.build(table, "fixed")
    codes, lens = d_ppe.row_codes_device(ranks)
    col_v = build_vbs(codes, lens, deep_mode=deep_mode)
    col_b = build_byteslice(ranks, d_fix.assignment.width_bits)
    del codes, lens
    torch.cuda.synchronize()
    t_enc = time.perf_counter() - t0
    return {"values": vals, "ranks": ranks, "table": table, "d_ppe": d_ppe, "d_fix": d_fix,
            "col_v": col_v, "col_b": col_b, "t_gen": t_gen, "t_encode": t_enc}


def alg_bytes_for(col, layout, pred, d_exist):
    """Algorithmic bytes from the reference-identical stats depth."""
    from paper_2209_00220_b200.byteslice import scan_byteslice
    from paper_2209_00220_b200.roofline import scan_alg_bytes
    from paper_2209_00220_b200.vbs import scan_vbs
    if layout == "ppvbs":
        _, st = scan_vbs(col, pred)
        st = st.materialize()
        return scan_alg_bytes(st.block_depth, "ppvbs", col.max_len, d_exist), st
    _, st = scan_byteslice(col, pred)
    st = st.materialize()
    return scan_alg_bytes(st.block_depth, "byteslice", col.n_slices), st


# ------------------------------------------------------------ CPU oracle
def cpu_reference_setup(n_full: int, m: int, threads: int):
    """Host-only prep of the cfg2 column sample for the oracle port: full
    dictionary from chunked PCG64 draws + bincount, first m rows encoded."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle as O
    cdf = np.cumsum(O.zipf_pmf(ZIPF_S, 1 << DOMAIN_BITS))
    cdf[-1] = 1.0
    rng = np.random.default_rng(SEED)
    counts = np.zeros(1 << DOMAIN_BITS, np.int64)
    sample = None
    chunk = 1 << 24
    pool = ThreadPoolExecutor(threads)
    done = 0
    while done < n_full:
        k = min(chunk, n_full - done)
        u = rng.random(k)
        parts = np.array_split(u, threads)
        vs = list(pool.map(lambda a: np.searchsorted(cdf, a, side="right"), parts))
        v = np.concatenate(vs)
        if sample is None:
            sample = v[:m].astype(np.int64)
        counts += np.bincount(v, minlength=1 << DOMAIN_BITS)
        done += k
    pool.shutdown()
    uniq = np.flatnonzero(counts).astype(np.int64)
    w = counts[uniq]
    dppe = O.OracleDict(uniq, w, "prefix_preserving")
    dfix = O.OracleDict(uniq, w, "fixed")
    ranks = np.searchsorted(uniq, sample)
    col = O.vbs_build(*dppe.row_codes(ranks))
    planes = O.bs_build(ranks, dfix.width_bits)
    wins = window_bounds(uniq, w, n_full)
    preds = []
    for p, lo, hi in wins:
        preds.append(("ppvbs", p, dppe.encode_literal("BETWEEN", lo, hi)))
        preds.append(("byteslice", p, dfix.encode_literal("BETWEEN", lo, hi)))
    return col, planes, dfix.width_bits, preds, len(sample)


def cpu_reference_pass(setup, threads):
    import oracle as O
    col, planes, w, preds, m = setup
    t = {}
    for layout, p, pr in preds:
        t0 = time.perf_counter()
        if layout == "ppvbs":
            O.vbs_scan(col, pr, threads=threads)
        else:
            O.bs_scan(planes, w, m, pr, threads=threads)
        t[(layout, p)] = time.perf_counter() - t0
    return t


def cpu_baseline(n_full, m, threads, reps=3):
    setup = cpu_reference_setup(n_full, m, threads)
    cpu_reference_pass(setup, threads)  # warm-up
    totals = [sum(cpu_reference_pass(setup, threads).values()) for _ in range(reps)]
    tmed = statistics.median(totals)
    # the paper's one-core methodology: the same sample on 1 thread
    t1 = sum(cpu_reference_pass(setup, 1).values())
    return {"value": round(8 * m / tmed / 1e9, 6), "unit": "Gcodes/s", "cores": threads,
            "kind": "port",
            "sample": f"first {m} rows of the cfg2 column (dictionary from all {n_full} rows), "
                      f"4 BETWEEN windows x 2 layouts, numpy oracle with {threads} threads, "
                      f"median of {reps} passes after 1 warm-up",
            "threads_1": {"value": round(8 * m / t1 / 1e9, 6), "unit": "Gcodes/s", "cores": 1,
                          "sample": "same sample, one pass on 1 thread"}}


def cfg5_reference_setup(m: int):
    """Host-only cfg5 sample for the oracle port: the first m rows of chunk 0
    of every column (the reference generators, the same seeds as the GPU
    arm).  Dictionaries come from the expected 2^32-row Zipf counts
    rint(pmf * 2^32) (a host bincount of 2^32 draws would take ~15 min);
    u0/u1 quantiles are the sample's nearest ranks."""
    import oracle as O
    import bench_cfg5 as C
    cols, preds = {}, {}
    pmf = O.zipf_pmf(C.ZIPF_S, 1 << C.ZIPF_BITS)
    w = np.rint(pmf * float(1 << 32)).astype(np.int64)
    uniq = np.flatnonzero(w).astype(np.int64)
    w = w[uniq]
    cum = np.cumsum(w)
    ntot = int(cum[-1])

    def qz(x):
        return int(uniq[np.searchsorted(cum, min(ntot - 1, int(x * ntot)), side="right")])
    for ci, (nm, kind) in enumerate(C.COLS):
        if kind == "uniform":
            v = C.gen_host(ci, kind, 0, m).astype(np.int64)
            codes = (v + (1 << 31)).astype(np.uint64)
            cols[nm] = ("bs", O.bs_build(codes, 32))
            srt = np.sort(codes)
            x = 0.10 if nm == "u0" else 0.50
            q = int(srt[min(m - 1, int(x * m))])
            preds[nm] = O.pred_compare("LT" if nm == "u0" else "GE", q, 4)
        else:
            v = O.gen_zipf(C.ZIPF_S, C.ZIPF_BITS, m, C.chunk_seed(ci, 0))
            d = O.OracleDict(uniq, w, "prefix_preserving")
            cols[nm] = ("vbs", O.vbs_build(*d.row_codes(d.encode_rows(v))))
            preds[nm] = (d.encode_literal("BETWEEN", qz(0.80), qz(0.95)) if nm == "z0"
                         else d.encode_literal("LE", qz(0.60)))
    return cols, preds, m


def cfg5_reference_pass(setup, threads: int) -> float:
    import oracle as O
    cols, preds, m = setup

    def one(nm, mask):
        kind, c = cols[nm]
        if kind == "bs":
            return O.bs_scan(c, 32, m, preds[nm], mask, threads=threads)[0]
        return O.vbs_scan(c, preds[nm], mask, threads=threads)[0]
    t0 = time.perf_counter()
    for nm in ("u0", "u1", "z0", "z1"):
        one(nm, None)
    run = None
    for nm in ("u0", "u1", "z0", "z1"):
        run = one(nm, run)
    O.words_to_rows(run, m)
    return time.perf_counter() - t0


def run_reference_cfg5(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    probe = cfg5_reference_setup(1 << 18)
    cfg5_reference_pass(probe, threads)
    per_row = cfg5_reference_pass(probe, threads) / (1 << 18)
    budget = 120.0 / max(1, args.steps + args.warmup)
    m = max(1 << 14, min(int(budget / per_row) // 1024 * 1024, 1 << 24))
    setup = probe if m == (1 << 18) else cfg5_reference_setup(m)
    for _ in range(args.warmup):
        cfg5_reference_pass(setup, threads)
    total = sum(cfg5_reference_pass(setup, threads) for _ in range(args.steps))
    value = 8 * m * args.steps / total / 1e9
    sample = (f"first {m} rows of chunk 0 of each of the 4 cfg5 columns, the 5 queries "
              f"(AND pipelined) per step, numpy oracle port on {threads} threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC5, "value": round(value, 6), "unit": "Gcodes/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": "cfg5: 4 columns x 2^32 rows (u0,u1 uniform int32 ByteSlice "
                               "w=32; z0,z1 Zipf(1.1)/2^24 PP-VBS), 5 queries per step",
                   "rows": m, "rows_total": 8 << 29,
                   "sample": "bounded per-step sample (CPU)"},
        "cpu_baseline": {"value": round(value, 6), "unit": "Gcodes/s", "cores": threads,
                         "kind": "port", "sample": sample},
        "e2e": {"value": round(value, 6), "unit": "Gcodes/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}), flush=True)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n_full = 1 << args.rows_log2
    # size each step so warm-up + K steps take ~120 s of CPU time
    probe_m = 1 << 18
    setup = cpu_reference_setup(n_full, probe_m, threads)
    cpu_reference_pass(setup, threads)
    t_probe = sum(cpu_reference_pass(setup, threads).values())
    per_row = t_probe / probe_m
    budget = 120.0 / max(1, args.steps + args.warmup)
    m = int(budget / per_row) // 1024 * 1024
    m = max(1024, min(m, 1 << 24, n_full))
    setup = setup if m == probe_m else cpu_reference_setup(n_full, m, threads)
    for _ in range(args.warmup):
        cpu_reference_pass(setup, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cpu_reference_pass(setup, threads)
    total = time.perf_counter() - t0
    value = 8 * m * args.steps / total / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "Gcodes/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": "cfg2: Zipf(1.2)/2^20 column, BETWEEN p=0.1/1/10/50% on "
                               "PP-VBS and ByteSlice", "rows": m, "rows_full_column": n_full,
                   "sample": "bounded prefix sample per step (CPU)"},
        "cpu_baseline": {"value": round(value, 6), "unit": "Gcodes/s", "cores": threads,
                         "kind": "port",
                         "sample": f"first {m} rows of the 2^{args.rows_log2}-row cfg2 column"},
        "e2e": {"value": round(value, 6), "unit": "Gcodes/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- B200 arm
def run_b200(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # functional check of the N > 1 path on a one-GPU box (never a perf
    # number): BSB_FORCE_DEVICE=0 BSB_DIST_BACKEND=gloo puts every rank on
    # cuda:0 with host-staged collectives
    local = int(os.environ.get("BSB_FORCE_DEVICE", local))
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("BSB_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    try:
        if args.workload == "cfg5":
            out = run_cfg5(args, world, rank, local)
        else:
            out = run_cfg2(args, world, rank, local)
        if rank == 0 and out is not None:
            print(json.dumps(out), flush=True)
    finally:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()


METRIC5 = ("scan Gcodes/s (cfg5: 4 columns x 2^32 rows row-range sharded; u0<q10, u1>=q50, "
           "z0 BETWEEN q80,q95, z1<=q60 and their 4-way AND + global row ids)")
KERNEL5 = {"u0": "bs_scan_kernel<LT> (ByteSlice w=32, bit-plane sectors)",
           "u1": "bs_scan_kernel<GE> (ByteSlice w=32, bit-plane sectors)",
           "z0": "vbs_ds_kernel<BETWEEN> (PP-VBS SLICED, deep-row space)",
           "z1": "vbs_ds_kernel<LE, LM=2> (PP-VBS SLICED, deep-row space; the 1-byte-code rows "
                 "settled by the literal, no first-slice bytes read)",
           "and4": "bsb_conj_scan: bs_conj_kernel (u0 AND u1, TMA-staged, AND in registers) "
                   "+ z0 leg + z1 leg, each vbs_dsm_kernel (work compacted to the masked-in "
                   "blocks) when the running count is at most 6 % of the rows, else "
                   "vbs_ds_kernel<EPI> (running mask AND-ed in the epilogue); both are "
                   "launched, gated on the device-resident count"}


def run_cfg5(args, world, rank, local):
    """cfg5 headline (bench_cfg5.py): strong scaling over row-range shards."""
    import torch
    import torch.distributed as dist

    import bench_cfg5 as C
    from paper_2209_00220_b200 import _lib
    from paper_2209_00220_b200.roofline import hbm_peak

    _lib.load()
    seg_rows = 1 << args.seg_log2
    t0 = time.perf_counter()
    tab = C.Cfg5Table(world, rank, seg_rows)
    t_table = time.perf_counter() - t0
    step = C.Cfg5Step(tab, 1)
    step.run_query("and4", torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    cap = int(step.counts[C.QUERIES.index("and4")].sum().item())
    step.ids = torch.empty(max(cap, 1), dtype=torch.int64, device="cuda")
    t0 = time.perf_counter()
    sel = C.check_parity(tab, step)          # raises on any mismatch
    t_parity = time.perf_counter() - t0
    t0 = time.perf_counter()
    ab = C.alg_bytes(tab)
    t_alg = time.perf_counter() - t0
    cpu = None
    if rank == 0 and world == 1 and not args.profile and not args.no_cpu_baseline:
        thr = os.cpu_count() or 1
        cs = C.cpu_sample(tab, 1 << 22, thr)
        cpu = {"value": round(cs["all"], 6), "unit": "Gcodes/s", "cores": thr, "kind": "port",
               "sample": f"first {cs['rows']} rows of segment 0 of each column (global "
                         f"dictionaries and quantiles of the full table): the 5 cfg5 queries "
                         f"(AND pipelined) with the numpy oracle on {thr} threads, median "
                         f"after 1 warm-up",
               "threads_1": {"value": round(cs["one"], 6), "unit": "Gcodes/s", "cores": 1}}
        import bench_cpu
        cpu["cpu_model"] = bench_cpu.cpu_model()
        cpu["extras"] = bench_cpu.cpu_extras()
    tab.free_raw()
    # ---- the step as one CUDA graph (C ABI calls + two tiny torch reductions)
    nst = args.cfg5_streams
    streams = [torch.cuda.Stream() for _ in range(nst)]
    graph = None
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        capst = streams[0]
        capst.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(graph, stream=capst):
            for st in streams[1:]:
                st.wait_stream(capst)
            step.local(streams)
        torch.cuda.current_stream().wait_stream(capst)

    gath = torch.zeros(world, len(C.QUERIES), dtype=torch.int64, device="cuda")
    gath_list = list(gath.unbind(0))  # (gloo functional check only)
    nccl = world > 1 and dist.get_backend() == "nccl"

    def one_step():
        if graph is not None:
            graph.replay()
        else:
            cur = torch.cuda.current_stream()
            for st in streams:
                st.wait_stream(cur)
            step.local(streams)
            cur.wait_stream(streams[0])
        if world > 1 and nccl:
            dist.all_gather_into_tensor(gath, step.totals)
        elif world > 1:
            dist.all_gather(gath_list, step.totals)
        else:
            gath[0].copy_(step.totals)

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    if not args.profile:
        clocks.start()
        time.sleep(0.3)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0.record()
    for _ in range(args.steps):
        one_step()
    ev1.record()
    torch.cuda.synchronize()
    total_ms = ev0.elapsed_time(ev1)
    if world > 1:
        dist.barrier()
    clk = clocks.stop() if not args.profile else None
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    # the timed steps reproduce the checked counts; global counts and offsets
    got = gath.cpu().numpy()
    for qi, q in enumerate(C.QUERIES):
        if int(got[rank, qi]) != sel[q]:
            raise AssertionError(f"cfg5 {q}: timed count {got[rank, qi]} != checked {sel[q]}")
    glob = {q: int(got[:, qi].sum()) for qi, q in enumerate(C.QUERIES)}
    id_offset = int(got[:rank, C.QUERIES.index("and4")].sum())
    # ---- per-kernel (per C ABI call) durations for the roofline
    kt = C.kernel_times(step)
    S = len(tab.segs)
    peak, peak_src = hbm_peak(ROOT)
    queries = {}
    for q in C.QUERIES:
        gbs = ab[q] / S / (kt[q] * 1e-3) / 1e9
        queries[q] = {"kernel": KERNEL5[q], "us_per_segment": round(kt[q] * 1e3, 2),
                      "alg_bytes_per_code": round(ab[q] / (S * seg_rows), 4),
                      "alg_gbs": round(gbs, 1), "frac": round(gbs / peak, 4),
                      "selected_global": glob[q],
                      "predicate": tab.literals.get(q, "u0 AND u1 AND z0 AND z1")}
    # the dominant KERNEL: the single-predicate scans are one kernel each; the
    # AND is a chain of three (its legs run the same kernels as the singles)
    dom = max(("u0", "u1", "z0", "z1"), key=lambda q: kt[q])
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic_cfg5.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(dom)
        except (OSError, ValueError):
            traffic = None
    ms_step = total_ms / args.steps
    codes_per_step = 8 * tab.n_total
    value = codes_per_step / (ms_step * 1e-3) / 1e9
    whole = sum(ab.values())
    t5 = torch.tensor([float(whole)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t5)
    step_frac = float(t5.item()) / (ms_step * 1e-3) / 1e9 / (peak * world)
    e2e = None
    if not args.profile:
        e2e = measure_e2e_cfg5(tab, args.e2e_steps, world)
    if rank != 0:
        return None
    dq = queries[dom]
    out = {
        "metric": METRIC5, "value": round(value, 3), "unit": "Gcodes/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded numpy PCG64 draws with the reference generators; "
                "8 fixed chunks per column, identical at every N)",
        "config": {"workload": "cfg5: 4 columns x 2^32 rows (u0,u1 uniform int32 ByteSlice "
                               "w=32; z0,z1 Zipf(1.1)/2^24 PP-VBS with global dictionaries), "
                               "row-range sharded; 5 queries per step",
                   "rows_total": tab.n_total, "segments": C.N_CHUNKS, "segment_rows": seg_rows,
                   "segments_per_gpu": S, "codes_per_step": codes_per_step,
                   "parallelism": f"row-range shards x{world}" if world > 1 else "single GPU",
                   "collectives_per_step": "1 NCCL all_gather of 5 int64 counts per rank"
                                           if world > 1 else "none (N=1)",
                   "l2": f"inputs larger than L2 ({tab.col_bytes() / 1e9:.1f} GB of encoded "
                         f"columns per GPU)",
                   "launch": (f"CUDA graph of the rank's C ABI calls on {nst} forked streams"
                              if graph is not None else "eager C ABI calls")},
        "roofline": {"bound": "hbm", "kernel": dq["kernel"], "query": dom,
                     "achieved": dq["alg_gbs"], "peak": peak, "unit": "GB/s",
                     "frac": dq["frac"], "peak_source": peak_src, "traffic": traffic,
                     "traffic_source": "profiles/ncu_traffic_cfg5.json (ncu dram read+write "
                                       "per launch)" if traffic else None,
                     "alg_bytes_per_launch": int(ab[dom] / S),
                     "us_per_launch": dq["us_per_segment"],
                     # the kernel runs once alone and once as an AND leg per segment
                     "step_share_est": round(2 * kt[dom] / sum(kt.values()), 3),
                     "whole_step_frac": round(step_frac, 4)},
        "queries": queries,
        "parity": {"checked": "every segment's bitvector of every query == packed device "
                              "filter of its raw values; AND global row ids == filter rows + "
                              "segment start; counts", "segments_checked": S,
                   "selected_rank0": sel, "and4_id_offset_rank0": id_offset},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": None,
        "clocks": clk,
        "build_s": {"table": round(t_table, 2), "gen": round(tab.t_gen, 2),
                    "dictionaries": round(tab.t_dict, 2), "layouts": round(tab.t_build, 2),
                    "parity": round(t_parity, 2), "alg_bytes": round(t_alg, 2)},
    }
    # this library's kernels in the rank's step, per segment: one per single
    # scan (4); the AND chain's fused ByteSlice pair + a compacted and an
    # epilogue-masked kernel per PP-VBS leg, one of which exits at its gate (5);
    # the compaction's tile popcount and emit (2; CUB's scan between them is
    # not counted)
    out["gpu_launches"] = int(args.steps * S * (4 + 5 + 2))
    if world == 1 and not args.profile and not args.no_extra:
        del graph, step, tab
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        out["configs"] = measure_configs_after_cfg5(args, world, rank, local)
    return out


def measure_configs_after_cfg5(args, world, rank, local) -> dict:
    """cfg2 (8 BETWEEN scans, the round-1 headline), cfg3 lookups, cfg1, cfg4."""
    import torch
    out = {}
    a2 = argparse.Namespace(**vars(args))
    a2.steps, a2.warmup, a2.workload = 100, 10, "cfg2"
    t0 = time.perf_counter()
    try:
        out["cfg2"] = run_cfg2(a2, world, rank, local, emit_extras=False)
    except Exception as exc:  # noqa: BLE001 - recorded, not swallowed
        out["cfg2"] = {"error": f"{type(exc).__name__}: {exc}"}
    out["cfg2"]["wall_s"] = round(time.perf_counter() - t0, 1)
    torch.cuda.empty_cache()
    if not args.no_lookup:
        t0 = time.perf_counter()
        try:
            out["cfg3"] = measure_lookups(max(3, args.lookup_steps), 28)
        except Exception as exc:  # noqa: BLE001
            out["cfg3"] = {"error": f"{type(exc).__name__}: {exc}"}
        if isinstance(out["cfg3"], dict):
            out["cfg3"]["wall_s"] = round(time.perf_counter() - t0, 1)
    torch.cuda.empty_cache()
    out.update(measure_extra_configs(None))
    return out


def measure_e2e_cfg5(tab, steps, world) -> dict:
    """The 5 cfg5 queries end to end through the public API on the rank's
    first segment of every column with the encoded columns in pinned HOST
    memory: every step uploads the 4 segment columns, runs the scans, the
    conjunction and the row-id compaction, and reads back every result
    bitvector, the counts and the AND's global row ids."""
    import torch
    import torch.distributed as dist

    from paper_2209_00220_b200.byteslice import ByteSliceColumn, scan_byteslice
    from paper_2209_00220_b200.engine import conj_scan
    from paper_2209_00220_b200.vbs import VbsColumn, scan_vbs

    names = ("u0", "u1", "z0", "z1")
    pairs, dcols = [], {}
    for nm in names:
        c = tab.cols[nm][0]
        if tab.layout[nm] == "byteslice":
            h = c.planes.cpu().pin_memory()
            d = torch.empty_like(c.planes)
            pairs.append((h, d))
            dcols[nm] = ByteSliceColumn(c.n_rows, c.width_bits, c.lanes, c.stride, d)
            continue
        K = c.max_len

        def cp(t):
            if t is None:
                return None
            h = t.cpu().pin_memory()
            d = torch.empty_like(t)
            pairs.append((h, d))
            return d
        bs1 = cp(c.bs1)
        deep = [cp(t) for t in c.deep]
        exist = [None] + [cp(c.exist[j]) for j in range(1, K)]
        bdir = [None] + [cp(c.block_dir[j]) for j in range(1, K)]
        rex = None if c.rexist is None else [cp(t) for t in c.rexist]
        dcols[nm] = VbsColumn(c.n_rows, K, c.lanes, c.stride, bs1, deep, exist, bdir,
                              c.level_rows, c.deep_mode, rex, c.deep1_range)
    h2d = sum(h.numel() * h.element_size() for h, _ in pairs)
    n = tab.seg_rows
    nw = n // 32
    res_h = [torch.empty(nw, dtype=torch.int32).pin_memory() for _ in range(5)]
    cnt_h = torch.empty(5, dtype=torch.int64).pin_memory()
    ids_h = [None]
    r0 = tab.seg_starts[0]

    def step():
        for h, d in pairs:
            d.copy_(h, non_blocking=True)
        bvs = []
        for nm in names:
            fn = scan_vbs if tab.layout[nm] == "ppvbs" else scan_byteslice
            bvs.append(fn(dcols[nm], tab.preds[nm])[0])
        andb = conj_scan([(tab.layout[nm], dcols[nm]) for nm in names],
                         [tab.preds[nm] for nm in names])
        bvs.append(andb)
        for i, b in enumerate(bvs):
            res_h[i].copy_(b.dwords, non_blocking=True)
            cnt_h[i:i + 1].copy_(b.count_device(), non_blocking=True)
        ids = andb.row_ids(row_offset=r0)        # syncs for the count (public API)
        ids_h[0] = ids.cpu()
        return ids.numel()

    nsel = step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / steps
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    d2h = 5 * nw * 4 + 5 * 8 + 8 * nsel
    return {"value": round(world * 8 * n / (ms * 1e-3) / 1e9, 3), "unit": "Gcodes/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": round(ms, 3), "steps": steps,
            "what": "public API (scan_byteslice / scan_vbs / engine.conj_scan / row_ids) on "
                    "each rank's first segment (2^29 rows) of the 4 columns: encoded columns "
                    "uploaded from pinned host memory every step, 5 result bitvectors + counts "
                    "+ the AND's global row ids read back every step"}


def run_cfg2(args, world, rank, local, emit_extras=True):
    """The cfg2 step (configs[1]): 8 BETWEEN scans of the 2^28-row Zipf(1.2)
    column on PP-VBS and ByteSlice.  Returns rank 0's JSON dict."""
    import torch
    import torch.distributed as dist

    from paper_2209_00220_b200 import _lib
    from paper_2209_00220_b200.byteslice import scan_byteslice
    from paper_2209_00220_b200.predicate import Op, Predicate
    from paper_2209_00220_b200.roofline import hbm_peak
    from paper_2209_00220_b200.vbs import scan_vbs
    _lib.load()

    n = 1 << args.rows_log2
    data = build_cfg2(n, args.deep_mode)
    col_v, col_b = data["col_v"], data["col_b"]
    table = data["table"]
    wins = window_bounds(table.values, table.weights, n)
    exist_h = [col_v.mask_words(j) for j in range(2, col_v.max_len + 1)]
    scans = []  # (layout, p, column, pred, alg_bytes, stats)
    for p, lo, hi in wins:
        pv = data["d_ppe"].encode_literal(Predicate("c", Op.BETWEEN, lo, hi))
        pb = data["d_fix"].encode_literal(Predicate("c", Op.BETWEEN, lo, hi))
        ab_v, st_v = alg_bytes_for(col_v, "ppvbs", pv, exist_h)
        ab_b, st_b = alg_bytes_for(col_b, "byteslice", pb, None)
        scans.append(("ppvbs", p, col_v, pv, ab_v, st_v))
        scans.append(("byteslice", p, col_b, pb, ab_b, st_b))
    # parity guard (cheap): both layouts must agree on every window
    sel = {}
    for layout, p, col, pred, _, _ in scans:
        fn = scan_vbs if layout == "ppvbs" else scan_byteslice
        bv, _ = fn(col, pred)
        sel.setdefault(p, []).append(bv)
    for p, (a, b) in sel.items():
        assert torch.equal(a.dwords, b.dwords), f"layouts disagree at p={p}"
    counts_ref = {p: a.count() for p, (a, b) in sel.items()}
    del sel

    stream = torch.cuda.current_stream()
    cnt_buf = torch.zeros(len(scans), dtype=torch.int64, device="cuda")
    gather = [torch.zeros_like(cnt_buf) for _ in range(world)] if world > 1 else None

    # the timed step calls the C ABI directly (the drop-in boundary) with
    # preallocated result words and count slots: no per-scan allocation and
    # no extra copy kernels between the scans
    import ctypes

    from paper_2209_00220_b200.device import stream as cur_stream
    lib = _lib.load()
    nwords = -(-n // 32)
    outs = [torch.empty(nwords, dtype=torch.int32, device="cuda") for _ in scans]
    cpreds = [pred.to_c() for (_l, _p, _c, pred, _a, _s) in scans]
    sptr = cur_stream()
    calls = []
    for i, (layout, p, col, pred, _, _) in enumerate(scans):
        fn = lib.bsb_vbs_scan if layout == "ppvbs" else lib.bsb_byteslice_scan
        calls.append((fn, col.desc_ref, ctypes.byref(cpreds[i]), outs[i].data_ptr(),
                      cnt_buf.data_ptr() + 8 * i))

    def step(events=None):
        for i, (fn, desc, cp, optr, cptr) in enumerate(calls):
            if events is not None:
                events[i][0].record(stream)
            rc = fn(desc, cp, None, optr, cptr, None, None, sptr)
            if events is not None:
                events[i][1].record(stream)
            if rc:
                _lib.check(rc, "scan")
        if world > 1:
            dist.all_gather(gather, cnt_buf)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    graph = None
    if not args.no_graph:
        # the 8-scan step as one CUDA graph (launch-bound inner loop): the C ABI
        # calls are captured on a side stream; no allocation happens inside
        # The 8 scans are independent: with --streams S they are captured on S
        # forked streams (scan i on stream i mod S; S = 2 puts the PP-VBS and
        # the ByteSlice scans on their own streams), so one kernel fills the
        # SMs another's last wave leaves idle.
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        sides = [cap] + [torch.cuda.Stream() for _ in range(args.streams - 1)]
        cap.wait_stream(stream)
        with torch.cuda.graph(graph, stream=cap):
            for sd in sides[1:]:
                sd.wait_stream(cap)
            for i, (fn, desc, cp, optr, cptr) in enumerate(calls):
                st_ = sides[i % args.streams]
                _lib.check(fn(desc, cp, None, optr, cptr, None, None, st_.cuda_stream), "scan")
            for sd in sides[1:]:
                cap.wait_stream(sd)
        stream.wait_stream(cap)
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    if not args.profile:
        clocks.start()
        time.sleep(0.3)
    per_launch = [[[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)]
                   for _ in scans] for _ in range(args.steps)]
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    if graph is not None:
        # headline: the captured 8-scan step replayed K times
        ev0.record(stream)
        for k in range(args.steps):
            graph.replay()
            if world > 1:
                dist.all_gather(gather, cnt_buf)
        ev1.record(stream)
        torch.cuda.synchronize()
        total_ms = ev0.elapsed_time(ev1)
        # per-kernel durations for the roofline: the same step launched eagerly
        for k in range(args.steps):
            step(per_launch[k])
        torch.cuda.synchronize()
    else:
        ev0.record(stream)
        for k in range(args.steps):
            step(per_launch[k])
        ev1.record(stream)
        torch.cuda.synchronize()
        total_ms = ev0.elapsed_time(ev1)
    if world > 1:
        dist.barrier()
    clk = clocks.stop() if not args.profile else None
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    got = cnt_buf.cpu().tolist()  # counts of the last step equal the untimed check
    for i, (layout, p, *_r) in enumerate(scans):
        assert got[i] == counts_ref[p], (layout, p, got[i], counts_ref[p])

    # per-kernel durations (stream-ordered CUDA events around each launch)
    dur = {i: [per_launch[k][i][0].elapsed_time(per_launch[k][i][1])
               for k in range(args.steps)] for i in range(len(scans))}
    by_layout = {}
    for i, (layout, p, col, pred, ab, st) in enumerate(scans):
        e = by_layout.setdefault(layout, {"ms": 0.0, "alg_bytes": 0, "windows": {}})
        mean_ms = statistics.mean(dur[i])
        e["ms"] += mean_ms
        e["alg_bytes"] += ab
        e["windows"][str(p)] = {"us": round(mean_ms * 1e3, 2),
                                "gcodes_s": round(n / (mean_ms * 1e-3) / 1e9, 2),
                                "alg_bytes_per_code": round(ab / n, 4),
                                "ref_total_bytes_per_code": round(st.total_bytes / n, 4),
                                "selected": counts_ref[p]}
    peak, peak_src = hbm_peak(ROOT)
    for layout, e in by_layout.items():
        e["gbs"] = e["alg_bytes"] / (e["ms"] * 1e-3) / 1e9
        e["frac"] = e["gbs"] / peak
        e["gcodes_s"] = 4 * n / (e["ms"] * 1e-3) / 1e9
    dom = max(by_layout, key=lambda k: by_layout[k]["ms"])
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(dom)
        except (OSError, ValueError):
            traffic = None
    ms_step = total_ms / args.steps
    value = world * len(scans) * n / (ms_step * 1e-3) / 1e9

    out = None
    if rank == 0:
        e2e = None if args.profile else measure_e2e(data, scans, args.e2e_steps, n, world)
        lookups = None
        if emit_extras and not args.profile and not args.no_lookup:
            torch.cuda.empty_cache()
            lookups = measure_lookups(max(3, args.lookup_steps), args.rows_log2)
        extra = None
        if emit_extras and not args.profile and not args.no_extra:
            extra = measure_extra_configs(data)
        cpu = None
        if world == 1 and not args.profile and not args.no_cpu_baseline:
            cpu = cpu_baseline(n, 1 << 22, os.cpu_count() or 1)
        dom_e = by_layout[dom]
        kname = ("vbs_ds_kernel<BETWEEN> (PP-VBS, SLICED layout scanned in deep-row space)"
                 if dom == "ppvbs" and col_v.deep_mode == _lib.DEEP_SLICED else
                 f"scan_kernel<{dom}, BETWEEN>")
        out = {
            "metric": METRIC, "value": round(value, 3), "unit": "Gcodes/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (seeded numpy PCG64 Zipf draws, reference generator)",
            "config": {"workload": f"cfg2: 2^{args.rows_log2}-row Zipf(1.2)/2^20 column, "
                                   f"BETWEEN windows p=0.1/1/10/50% on PP-VBS "
                                   f"(K={col_v.max_len}) and ByteSlice (w={col_b.width_bits})",
                       "rows_per_gpu": n, "scans_per_step": len(scans),
                       "l2": f"inputs larger than L2 (PP-VBS {col_bytes(col_v) / 1e6:.0f} MB, "
                             f"ByteSlice {col_bytes(col_b) / 1e6:.0f} MB per column)",
                       "parallelism": f"row shards x{world}" if world > 1 else "single GPU",
                       "launch": (f"CUDA graph of the 8 scans (C ABI calls captured; "
                                  f"{args.streams} stream{'s' if args.streams > 1 else ''}: "
                                  f"{'scan i on stream i mod ' + str(args.streams) if args.streams > 1 else 'serial'})")
                                 if graph is not None else "eager C ABI calls"},
            "roofline": {"bound": "hbm", "kernel": kname,
                         "achieved": round(dom_e["gbs"], 1), "peak": peak, "unit": "GB/s",
                         "frac": round(dom_e["frac"], 4), "peak_source": peak_src,
                         "traffic": traffic,
                         "traffic_source": "profiles/ncu_traffic.json (dram read+write per "
                                           "launch, mean of the 4 windows)",
                         # physical DRAM bytes per launch over the same launch time: below
                         # the algorithmic fraction when the kernel skips bytes the
                         # reference reads (PP-VBS: level-1 slice of rows that cannot match)
                         "dram_gbs": (round(traffic / (dom_e["ms"] / 4 * 1e-3) / 1e9, 1)
                                      if traffic else None),
                         "dram_frac": (round(traffic / (dom_e["ms"] / 4 * 1e-3) / 1e9 / peak, 4)
                                       if traffic else None),
                         "alg_bytes_per_launch": int(dom_e["alg_bytes"] / 4),
                         "alg_bytes_per_step": int(dom_e["alg_bytes"])},
            "layouts": {k: {"gcodes_s": round(v["gcodes_s"], 2), "hbm_gbs": round(v["gbs"], 1),
                            "frac": round(v["frac"], 4), "windows": v["windows"]}
                        for k, v in by_layout.items()},
            "lookup": lookups,
            "configs": extra,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": len(scans) * args.steps,
            "clocks": clk,
            "build_s": {"gen_zipf": round(data["t_gen"], 3),
                        "encode_and_layouts": round(data["t_encode"], 3)},
        }
    return out


def measure_extra_configs(data) -> dict:
    """SURVEY.md §8(d) cfg1 / cfg4 (bench_cfgs.py); a failure is reported in
    the line instead of hiding the headline.  (cfg5 is bench.py's own
    workload, bench_cfg5.py.)"""
    import torch

    import bench_cfgs
    out = {}
    for name, fn in (("cfg1", bench_cfgs.measure_cfg1), ("cfg4", bench_cfgs.measure_cfg4)):
        torch.cuda.empty_cache()
        t0 = time.perf_counter()
        try:
            out[name] = fn()
        except Exception as exc:  # noqa: BLE001 - recorded, not swallowed
            out[name] = {"error": f"{type(exc).__name__}: {exc}"}
        out[name]["wall_s"] = round(time.perf_counter() - t0, 1)
    return out


def measure_lookups(steps: int, log2n: int = 28, only: str | None = None):
    """cfg3 (BASELINE.json configs[2]): 2^28-row ByteSlice column of 24-bit
    uniform codes (identity codes = values) and a 2^28-row Zipf(1.0)/2^20
    PP-VBS column; lookups of 2^24 random row ids (unsorted and sorted) and of
    the rows selected by 1% / 20% random bitvectors, reconstructing int32
    values (PP-VBS: fused decode through the dictionary).  Seeds follow
    SURVEY.md §8(d)."""
    import torch

    from paper_2209_00220_b200 import ColumnKind, Dictionary, FrequencyTable, ZipfSpec
    from paper_2209_00220_b200.bitvector import DeviceBitVector
    from paper_2209_00220_b200.byteslice import build_byteslice, lookup_byteslice_rows
    from paper_2209_00220_b200.datagen import gen_zipf_device
    from paper_2209_00220_b200.device import to_dev_u32
    from paper_2209_00220_b200.dictionary import freq_table_and_ranks
    from paper_2209_00220_b200.roofline import hbm_peak, lookup_alg_bytes_rows
    from paper_2209_00220_b200.vbs import build_vbs, lookup_vbs_rows_dec

    n = 1 << log2n
    m = 1 << (log2n - 4)
    rng3 = np.random.default_rng(3)
    codes = torch.from_numpy(rng3.integers(0, 1 << 24, n, dtype=np.int64)).cuda()
    col_b = build_byteslice(codes, 24)
    raw_b = codes.to(torch.int32)  # parity check of every lookup against the raw values
    del codes
    vals = gen_zipf_device(ZipfSpec(1.0, 20, n, seed=4))
    raw_v = vals.to(torch.int32)
    u, c, ranks = freq_table_and_ranks(vals)
    d = Dictionary.build(FrequencyTable(u.cpu().numpy(), c.cpu().numpy(), ColumnKind.NUMERIC),
                         "prefix_preserving")
    cv, lv = d.row_codes_device(ranks)
    col_v = build_vbs(cv, lv)
    del cv, lv, ranks
    ids = np.random.default_rng(5).integers(0, n, m)
    sets = {"ids_unsorted": ids, "ids_sorted": np.sort(ids)}
    bvs = {}
    rng6 = np.random.default_rng(6)
    for p in (0.01, 0.20):
        flags = rng6.random(n) < p
        words = np.packbits(flags, bitorder="little").view(np.uint32)
        bvs[f"bits_{int(p * 100)}pct"] = (words, np.flatnonzero(flags))
        del flags
    peak, _ = hbm_peak(ROOT)
    exist_v = [col_v.mask_words(j) for j in range(2, col_v.max_len + 1)]
    out = {}
    gathered = {}

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / steps

    import ctypes

    from paper_2209_00220_b200 import _lib
    from paper_2209_00220_b200.device import stream
    lib = _lib.load()
    dec_v = d.dev_decoder
    cnt = torch.empty(1, dtype=torch.int64, device="cuda")

    for name, rows in list(sets.items()) + [(k, v[1]) for k, v in bvs.items()]:
        is_bits = name.startswith("bits")
        if is_bits:
            dbits = DeviceBitVector(n, to_dev_u32(bvs[name][0]))
            nsel = len(rows)
            o64 = torch.empty(max(nsel, 1), dtype=torch.int64, device="cuda")
            o32 = torch.empty(max(nsel, 1), dtype=torch.int32, device="cuda")
        else:
            drows = torch.from_numpy(rows).cuda()
        for layout in ("byteslice", "ppvbs"):
            if only and only not in f"{layout}/{name}":
                continue
            if is_bits and layout == "byteslice":
                # fused bitvector -> codes (identity codes: code = value)
                fn = lambda: lib.bsb_byteslice_lookup_bits(
                    col_b.desc_ref, dbits.dwords.data_ptr(), None, o64.data_ptr(), None,
                    None, cnt.data_ptr(), stream())
            elif is_bits:
                # fused bitvector -> PP-VBS codes -> PPE tree decode -> int32 values
                fn = lambda: lib.bsb_vbs_lookup_bits(
                    col_v.desc_ref, dbits.dwords.data_ptr(), ctypes.byref(dec_v), None, None,
                    o32.data_ptr(), cnt.data_ptr(), stream())
            elif layout == "byteslice":
                # public API, int32 values out (identity codes: code = value);
                # long unsorted id lists are gathered in row order
                fn = lambda: lookup_byteslice_rows(col_b, drows, out_dtype=torch.int32)
            else:
                fn = lambda: lookup_vbs_rows_dec(col_v, drows, dec_v, out_dtype=torch.int32)
            ms = timed(fn)
            raw = raw_b if layout == "byteslice" else raw_v
            if not is_bits:
                gathered[(layout, name)] = got = fn()
                if not torch.equal(got.to(torch.int32), raw[drows]):
                    raise RuntimeError(f"{layout}/{name}: looked-up values != raw values")
            else:
                fn()
                got = (o64 if layout == "byteslice" else o32)[:nsel].to(torch.int32)
                if not torch.equal(got, raw[torch.from_numpy(rows).cuda()]):
                    raise RuntimeError(f"{layout}/{name}: fused lookup values != raw values")
            if is_bits and int(cnt.item()) != nsel:
                raise RuntimeError(f"{layout}/{name}: fused lookup count mismatch")
            K = col_b.n_slices if layout == "byteslice" else col_v.max_len
            ob = 8 if (is_bits and layout == "byteslice") else 4
            ab = lookup_alg_bytes_rows(
                rows, K, layout, None if layout == "byteslice" else exist_v,
                out_bytes=ob, id_bytes=0 if is_bits else 8,
                table_bytes=0 if layout == "byteslice" else d.dev_decoder_bytes)
            if is_bits:
                ab += 4 * (-(-n // 32))
            out[f"{layout}/{name}"] = {
                "rows": int(len(rows)), "ms": round(ms, 4),
                "mrows_s": round(len(rows) / (ms * 1e-3) / 1e6, 1),
                "alg_gbs": round(ab / (ms * 1e-3) / 1e9, 1),
                "frac": round(ab / (ms * 1e-3) / 1e9 / peak, 4)}
    # the unsorted-id gathers (sorted internally, scattered back) must equal
    # the sorted-id gathers in input order
    back = torch.from_numpy(np.argsort(ids, kind="stable")).cuda()
    for layout in ("byteslice", "ppvbs"):
        if (layout, "ids_unsorted") in gathered and (layout, "ids_sorted") in gathered:
            if not torch.equal(gathered[(layout, "ids_unsorted")][back],
                               gathered[(layout, "ids_sorted")]):
                raise RuntimeError(f"{layout}: unsorted and sorted id lookups disagree")
    return out


def col_bytes(col) -> int:
    if hasattr(col, "planes"):
        return col.planes.numel()
    b = col.bs1.numel()
    if col.deep[0] is not None:
        b += col.deep[0].numel()
    for j in range(1, col.max_len):
        if col.deep[j] is not None:
            b += col.deep[j].numel() * col.deep[j].element_size()
        b += col.exist[j].numel() * 4
        if col.block_dir[j] is not None:
            b += col.block_dir[j].numel() * 8
        if col.rexist is not None and col.rexist[j] is not None:
            b += col.rexist[j].numel() * 4
    return b


def measure_e2e(data, scans, steps, n, world):
    """Same 8 scans through the public API with the encoded columns in pinned
    HOST memory: every step uploads the column arrays, scans, and reads the
    result bitvectors + counts back.  Three streams pipeline consecutive
    steps (upload of step k+1 overlaps the read-back of step k; PCIe is full
    duplex) over two device copies of the columns and two result sets."""
    import torch

    from paper_2209_00220_b200.byteslice import ByteSliceColumn, scan_byteslice
    from paper_2209_00220_b200.vbs import VbsColumn, scan_vbs
    col_v, col_b = data["col_v"], data["col_b"]
    K = col_v.max_len
    host_v = [col_v.bs1.cpu().pin_memory()]
    for j in range(1, K):
        for t in (col_v.deep[j], col_v.exist[j], col_v.block_dir[j]):
            host_v.append(None if t is None else t.cpu().pin_memory())
    host_r = [None] + [None if (col_v.rexist is None or col_v.rexist[j] is None)
                       else col_v.rexist[j].cpu().pin_memory() for j in range(1, K)]
    host_b = col_b.planes.cpu().pin_memory()
    host_d0 = None if col_v.deep[0] is None else col_v.deep[0].cpu().pin_memory()

    def device_copy():
        dv = [None if h is None else torch.empty(h.shape, dtype=h.dtype, device="cuda")
              for h in host_v]
        dr = [None if h is None else torch.empty(h.shape, dtype=h.dtype, device="cuda")
              for h in host_r]
        db = torch.empty_like(col_b.planes)
        d0 = None if host_d0 is None else torch.empty_like(host_d0, device="cuda")
        cv = VbsColumn(col_v.n_rows, K, col_v.lanes, col_v.stride, dv[0],
                       [d0] + [dv[1 + 3 * (j - 1)] for j in range(1, K)],
                       [None] + [dv[2 + 3 * (j - 1)] for j in range(1, K)],
                       [None] + [dv[3 + 3 * (j - 1)] for j in range(1, K)], col_v.level_rows,
                       col_v.deep_mode, dr)
        cb = ByteSliceColumn(col_b.n_rows, col_b.width_bits, col_b.lanes, col_b.stride, db)
        pairs = [(h, d) for h, d in zip(host_v + host_r + [host_b, host_d0],
                                        dv + dr + [db, d0])
                 if h is not None]
        return cv, cb, pairs

    bufs = [device_copy(), device_copy()]
    nw = -(-n // 32)
    out_h = [torch.empty(nw, dtype=torch.int32).pin_memory() for _ in scans]
    cnt_h = torch.empty(len(scans), dtype=torch.int64).pin_memory()
    h2d = sum(h.numel() * h.element_size() for h, _ in bufs[0][2])
    d2h = len(scans) * (nw * 4 + 8)
    s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()
    s_cmp = torch.cuda.current_stream()
    res = [[torch.empty(nw, dtype=torch.int32, device="cuda") for _ in scans] for _ in range(2)]
    cnt_d = [torch.empty(len(scans), dtype=torch.int64, device="cuda") for _ in range(2)]
    ev_scan = [torch.cuda.Event(), torch.cuda.Event()]
    ev_down = [torch.cuda.Event(), torch.cuda.Event()]
    ev_up = [torch.cuda.Event(), torch.cuda.Event()]
    k_step = [0]

    def step():
        k = k_step[0] % 2
        k_step[0] += 1
        cv, cb, pairs = bufs[k]
        with torch.cuda.stream(s_up):
            s_up.wait_event(ev_scan[k])  # scans two steps back read this copy
            for h, d in pairs:
                d.copy_(h, non_blocking=True)
            ev_up[k].record(s_up)
        s_cmp.wait_event(ev_up[k])
        s_cmp.wait_event(ev_down[k])  # result buffers of two steps back read out
        for i, (layout, p, _c, pred, _a, _s) in enumerate(scans):
            bv, _ = (scan_vbs(cv, pred) if layout == "ppvbs" else scan_byteslice(cb, pred))
            res[k][i].copy_(bv.dwords)
            cnt_d[k][i:i + 1].copy_(bv._count)
        ev_scan[k].record(s_cmp)
        with torch.cuda.stream(s_dn):
            s_dn.wait_event(ev_scan[k])
            for i in range(len(scans)):
                out_h[i].copy_(res[k][i], non_blocking=True)
            cnt_h.copy_(cnt_d[k], non_blocking=True)
            ev_down[k].record(s_dn)

    step()
    step()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(s_up)
    for _ in range(steps):
        step()
    s_up.wait_stream(s_dn)
    s_up.wait_stream(s_cmp)
    ev1.record(s_up)
    ev1.synchronize()
    ms = ev0.elapsed_time(ev1) / steps
    # resident variant: columns stay in HBM, only results come back
    def step_res():
        for i, (layout, p, col, pred, _a, _s) in enumerate(scans):
            fn = scan_vbs if layout == "ppvbs" else scan_byteslice
            bv, _ = fn(col, pred)
            out_h[i].copy_(bv.dwords, non_blocking=True)
            cnt_h[i:i + 1].copy_(bv._count, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    step_res()
    ev0.record()
    for _ in range(steps):
        step_res()
    ev1.record()
    ev1.synchronize()
    ms_res = ev0.elapsed_time(ev1) / steps
    return {"value": round(world * len(scans) * n / (ms * 1e-3) / 1e9, 3), "unit": "Gcodes/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": round(ms, 3), "steps": steps,
            "what": "public scan API; encoded columns uploaded from pinned host memory every "
                    "step; result bitvectors + counts read back every step; consecutive "
                    "steps pipelined over upload / scan / read-back streams",
            "resident": {"value": round(world * len(scans) * n / (ms_res * 1e-3) / 1e9, 3),
                         "ms_per_step": round(ms_res, 3), "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": int(d2h)}}


def main():
    args = parse()
    if args.steps is None:
        args.steps = 30 if args.workload == "cfg5" else 400
    if args.warmup is None:
        args.warmup = 5 if args.workload == "cfg5" else 20
    if args.impl == "reference":
        (run_reference_cfg5 if args.workload == "cfg5" else run_reference)(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
