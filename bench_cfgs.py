"""Secondary measurements for bench.py: SURVEY.md §8(d) cfg1 and cfg4.
Each returns a JSON-able dict that bench.py attaches to its line under
"configs"; every timed number is device time from CUDA events
on the launching stream, after warm-up, and every workload is checked against
a host numpy filter of the same raw values before it is timed.

  cfg1  ByteSlice LT scan + fused bitvector lookup, 2^24 rows, w=16
        (32 MiB column: 16 distinct replicas rotated so L2 never holds one)
  cfg4  16 columns x 2^27 rows through the advisor (GPU wall-clock AUC), then
        the 4-predicate conjunction as ONE fused device pass + 3 projections
        decoded on the device + SUM(u32)
(cfg5, the 2^32-row sharded table, is bench.py's headline: bench_cfg5.py.)
"""

from __future__ import annotations

import time

import numpy as np


def _events():
    import torch
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def _time(fn, reps: int, warmup: int = 3) -> float:
    """Mean device ms of fn over reps (events bracket the batch)."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a, b = _events()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def _q(uniq: np.ndarray, counts: np.ndarray, n: int, x: float) -> int:
    """Nearest-rank quantile sorted(values)[min(n-1, floor(x*n))] from a
    frequency table (reference advisor.py:56-59)."""
    cum = np.cumsum(counts)
    return int(uniq[np.searchsorted(cum, min(n - 1, int(x * n)), side="right")])


def _alg_bytes(cols, preds):
    """Pipelined algorithmic bytes of a conjunction: each
    predicate's own slice/mask terms over the blocks still live, in the order
    engine.conj_scan evaluates them (engine.conj_order)."""
    from paper_2209_00220_b200.byteslice import scan_byteslice
    from paper_2209_00220_b200.engine import conj_order
    from paper_2209_00220_b200.roofline import scan_alg_bytes
    from paper_2209_00220_b200.vbs import scan_vbs
    order = conj_order([c[0] for c in cols])
    cols = [cols[i] for i in order]
    preds = [preds[i] for i in order]
    total, running = 0, None
    for (lay, c, ex), p in zip(cols, preds):
        fn = scan_vbs if lay == "ppvbs" else scan_byteslice
        bv, st = fn(c, p, running)
        st = st.materialize()
        total += scan_alg_bytes(st.block_depth, lay, c.max_len if lay == "ppvbs" else c.n_slices,
                                ex, masked=running is not None)
        running = bv
    return total


# --------------------------------------------------------------------- cfg1
def measure_cfg1(reps: int = 50) -> dict:
    import torch

    from paper_2209_00220_b200 import _lib
    from paper_2209_00220_b200.byteslice import build_byteslice, scan_byteslice
    from paper_2209_00220_b200.device import stream
    from paper_2209_00220_b200.predicate import Op, ResolvedPredicate
    from paper_2209_00220_b200.roofline import hbm_peak, scan_alg_bytes

    n, w = 1 << 24, 16
    codes = np.random.default_rng(1).integers(0, 65536, n)
    want = codes < 6554
    replicas = [build_byteslice(codes, w) for _ in range(16)]
    pred = ResolvedPredicate.compare(Op.LT, 6554, 2)
    bv, st = scan_byteslice(replicas[0], pred)
    assert bv.count() == int(want.sum()), "cfg1 scan count"
    ab = scan_alg_bytes(st.materialize().block_depth, "byteslice", 2)
    nsel = int(want.sum())
    lib = _lib.load()
    out = torch.empty(nsel, dtype=torch.int64, device="cuda")
    cnt = torch.empty(1, dtype=torch.int64, device="cuda")
    # lookup parity: fused bitvector -> codes (identity dictionary: code = value)
    _lib.check(lib.bsb_byteslice_lookup_bits(replicas[0].desc_ref, bv.dwords.data_ptr(), None,
                                             out.data_ptr(), None, None, cnt.data_ptr(),
                                             stream()), "cfg1 lookup")
    assert np.array_equal(out.cpu().numpy(), codes[want]), "cfg1 lookup values"
    outs = [torch.empty(n // 32, dtype=torch.int32, device="cuda") for _ in replicas]
    cnts = [torch.empty(1, dtype=torch.int64, device="cuda") for _ in replicas]
    cp = pred.to_c()
    it = [0]

    def scan():
        i = it[0] % 16
        it[0] += 1
        lib.bsb_byteslice_scan(replicas[i].desc_ref, ctypes_ref(cp), None,
                               outs[i].data_ptr(), cnts[i].data_ptr(), None, None, stream())

    ms_eager = _time(scan, reps)
    # 2^24 rows are ~17 MB: a scan is a few microseconds of GPU work, below the
    # cost of one Python-side launch.  The headline number replays the 16
    # rotated scans as one CUDA graph of C ABI calls (as bench.py's step).
    # The reference's scan_byteslice returns the result words (its count is a
    # separate ResultBitVector method), so the headline calls pass count =
    # NULL; the same graph with the count (one memset node + atomics per
    # scan) is reported beside it.
    def graph_ms(with_count: bool) -> float:
        for o in outs:
            o.fill_(-1)
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(graph, stream=cap):
            for i in range(16):
                _lib.check(lib.bsb_byteslice_scan(
                    replicas[i].desc_ref, ctypes_ref(cp), None, outs[i].data_ptr(),
                    cnts[i].data_ptr() if with_count else None, None, None, cap.cuda_stream),
                    "cfg1 scan")
        torch.cuda.current_stream().wait_stream(cap)
        ms = _time(graph.replay, max(3, reps // 16)) / 16
        want_w = bv.dwords
        for i in range(16):
            assert torch.equal(outs[i], want_w), "cfg1 graph scan words"
            if with_count:
                assert int(cnts[i].item()) == nsel, "cfg1 graph scan count"
        return ms

    ms_scan = graph_ms(False)
    ms_scan_cnt = graph_ms(True)
    bvs = []
    for i in range(16):
        b, _ = scan_byteslice(replicas[i], pred)
        bvs.append(b)

    def look():
        i = it[0] % 16
        it[0] += 1
        lib.bsb_byteslice_lookup_bits(replicas[i].desc_ref, bvs[i].dwords.data_ptr(), None,
                                      out.data_ptr(), None, None, cnt.data_ptr(), stream())

    ms_look = _time(look, reps)
    peak, _ = hbm_peak()
    return {
        "workload": "cfg1: 2^24 uniform 16-bit codes, ByteSlice w=16, LT 6554, then fused "
                    "bitvector lookup of the 1,676,081-ish matches (16 rotated replicas)",
        "rows": n, "selected": nsel,
        "scan": {"us": round(ms_scan * 1e3, 2), "gcodes_s": round(n / ms_scan / 1e6, 1),
                 "alg_bytes_per_code": round(ab / n, 4),
                 "frac": round(ab / (ms_scan * 1e-3) / 1e9 / peak, 4),
                 "timing": "CUDA graph of the 16 rotated C ABI scans (result words, count = "
                           "NULL as the reference's scan), per scan",
                 "with_count_us": round(ms_scan_cnt * 1e3, 2),
                 "eager_us": round(ms_eager * 1e3, 2)},
        "lookup": {"us": round(ms_look * 1e3, 2),
                   "mrows_s": round(nsel / ms_look / 1e3, 1)},
    }


def ctypes_ref(x):
    import ctypes
    return ctypes.byref(x)


# --------------------------------------------------------------------- cfg4
CFG4_UNIFORM = {"u08": 8, "u12": 12, "u16": 16, "u20": 20, "u24": 24, "u32": 32, "u16b": 16,
                "u24b": 24}
CFG4_ZIPF = {"z08": (0.8, 8), "z12": (1.0, 12), "z16": (1.5, 16), "z20": (0.8, 20),
             "z24": (1.0, 24), "z24b": (1.5, 24), "z16b": (1.0, 16), "z12b": (0.8, 12)}


def measure_cfg4(reps: int = 20, log2n: int = 27, advise_count: int = 100) -> dict:
    import torch

    from paper_2209_00220_b200 import ColumnKind, ZipfSpec
    from paper_2209_00220_b200.datagen import gen_zipf_device
    from paper_2209_00220_b200.engine import conj_scan, ingest_arrays, lookup_decode_bits
    from paper_2209_00220_b200.predicate import Op, Predicate
    from paper_2209_00220_b200.roofline import hbm_peak

    n = 1 << log2n
    names = list(CFG4_UNIFORM) + list(CFG4_ZIPF)
    cols = {}
    t0 = time.perf_counter()
    for i, nm in enumerate(names):
        seed = 100 + i
        if nm in CFG4_UNIFORM:
            w = CFG4_UNIFORM[nm]
            rng = np.random.default_rng(seed)
            v = (rng.integers(-(1 << 31), 1 << 31, n) if w == 32 else rng.integers(0, 1 << w, n))
            cols[nm] = torch.from_numpy(v).cuda()
        else:
            s, d = CFG4_ZIPF[nm]
            cols[nm] = gen_zipf_device(ZipfSpec(s, d, n, seed))
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    store, report = ingest_arrays(cols, advise_cost="wall", advise_count=advise_count)
    torch.cuda.synchronize()
    t_ingest = time.perf_counter() - t0
    advice = {e["name"]: {"layout": e["layout"], **({k: round(v, 9) for k, v in
                                                      e["advice"].items() if k != "chosen"}
                                                     if "advice" in e else {})}
              for e in store.manifest["columns"]}

    def q(nm, x):
        t = store.columns[nm].dictionary.table
        return _q(t.values, t.weights, n, x)

    preds = [Predicate("u16", Op.LT, 32768),
             Predicate("z12", Op.BETWEEN, q("z12", 0.2), q("z12", 0.9)),
             Predicate("u24", Op.GE, q("u24", 0.6)),
             Predicate("z16", Op.LE, q("z16", 0.7))]
    proj = ["u32", "z24", "u20"]
    # host check of the conjunction and SUM(u32)
    h = {nm: cols[nm].cpu().numpy() for nm in ("u16", "z12", "u24", "z16", "u32")}
    m = ((h["u16"] < 32768) & (h["z12"] >= preds[1].value) & (h["z12"] <= preds[1].value_high)
         & (h["u24"] >= preds[2].value) & (h["z16"] <= preds[3].value))
    want_count, want_sum = int(m.sum()), int(h["u32"][m].astype(np.int64).sum())
    m_host = m
    del h
    stored = [store.columns[p.column] for p in preds]
    rps = [s.dictionary.encode_literal(p) for s, p in zip(stored, preds)]
    pairs = [(s.layout, s.column) for s in stored]
    sel = conj_scan(pairs, rps)
    assert sel.count() == want_count, "cfg4 conjunction count"
    # word-for-word against the raw-value filter (tests/helpers.py:35-52)
    from bench_cfg5 import pack_bools
    dflags = torch.from_numpy(m_host).cuda()
    assert torch.equal(sel.dwords, pack_bools(dflags)), "cfg4 conjunction words"
    for nm in ("u32", "z24", "u20"):
        got = lookup_decode_bits(store.columns[nm], sel)
        assert torch.equal(got, cols[nm][dflags]), f"cfg4 projection {nm}"
    del dflags
    got_sum = int(lookup_decode_bits(store.columns["u32"], sel).sum().item())
    assert got_sum == want_sum, "cfg4 SUM(u32)"
    ms_scan = _time(lambda: conj_scan(pairs, rps), reps)
    ms_look = {}
    for nm in proj:
        ms_look[nm] = _time(lambda nm=nm: lookup_decode_bits(store.columns[nm], sel), reps)
    ex = []
    for s in stored:
        ex.append([s.column.mask_words(j) for j in range(2, s.column.max_len + 1)]
                  if s.layout == "ppvbs" else None)
    ab = _alg_bytes([(s.layout, s.column, e) for s, e in zip(stored, ex)], rps)
    peak, _ = hbm_peak()
    # advisor timing on the device: bytes mode per column, and wall mode twice
    # on the columns whose AUCs are closest (the decision must not flip)
    from paper_2209_00220_b200.advisor import advise_column
    adv = {}
    for nm in ("z16", "u16"):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a = advise_column(nm, cols[nm], ColumnKind.NUMERIC, count=advise_count, cost="bytes")
        torch.cuda.synchronize()
        adv[f"{nm}/bytes"] = {"s": round(time.perf_counter() - t0, 3), "chosen": a.chosen}
    close = sorted((abs(e["advice"]["auc_byteslice"] - e["advice"]["auc_ppvbs"]) /
                    max(e["advice"]["auc_byteslice"], e["advice"]["auc_ppvbs"]), e["name"])
                   for e in store.manifest["columns"] if "advice" in e)[:2]
    for _, nm in close:
        picks = []
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            a = advise_column(nm, cols[nm], ColumnKind.NUMERIC, count=advise_count, cost="wall")
            picks.append(a.chosen)
        adv[f"{nm}/wall"] = {"s": round(time.perf_counter() - t0, 3), "chosen": picks,
                             "ingest_choice": advice[nm]["layout"],
                             "stable": len(set(picks + [advice[nm]["layout"]])) == 1}
    return {
        "advisor_device": adv,
        "workload": "cfg4: 16 columns x 2^27 (8 uniform, 8 Zipf; seeds 100+i), advisor in GPU "
                    "wall mode, query u16<32768 AND z12 BETWEEN q(.2),q(.9) AND u24>=q(.6) AND "
                    "z16<=q(.7) -> u32, z24, u20 + SUM(u32)",
        "rows": n, "selected": want_count, "sum_u32": want_sum,
        "advisor": advice, "gen_s": round(t_gen, 2), "ingest_s": round(t_ingest, 2),
        "conj_scan": {"us": round(ms_scan * 1e3, 2),
                      "gcodes_s": round(4 * n / ms_scan / 1e6, 1),
                      "alg_bytes": int(ab),
                      "frac": round(ab / (ms_scan * 1e-3) / 1e9 / peak, 4),
                      "layouts": [s.layout for s in stored]},
        "lookups": {nm: {"us": round(t * 1e3, 2), "mrows_s": round(want_count / t / 1e3, 1),
                         "layout": store.columns[nm].layout} for nm, t in ms_look.items()},
    }
