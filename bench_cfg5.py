"""cfg5 (BASELINE.json configs[4]): the row-range sharded scan that bench.py
measures as its headline at every N.

Table: 4 columns x 2^32 rows, generated as 8 fixed 2^29-row chunks per
column (seed 500 + 10*col + chunk), so the data is the same
at 1/2/4/8 GPUs:
  u0, u1  int32 uniform over the full range, stored as bias-identity codes
          value + 2^31 (uint32, order preserving) in ByteSlice w=32;
  z0, z1  Zipf(1.1) over 2^24 (the reference generator per chunk), each with
          its own global PPE dictionary (ppe_numerical over the all-reduced
          per-value counts of all 2^32 rows), stored as PP-VBS.
Each chunk is one stored row-range segment; rank r owns segments
sharded.owned_segments(8, N, r) (strong scaling: the total is fixed).

Queries: u0 < q(.10), u1 >= q(.50), z0 BETWEEN q(.80) AND
q(.95), z1 <= q(.60), each alone and as the 4-way AND; the AND's matches are
compacted into global int64 row ids.  q = exact nearest-rank quantiles over
all 2^32 rows (radix select over all ranks for u0/u1, cumulative global
counts for z0/z1).

One step = the 5 queries over the rank's segments (scans, per-query counts,
the AND's row-id compaction) replayed as one CUDA graph, then ONE NCCL
all_gather of the per-rank counts (global counts + each rank's id offset).
Codes scanned per step: 8 x 2^32 (4 single predicates + 4 in the AND).

Before timing, every segment's bitvector of every query is compared word
for word with a device filter of that segment's raw values (the reference's
naive_filter, tests/helpers.py:35-52), and the compacted ids with the raw
filter's row numbers + segment start.
"""

from __future__ import annotations

import ctypes
import os
import statistics
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

N_CHUNKS = 8
ZIPF_S, ZIPF_BITS = 1.1, 24
COLS = (("u0", "uniform"), ("u1", "uniform"), ("z0", "zipf"), ("z1", "zipf"))
QUERIES = ("u0", "u1", "z0", "z1", "and4")


def chunk_seed(ci: int, chunk: int) -> int:
    return 500 + 10 * ci + chunk


def gen_host(ci: int, kind: str, chunk: int, rows: int) -> np.ndarray:
    """Host PCG64 draws of one chunk: int32 values (uniform) or the float64
    uniforms that gen_zipf maps through the CDF (datagen.py:50-56)."""
    rng = np.random.default_rng(chunk_seed(ci, chunk))
    if kind == "uniform":
        return rng.integers(-(1 << 31), 1 << 31, rows, dtype=np.int32)
    return rng.random(rows)


def pack_bools(flags):
    """torch bool[n] -> int32 words, LSB-first (bitvector.py:3-5)."""
    import torch
    n = flags.numel()
    nw = -(-n // 32)
    f = torch.zeros(nw * 32, dtype=torch.int64, device=flags.device)
    f[:n] = flags.to(torch.int64)
    sh = torch.arange(32, device=flags.device, dtype=torch.int64)
    return (f.view(nw, 32) << sh).sum(1).to(torch.int32)


def _q_from_counts(counts: np.ndarray, n: int, x: float) -> int:
    cum = np.cumsum(counts)
    return int(np.searchsorted(cum, min(n - 1, int(x * n)), side="right"))


class Cfg5Table:
    """This rank's segments of the cfg5 table, built on the device."""

    def __init__(self, world: int, rank: int, seg_rows: int = 1 << 29, group=None,
                 keep_raw: bool = True, log=print, only_segments=None):
        import torch
        import torch.distributed as dist

        from paper_2209_00220_b200 import ColumnKind, Dictionary, FrequencyTable, _lib
        from paper_2209_00220_b200.byteslice import build_byteslice
        from paper_2209_00220_b200.datagen import _cdf, ZipfSpec
        from paper_2209_00220_b200.device import stream
        from paper_2209_00220_b200.predicate import Op, Predicate, ResolvedPredicate
        from paper_2209_00220_b200.sharded import global_nearest_rank_u32, owned_segments
        from paper_2209_00220_b200.vbs import build_vbs

        self.world, self.rank = world, rank
        self.seg_rows = seg_rows
        self.n_total = N_CHUNKS * seg_rows
        self.segs = list(owned_segments(N_CHUNKS, world, rank))
        if only_segments is not None:  # diagnostics: a subset (dictionaries from it alone)
            self.segs = [s for s in self.segs if s in only_segments]
            self.n_total = len(self.segs) * seg_rows
        self.seg_starts = [s * seg_rows for s in self.segs]
        dev = torch.device("cuda", torch.cuda.current_device())
        dist_on = world > 1
        t0 = time.perf_counter()
        lib = _lib.load()
        cdf = torch.from_numpy(_cdf(ZipfSpec(ZIPF_S, ZIPF_BITS, 1, 0))).to(dev)
        # ---- raw values (device int32), host PCG64 on a thread pool
        raw = {nm: [None] * len(self.segs) for nm, _ in COLS}
        tasks = [(ci, nm, kind, si, s) for ci, (nm, kind) in enumerate(COLS)
                 for si, s in enumerate(self.segs)]
        threads = max(1, min(8, (os.cpu_count() or 2) // max(1, min(world, 8)) or 1))
        with ThreadPoolExecutor(threads) as pool:
            futs = {pool.submit(gen_host, ci, kind, s, seg_rows): (nm, kind, si)
                    for ci, nm, kind, si, s in tasks}
            for f in futs:
                nm, kind, si = futs[f]
                h = f.result()
                if kind == "uniform":
                    raw[nm][si] = torch.from_numpy(h).to(dev)
                else:
                    out = torch.empty(seg_rows, dtype=torch.int64, device=dev)
                    for p0 in range(0, seg_rows, 1 << 26):
                        u = torch.from_numpy(h[p0:p0 + (1 << 26)]).to(dev)
                        _lib.check(lib.bsb_zipf_from_uniform(
                            u.data_ptr(), u.numel(), cdf.data_ptr(), 1 << ZIPF_BITS,
                            out[p0:].data_ptr(), stream()), "gen_zipf")
                    raw[nm][si] = out.to(torch.int32)
                    del out
                del h
        torch.cuda.synchronize()
        self.t_gen = time.perf_counter() - t0
        t0 = time.perf_counter()
        # ---- global statistics: quantiles of u0/u1, per-value counts of z0/z1
        biased = lambda t: t.to(torch.int64) + (1 << 31)  # noqa: E731
        qu0 = global_nearest_rank_u32([biased(t) for t in raw["u0"]], [0.10], self.n_total,
                                      group)[0]
        qu1 = global_nearest_rank_u32([biased(t) for t in raw["u1"]], [0.50], self.n_total,
                                      group)[0]
        self.dicts, self.rank_lut = {}, {}
        for nm in ("z0", "z1"):
            w = torch.zeros(1 << ZIPF_BITS, dtype=torch.int64, device=dev)
            for t in raw[nm]:
                for p in torch.split(t, 1 << 27):
                    w += torch.bincount(p.to(torch.int64), minlength=1 << ZIPF_BITS)
            if dist_on:
                dist.all_reduce(w, group=group)
            present = w > 0
            uniq = torch.nonzero(present).flatten()
            self.rank_lut[nm] = (torch.cumsum(present.to(torch.int64), 0) - 1)
            table = FrequencyTable(uniq.cpu().numpy(), w[uniq].cpu().numpy(), ColumnKind.NUMERIC)
            self.dicts[nm] = Dictionary.build(table, "prefix_preserving")
        self.t_dict = time.perf_counter() - t0
        # ---- predicates
        self.bounds = {}
        d0, d1 = self.dicts["z0"], self.dicts["z1"]
        t0v, t1v = d0.table, d1.table
        z0lo = int(t0v.values[_q_from_counts(t0v.weights, self.n_total, 0.80)])
        z0hi = int(t0v.values[_q_from_counts(t0v.weights, self.n_total, 0.95)])
        z1q = int(t1v.values[_q_from_counts(t1v.weights, self.n_total, 0.60)])
        self.preds = {
            "u0": ResolvedPredicate.compare(Op.LT, qu0, 4),
            "u1": ResolvedPredicate.compare(Op.GE, qu1, 4),
            "z0": d0.encode_literal(Predicate("z0", Op.BETWEEN, z0lo, z0hi)),
            "z1": d1.encode_literal(Predicate("z1", Op.LE, z1q)),
        }
        self.raw_filter = {
            "u0": lambda v: v < qu0 - (1 << 31),
            "u1": lambda v: v >= qu1 - (1 << 31),
            "z0": lambda v: (v >= z0lo) & (v <= z0hi),
            "z1": lambda v: v <= z1q,
        }
        self.literals = {"u0": f"< {qu0 - (1 << 31)}", "u1": f">= {qu1 - (1 << 31)}",
                         "z0": f"BETWEEN {z0lo} AND {z0hi}", "z1": f"<= {z1q}"}
        # ---- layouts, one segment at a time
        t0 = time.perf_counter()
        self.cols = {nm: [] for nm, _ in COLS}
        self.layout = {"u0": "byteslice", "u1": "byteslice", "z0": "ppvbs", "z1": "ppvbs"}
        for nm, kind in COLS:
            for si in range(len(self.segs)):
                if kind == "uniform":
                    c = biased(raw[nm][si])
                    self.cols[nm].append(build_byteslice(c, 32))
                    del c
                else:
                    ranks = self.rank_lut[nm][raw[nm][si].to(torch.int64)]
                    codes, lens = self.dicts[nm].row_codes_device(ranks)
                    del ranks
                    self.cols[nm].append(build_vbs(codes, lens))
                    del codes, lens
                torch.cuda.empty_cache()
        del self.rank_lut
        torch.cuda.synchronize()
        self.t_build = time.perf_counter() - t0
        self.raw = raw if keep_raw else None
        if not keep_raw:
            del raw
            torch.cuda.empty_cache()

    # ------------------------------------------------------------------
    def col_bytes(self) -> int:
        total = 0
        for nm, _ in COLS:
            for c in self.cols[nm]:
                if hasattr(c, "planes"):
                    total += c.planes.numel()
                else:
                    total += c.bs1.numel()
                    for j in range(c.max_len):
                        if c.deep[j] is not None:
                            total += c.deep[j].numel() * c.deep[j].element_size()
                        if j >= 1:
                            total += c.exist[j].numel() * 4
                            if c.block_dir[j] is not None:
                                total += c.block_dir[j].numel() * 8
                            if c.rexist is not None and c.rexist[j] is not None:
                                total += c.rexist[j].numel() * 4
        return total

    def free_raw(self):
        import torch
        self.raw = None
        torch.cuda.empty_cache()


class Cfg5Step:
    """Preallocated result buffers + the C ABI calls of one step."""

    def __init__(self, tab: Cfg5Table, id_capacity: int):
        import torch

        from paper_2209_00220_b200 import _lib
        self.tab = tab
        self.lib = _lib.load()
        S = len(tab.segs)
        n = tab.seg_rows
        nw = -(-n // 32)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.words = {q: [torch.empty(nw, dtype=torch.int32, device=dev) for _ in range(S)]
                      for q in QUERIES}
        self.counts = torch.zeros(len(QUERIES), S, dtype=torch.int64, device=dev)
        self.totals = torch.zeros(len(QUERIES), dtype=torch.int64, device=dev)
        self.ids = torch.empty(max(1, id_capacity), dtype=torch.int64, device=dev)
        self.cpreds = {nm: tab.preds[nm].to_c() for nm in ("u0", "u1", "z0", "z1")}
        self.conj_refs = []
        for si in range(S):
            refs = (_lib.BsbColumnRef * 4)()
            for i, nm in enumerate(("u0", "u1", "z0", "z1")):
                c = tab.cols[nm][si]
                if tab.layout[nm] == "ppvbs":
                    refs[i].layout = _lib.LAYOUT_PPVBS
                    refs[i].vbs = ctypes.pointer(c._desc)
                else:
                    refs[i].layout = _lib.LAYOUT_BYTESLICE
                    refs[i].byteslice = ctypes.pointer(c._desc)
            self.conj_refs.append(refs)
        self.conj_preds = (_lib.BsbPred * 4)(*[self.cpreds[nm] for nm in ("u0", "u1", "z0",
                                                                           "z1")])
        self.kernels_per_step = None

    def calls(self, q: str, si: int):
        """(fn, args) of query q on segment si (C ABI)."""
        lib, tab = self.lib, self.tab
        out = self.words[q][si].data_ptr()
        cnt = self.counts[QUERIES.index(q), si:].data_ptr()
        if q == "and4":
            return lib.bsb_conj_scan, (4, self.conj_refs[si], self.conj_preds, None, out, cnt)
        col = tab.cols[q][si]
        fn = lib.bsb_vbs_scan if tab.layout[q] == "ppvbs" else lib.bsb_byteslice_scan
        return fn, (col.desc_ref, ctypes.byref(self.cpreds[q]), None, out, cnt, None, None)

    def run_query(self, q: str, sptr, events=None):
        from paper_2209_00220_b200 import _lib
        for si in range(len(self.tab.segs)):
            fn, args = self.calls(q, si)
            if events is not None:
                events[si][0].record()
            _lib.check(fn(*args, sptr), f"cfg5 {q}")
            if events is not None:
                events[si][1].record()

    def compact(self, sptr):
        """The AND's matches as global int64 row ids (ascending), no sync."""
        from paper_2209_00220_b200 import _lib
        import torch
        qi = QUERIES.index("and4")
        base = torch.cumsum(self.counts[qi], 0) - self.counts[qi]
        self._base = base
        for si, r0 in enumerate(self.tab.seg_starts):
            _lib.check(self.lib.bsb_bits_to_rows_at(
                self.words["and4"][si].data_ptr(), self.tab.seg_rows, r0,
                base[si:].data_ptr(), self.ids.data_ptr(), None, sptr), "cfg5 compact")

    def local(self, streams):
        """Everything rank-local of one step, forked over `streams` (query q
        on streams[q % len]); the caller joins them."""
        import torch

        from paper_2209_00220_b200.device import stream as cur_stream  # noqa: F401
        for i, q in enumerate(QUERIES):
            st = streams[i % len(streams)]
            with torch.cuda.stream(st):
                self.run_query(q, st.cuda_stream)
                if q == "and4":
                    self.compact(st.cuda_stream)
        main = streams[0]
        for st in streams[1:]:
            main.wait_stream(st)
        with torch.cuda.stream(main):
            torch.sum(self.counts, 1, out=self.totals)


def check_parity(tab: Cfg5Table, step: Cfg5Step, log=print) -> dict:
    """Every segment's bitvector of every query == the packed device filter
    of its raw values; AND's compacted ids == raw filter rows + segment start;
    counts == filter popcounts.  Raises on any mismatch."""
    import torch
    step.local([torch.cuda.current_stream()])
    torch.cuda.synchronize()
    n = tab.seg_rows
    got_ids = step.ids
    pos = 0
    sel = {q: 0 for q in QUERIES}
    for si in range(len(tab.segs)):
        want_and = None
        for nm, _ in COLS:
            v = tab.raw[nm][si]
            m = tab.raw_filter[nm](v)
            want_and = m if want_and is None else want_and & m
            w = pack_bools(m)
            if not torch.equal(step.words[nm][si], w):
                raise AssertionError(f"cfg5 {nm} segment {tab.segs[si]}: bitvector mismatch")
            c = int(m.sum().item())
            if int(step.counts[QUERIES.index(nm), si].item()) != c:
                raise AssertionError(f"cfg5 {nm} segment {tab.segs[si]}: count mismatch")
            sel[nm] += c
        if not torch.equal(step.words["and4"][si], pack_bools(want_and)):
            raise AssertionError(f"cfg5 AND segment {tab.segs[si]}: bitvector mismatch")
        rows = torch.nonzero(want_and).flatten() + tab.seg_starts[si]
        c = rows.numel()
        if int(step.counts[QUERIES.index("and4"), si].item()) != c:
            raise AssertionError(f"cfg5 AND segment {tab.segs[si]}: count mismatch")
        if not torch.equal(got_ids[pos:pos + c], rows):
            raise AssertionError(f"cfg5 AND segment {tab.segs[si]}: global row ids mismatch")
        pos += c
        sel["and4"] += c
    return sel


def alg_bytes(tab: Cfg5Table) -> dict:
    """Per-query algorithmic bytes summed over this rank's segments
    (reference-identical ScanStats depths; the AND
    pipelined with each later predicate's input-mask term)."""
    from paper_2209_00220_b200.byteslice import scan_byteslice
    from paper_2209_00220_b200.roofline import scan_alg_bytes
    from paper_2209_00220_b200.vbs import scan_vbs
    out = {q: 0 for q in QUERIES}
    for si in range(len(tab.segs)):
        running = None
        for nm, _ in COLS:
            c = tab.cols[nm][si]
            lay = tab.layout[nm]
            fn = scan_vbs if lay == "ppvbs" else scan_byteslice
            K = c.max_len if lay == "ppvbs" else c.n_slices
            ex = ([c.mask_words(j) for j in range(2, K + 1)] if lay == "ppvbs" else None)
            _, st = fn(c, tab.preds[nm])
            out[nm] += scan_alg_bytes(st.materialize().block_depth, lay, K, ex)
            bv, st = fn(c, tab.preds[nm], running)
            out["and4"] += scan_alg_bytes(st.materialize().block_depth, lay, K, ex,
                                          masked=running is not None)
            running = bv
    return out


def kernel_times(step: Cfg5Step, reps: int = 3) -> dict:
    """Mean device ms of each query's per-segment C ABI call (eager, events
    on the launching stream)."""
    import torch
    out = {}
    S = len(step.tab.segs)
    for q in QUERIES:
        evs = [[[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)]
                for _ in range(S)] for _ in range(reps)]
        for r in range(reps):
            step.run_query(q, torch.cuda.current_stream().cuda_stream, evs[r])
        torch.cuda.synchronize()
        out[q] = statistics.mean(e[0].elapsed_time(e[1]) for rr in evs for e in rr)
    return out


def cpu_sample(tab: Cfg5Table, m: int, threads: int, reps: int = 1) -> dict:
    """The oracle port of the reference algorithm on the first m rows of the
    rank's first segment of every column: the 5 queries (the AND pipelined,
    engine.py:322-332), all threads and 1 thread.  Returns Gcodes/s."""
    import oracle as O
    import torch
    h = {nm: tab.raw[nm][0][:m].cpu().numpy().astype(np.int64) for nm, _ in COLS}
    cols = {}
    for nm, kind in COLS:
        if kind == "uniform":
            cols[nm] = ("bs", O.bs_build((h[nm] + (1 << 31)).astype(np.uint64), 32))
        else:
            d = tab.dicts[nm]
            ranks = np.searchsorted(d.table.values, h[nm])
            cols[nm] = ("vbs", O.vbs_build(d.assignment.codes[ranks],
                                           d.assignment.lengths[ranks]))
    opreds = {nm: _opred(tab.preds[nm]) for nm in ("u0", "u1", "z0", "z1")}

    def one(nm, mask, th):
        kind, c = cols[nm]
        if kind == "bs":
            return O.bs_scan(c, 32, m, opreds[nm], mask, threads=th)[0]
        return O.vbs_scan(c, opreds[nm], mask, threads=th)[0]

    def run(th):
        t0 = time.perf_counter()
        for nm in ("u0", "u1", "z0", "z1"):
            one(nm, None, th)
        run_m = None
        for nm in ("u0", "u1", "z0", "z1"):
            run_m = one(nm, run_m, th)
        O.words_to_rows(run_m, m)
        return time.perf_counter() - t0

    run(threads)  # warm-up
    t_all = statistics.median(run(threads) for _ in range(reps))
    t_one = run(1)
    del torch
    return {"all": 8 * m / t_all / 1e9, "one": 8 * m / t_one / 1e9, "rows": m}


def _opred(rp):
    import oracle as O
    from paper_2209_00220_b200.predicate import Op
    if rp.is_trivial:
        return O.pred_const(rp.trivial)
    if rp.op is Op.BETWEEN:
        return O.pred_between(rp.code, rp.length, rp.code2, rp.length2)
    return O.pred_compare(rp.op.name, rp.code, rp.length)
