"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (the reference is mounted read-only there):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``bytestore`` from /root/reference/pkg/src unchanged, feeds it
seeded inputs and records inputs + outputs into ``tests/golden/*.npz``.  The
committed fixtures then pin both the CPU oracle (``oracle/``, CPU tests) and
the CUDA product (``-m gpu`` tests) on the GPU box, where /root/reference does
not exist.

Families:
  zipf.npz      gen_zipf draws (pins the numpy PCG64 + searchsorted stream)
  dict.npz      ppe_numerical / fixed_assignment codes, literal resolution,
                decode_padded
  bs.npz        ByteSlice build + scans (all ops, BETWEEN, masks) + stats +
                lookups
  vbs.npz       PP-VBS build + scans + stats + lookups (random and PPE codes)
  advisor.npz   advise_column(cost="bytes") points / AUCs / choices
  fixture.npz   numeric columns of the reference's fixture_1000.csv and the
                row ids of its pinned query (n_selected == 192)
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

from bytestore import bits as rbits  # noqa: E402
from bytestore.advisor import advise_column  # noqa: E402
from bytestore.bitvector import ResultBitVector  # noqa: E402
from bytestore.byteslice import build_byteslice, lookup_byteslice, scan_byteslice  # noqa: E402
from bytestore.datagen import ZipfSpec, gen_zipf  # noqa: E402
from bytestore.dictionary import (ColumnKind, Dictionary, build_frequency_table,  # noqa: E402
                                  fixed_assignment, ppe_numerical)
from bytestore.engine import ColumnSpec, Query, Schema, execute, ingest  # noqa: E402
from bytestore.predicate import Op, Predicate, ResolvedPredicate  # noqa: E402
from bytestore.vbs import build_vbs, lookup_vbs, scan_vbs  # noqa: E402

OPS = ["EQ", "NE", "LT", "LE", "GT", "GE"]


def _pred_tuple(r: ResolvedPredicate):
    if r.is_trivial:
        return [None, 0, 0, 0, 0, bool(r.trivial)]
    return [r.op.name, int(r.code), int(r.length), int(r.code2), int(r.length2), None]


def _stats(st, prefix, out):
    out[prefix + "words_loaded"] = np.asarray(st.words_loaded, np.int64)
    out[prefix + "bytes_loaded"] = np.asarray(st.bytes_loaded, np.int64)
    out[prefix + "block_depth"] = np.asarray(st.block_depth, np.int8)
    out[prefix + "misc"] = np.array([st.levels, st.blocks_total, st.blocks_skipped,
                                     st.mask_bytes, st.total_bytes], np.int64)


def gen_zipf_family():
    out, meta = {}, []
    specs = [(0.0, 12, 5000, 1), (1.0, 12, 5000, 3), (1.2, 20, 20000, 42),
             (1.5, 8, 3000, 7), (1.1, 24, 4096, 500), (0.8, 16, 4096, 101)]
    for i, (s, d, n, seed) in enumerate(specs):
        out[f"{i}/values"] = gen_zipf(ZipfSpec(s, d, n, seed))
        meta.append({"s": s, "d": d, "n": n, "seed": seed})
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, "zipf.npz"), **out)


def gen_dict_family():
    out, meta = {}, []
    rng = np.random.default_rng(2024)
    tables = [np.arange(300, 0, -1), np.arange(256, 0, -1), np.ones(70000, np.int64),
              np.array([5, 4, 3]), np.array([7])]
    w = np.ones(300, np.int64)
    w[7] = 0
    tables.append(w)
    for n in (2, 100, 255, 256, 300, 600, 2000, 5000):
        tables.append(rng.integers(1, 10**6, size=n))
        z = (1e6 / np.arange(1, n + 1) ** 1.2).astype(np.int64) + 1
        rng.shuffle(z)
        tables.append(z)
        spiky = np.ones(n, np.int64)
        spiky[rng.integers(0, n, size=max(1, n // 50))] = 10**6
        tables.append(spiky)
    # a realistic Zipf table (cfg2-like, smaller)
    v = gen_zipf(ZipfSpec(1.2, 20, 1 << 18, seed=42))
    tables.append(np.unique(v, return_counts=True)[1])
    for i, t in enumerate(tables):
        a = ppe_numerical(t)
        out[f"ppe{i}/weights"] = np.asarray(t, np.int64)
        out[f"ppe{i}/codes"] = a.codes
        out[f"ppe{i}/lengths"] = a.lengths
    out["n_ppe"] = np.array(len(tables))
    widths = [(n, fixed_assignment(n).width_bits) for n in
              (1, 2, 3, 4, 255, 256, 257, 300, 4096, 4097, 1 << 20, (1 << 20) + 1)]
    out["fixed_widths"] = np.array(widths, np.int64)

    # literal resolution + decode on a few numeric dictionaries
    res = []
    for k, (vals, scheme) in enumerate([
            (np.array([0, 2, 4]), "prefix_preserving"),
            (np.array([0, 2, 4]), "fixed"),
            (gen_zipf(ZipfSpec(1.2, 12, 20000, seed=5)), "prefix_preserving"),
            (gen_zipf(ZipfSpec(1.2, 12, 20000, seed=5)), "fixed"),
            (gen_zipf(ZipfSpec(1.0, 16, 50000, seed=6)), "prefix_preserving"),
            (rng.integers(-500, 500, size=3000), "prefix_preserving")]):
        table = build_frequency_table(vals, ColumnKind.NUMERIC)
        d = Dictionary.build(table, scheme)
        out[f"res{k}/values"] = np.asarray(vals, np.int64)
        lo, hi = int(table.values.min()), int(table.values.max())
        lits = sorted(set([lo - 1, lo, lo + 1, hi - 1, hi, hi + 1] +
                          rng.integers(lo - 3, hi + 4, size=25).tolist() +
                          rng.choice(table.values, size=10).tolist()))
        cases = []
        for lit in lits:
            for op in OPS:
                r = d.encode_literal(Predicate("c", Op[op], int(lit)))
                cases.append([op, int(lit), None] + _pred_tuple(r))
        for _ in range(20):
            a, b = sorted(rng.integers(lo - 3, hi + 4, size=2).tolist())
            r = d.encode_literal(Predicate("c", Op.BETWEEN, int(a), int(b)))
            cases.append(["BETWEEN", int(a), int(b)] + _pred_tuple(r))
        res.append({"scheme": scheme, "cases": cases})
        if scheme == "prefix_preserving":
            out[f"res{k}/padded"] = d.padded
            out[f"res{k}/decoded"] = d.decode_padded(d.padded)
    out["resolution"] = np.array(json.dumps(res))
    np.savez_compressed(os.path.join(HERE, "dict.npz"), **out)


def _bs_cases(rng):
    cols = []
    for w in (1, 7, 8, 11, 16, 20, 24, 32):
        for n in (97, 1000, 5000):
            cols.append((w, rng.integers(0, 1 << w, size=n, dtype=np.uint64)))
    # early-stop statistics case (tests/test_byteslice.py:91-103 shape)
    cols.append((11, rng.integers(0, 2048, size=32 * 2000, dtype=np.uint64)))
    return cols


def gen_bs_family():
    rng = np.random.default_rng(77)
    out, meta = {}, []
    for ci, (w, codes) in enumerate(_bs_cases(rng)):
        n = len(codes)
        col = build_byteslice(codes, w)
        out[f"{ci}/codes"] = codes
        out[f"{ci}/slices"] = col.slices
        mask = ResultBitVector.from_bools(rng.random(n) < 0.5)
        out[f"{ci}/mask"] = mask.words
        preds = []
        pool = [int(codes[3]), 0, (1 << w) - 1, int(codes[3]) ^ 1, int(codes[n // 2])]
        for lit in pool:
            for op in OPS:
                preds.append(ResolvedPredicate.compare(Op[op], lit, col.n_slices))
        a, b = sorted(int(x) for x in codes[[5, 9]])
        preds.append(ResolvedPredicate.between(a, col.n_slices, b, col.n_slices))
        preds.append(ResolvedPredicate.between(b, col.n_slices, a, col.n_slices))
        preds.append(ResolvedPredicate.constant(True))
        preds.append(ResolvedPredicate.constant(False))
        plist = []
        for pi, p in enumerate(preds):
            for mi, m in enumerate((None, mask)):
                res, st = scan_byteslice(col, p, m)
                key = f"{ci}/p{pi}m{mi}/"
                out[key + "words"] = res.words
                _stats(st, key, out)
            plist.append(_pred_tuple(p))
        sel = ResultBitVector.from_bools(rng.random(n) < 0.3)
        got, lst = lookup_byteslice(col, sel)
        out[f"{ci}/sel"] = sel.words
        out[f"{ci}/lookup"] = got
        out[f"{ci}/lookup_stats"] = np.array([lst.levels_touched, lst.bytes_loaded,
                                              lst.mask_bytes], np.int64)
        meta.append({"w": w, "n": n, "preds": plist})
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, "bs.npz"), **out)


def _random_vbs(rng, n, max_len):
    lens = rng.integers(1, max_len + 1, size=n).astype(np.uint8)
    byts = rng.integers(0, 256, size=(n, 8), dtype=np.uint64)
    byts[:, 0] |= np.uint64(1)          # final byte nonzero (codes never end in 0)
    codes = np.zeros(n, np.uint64)
    for k in range(8):
        use = lens > k
        codes[use] |= byts[use, k] << np.uint64(8 * k)
    return codes, lens


def gen_vbs_family():
    rng = np.random.default_rng(99)
    out, meta = {}, []
    cols = []
    cols.append((np.array([0x81, 0xC0, 0x77A9, 0x8189], np.uint64),
                 np.array([1, 1, 2, 2], np.uint8)))
    for n in (5, 32, 97, 1000, 4096):
        cols.append(_random_vbs(rng, n, 3))
    cols.append(_random_vbs(rng, 2048, 4))
    cols.append(_random_vbs(rng, 1500, 8))
    for s, d, n, seed in ((1.2, 20, 1 << 15, 42), (1.0, 12, 20000, 3), (1.5, 16, 20000, 9),
                          (0.0, 12, 20000, 4)):
        vals = gen_zipf(ZipfSpec(s, d, n, seed))
        t = build_frequency_table(vals, ColumnKind.NUMERIC)
        dp = Dictionary.build(t, "prefix_preserving")
        ranks = Dictionary.build(t, "fixed").encode_rows(vals)
        c, l = dp.row_codes(ranks)
        cols.append((c.astype(np.uint64), l.astype(np.uint8)))
    for ci, (codes, lens) in enumerate(cols):
        n = len(codes)
        col = build_vbs(codes, lens)
        K = col.max_len
        out[f"{ci}/codes"] = codes
        out[f"{ci}/lens"] = lens
        out[f"{ci}/bs1"] = col.slices[0]
        for j in range(2, K + 1):
            out[f"{ci}/bs{j}"] = col.slices[j - 1]
            out[f"{ci}/m{j}"] = col.mask_words(j).astype(np.uint32)
        out[f"{ci}/dir"] = col.block_dir
        mask = ResultBitVector.from_bools(rng.random(n) < 0.4)
        out[f"{ci}/mask"] = mask.words
        padded = [int(c) << (8 * (K - int(l))) for c, l in zip(codes, lens)]
        pool = []
        rows = rng.integers(0, n, size=5)
        for r in rows:
            pool.append((int(codes[r]), int(lens[r])))
        pool += [(1, 1), (0xFF, 1), (int(codes[rows[0]]) ^ 1, int(lens[rows[0]]))]
        if K >= 2:
            pool.append((int(codes[rows[1]]) >> 8 if lens[rows[1]] > 1 else 1,
                         max(1, int(lens[rows[1]]) - 1)))
        preds = []
        for lit, ll in pool:
            for op in OPS:
                preds.append(ResolvedPredicate.compare(Op[op], lit, ll))
        srt = sorted(range(n), key=lambda i: padded[i])
        for _ in range(4):
            a, b = sorted(rng.integers(0, n, size=2).tolist())
            ia, ib = srt[a], srt[b]
            preds.append(ResolvedPredicate.between(int(codes[ia]), int(lens[ia]),
                                                   int(codes[ib]), int(lens[ib])))
        preds.append(ResolvedPredicate.constant(True))
        preds.append(ResolvedPredicate.constant(False))
        plist = []
        for pi, p in enumerate(preds):
            for mi, m in enumerate((None, mask)):
                res, st = scan_vbs(col, p, m)
                key = f"{ci}/p{pi}m{mi}/"
                out[key + "words"] = res.words
                _stats(st, key, out)
            plist.append(_pred_tuple(p))
        for si, dens in enumerate((0.01, 0.3, 1.0)):
            sel = ResultBitVector.from_bools(rng.random(n) < dens)
            got, lst = lookup_vbs(col, sel)
            out[f"{ci}/sel{si}"] = sel.words
            out[f"{ci}/lookup{si}"] = got
            out[f"{ci}/lookup_stats{si}"] = np.array([lst.levels_touched, lst.bytes_loaded,
                                                      lst.mask_bytes], np.int64)
        meta.append({"n": n, "K": K, "preds": plist})
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, "vbs.npz"), **out)


def gen_advisor_family():
    out, meta = {}, []
    rng = np.random.default_rng(9)
    cols = [gen_zipf(ZipfSpec(0.0, 12, 100_000, seed=2)),
            gen_zipf(ZipfSpec(1.5, 12, 100_000, seed=2)),
            gen_zipf(ZipfSpec(1.2, 10, 30_000, seed=9)),
            rng.integers(0, 1 << 12, size=50_000, dtype=np.int64),
            gen_zipf(ZipfSpec(1.0, 8, 50_000, seed=4)),
            np.arange(1000) % 7]
    params = [(20, None), (20, None), (10, None), (20, None), (5, 2000), (5, None)]
    for i, (vals, (count, sub)) in enumerate(zip(cols, params)):
        a = advise_column("c", vals, ColumnKind.NUMERIC, count=count, cost="bytes",
                          subsample=sub)
        out[f"{i}/values"] = np.asarray(vals, np.int64)
        out[f"{i}/pts_bs"] = np.array([[p.selectivity, p.time] for p in a.points_byteslice])
        out[f"{i}/pts_vbs"] = np.array([[p.selectivity, p.time] for p in a.points_ppvbs])
        meta.append({"count": count, "subsample": sub, "chosen": a.chosen,
                     "auc_bs": a.auc_byteslice, "auc_vbs": a.auc_ppvbs})
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, "advisor.npz"), **out)


def gen_fixture_family():
    """Numeric columns of the reference fixture and its pinned conjunction."""
    csv = "/root/reference/pkg/tests/fixtures/fixture_1000.csv"
    schema = Schema([ColumnSpec("qty", Schema.parse_kind("numeric"), "byteslice"),
                     ColumnSpec("amount", Schema.parse_kind("numeric"), "ppvbs")])
    store, _ = ingest(csv, schema, policy="forced")
    q = execute(store, Query.conjunction(
        [Predicate("amount", Op.LE, 4), Predicate("qty", Op.GT, 50)], ["amount", "qty"]))
    assert q.n_selected == 192  # tests/test_acceptance.py:463
    out = {
        "qty": store.columns["qty"].dictionary.decode_ranks(
            lookup_byteslice(store.columns["qty"].column,
                             ResultBitVector.ones(store.n_rows))[0]).astype(np.int64),
        "amount": store.columns["amount"].dictionary.decode_padded(
            lookup_vbs(store.columns["amount"].column,
                       ResultBitVector.ones(store.n_rows))[0]).astype(np.int64),
        "selection": q.selection.words,
        "proj_amount": np.asarray(q.columns["amount"], np.int64),
        "proj_qty": np.asarray(q.columns["qty"], np.int64),
        "n_selected": np.array(q.n_selected),
    }
    np.savez_compressed(os.path.join(HERE, "fixture.npz"), **out)


def gen_bits_family():
    rng = np.random.default_rng(3)
    xs = rng.integers(0, 1 << 32, size=(500, 2), dtype=np.uint64)
    rows = []
    for src, mask in xs.tolist():
        rows.append([src, mask, rbits.pdep(src, mask), rbits.pext(src, mask)])
    np.savez_compressed(os.path.join(HERE, "bits.npz"), pdep_pext=np.array(rows, np.uint64))


if __name__ == "__main__":
    gen_bits_family()
    gen_zipf_family()
    gen_dict_family()
    gen_bs_family()
    gen_vbs_family()
    gen_advisor_family()
    gen_fixture_family()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
