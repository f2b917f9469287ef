"""Golden vectors for the baseline layouts (Bit-Packed, VBP, PE-VBP) produced
by the REFERENCE itself (bitpacked.py, vbp.py, dictionary.py, store.py).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_baseline.py

Records: packed bit streams / planes, scan words + VBP ScanStats for every
operator (with and without an input mask, BETWEEN as two pipelined legs),
lookups, prefix_free_assignment codes, and a store file holding all five
layouts (forced) written by `store.write_store`.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

from bytestore.bitpacked import build_bitpacked, lookup_bitpacked, scan_bitpacked  # noqa: E402
from bytestore.bitvector import ResultBitVector  # noqa: E402
from bytestore.datagen import ZipfSpec, gen_zipf  # noqa: E402
from bytestore.dictionary import (ColumnKind, Dictionary, build_frequency_table,  # noqa: E402
                                  prefix_free_assignment)
from bytestore.engine import ColumnSpec, Query, Schema, execute, ingest  # noqa: E402
from bytestore.predicate import Op, Predicate, ResolvedPredicate  # noqa: E402
from bytestore.store import write_store  # noqa: E402
from bytestore.vbp import build_vbp, lookup_vbp, pad_codes, scan_vbp  # noqa: E402

OPS = ["EQ", "NE", "LT", "LE", "GT", "GE"]


def stats_dict(st):
    return {"levels": st.levels, "blocks_total": st.blocks_total,
            "blocks_skipped": st.blocks_skipped,
            "words_loaded": [int(x) for x in st.words_loaded],
            "bytes_loaded": [int(x) for x in st.bytes_loaded],
            "mask_bytes": int(st.mask_bytes), "total_bytes": int(st.total_bytes),
            "block_depth": st.block_depth.astype(np.int8)}


def main():
    out, meta = {}, {"cases": []}
    rng = np.random.default_rng(950)
    ci = 0
    for n, w in ((1, 1), (33, 3), (1000, 7), (4099, 13), (20_000, 17), (9000, 32)):
        codes = rng.integers(0, 1 << w, n, dtype=np.uint64) if w < 64 else None
        bp = build_bitpacked(codes, w)
        vb = build_vbp(codes, w, "plain")
        out[f"c{ci}/codes"] = codes
        out[f"c{ci}/bits"] = bp.bits
        out[f"c{ci}/planes"] = vb.planes
        mask = ResultBitVector.from_bools(rng.random(n) < 0.6)
        out[f"c{ci}/mask"] = mask.words
        preds = []
        for k in range(3):
            lit = int(codes[rng.integers(0, n)])
            for op in OPS:
                preds.append(ResolvedPredicate.compare(Op[op], lit, (w + 7) // 8))
            a, b = sorted(int(x) for x in rng.choice(codes, 2))
            preds.append(ResolvedPredicate.between(a, (w + 7) // 8, b, (w + 7) // 8))
        preds += [ResolvedPredicate.constant(True), ResolvedPredicate.constant(False)]
        pl = []
        for pi, p in enumerate(preds):
            for mi, m in enumerate((None, mask)):
                r1 = scan_bitpacked(bp, p, m)
                r2, st = scan_vbp(vb, p, m)
                out[f"c{ci}/p{pi}/m{mi}/bp"] = r1.words
                out[f"c{ci}/p{pi}/m{mi}/vbp"] = r2.words
                for k2, v in stats_dict(st).items():
                    out[f"c{ci}/p{pi}/m{mi}/st/{k2}"] = np.asarray(v)
            pl.append([p.op.name if p.op else None, p.code, p.length, p.code2, p.length2,
                       p.trivial])
        sel = ResultBitVector.from_bools(rng.random(n) < 0.3)
        out[f"c{ci}/sel"] = sel.words
        out[f"c{ci}/lookup_bp"] = lookup_bitpacked(bp, sel)
        lv, lst = lookup_vbp(vb, sel)
        out[f"c{ci}/lookup_vbp"] = lv
        meta["cases"].append({"n": n, "w": w, "preds": pl})
        ci += 1
    # prefix-free (PE-VBP) dictionaries and padded-encoding columns
    pf = []
    for i, (s, d, n) in enumerate(((1.0, 8, 3000), (1.5, 12, 20000), (0.0, 6, 500))):
        v = gen_zipf(ZipfSpec(s, d, n, 960 + i))
        t = build_frequency_table(v, ColumnKind.NUMERIC)
        a = prefix_free_assignment(t.weights)
        out[f"pf{i}/values"] = v
        out[f"pf{i}/weights"] = t.weights
        out[f"pf{i}/codes"] = a.codes
        out[f"pf{i}/lengths"] = a.lengths
        out[f"pf{i}/width"] = np.array(a.width_bits)
        dct = Dictionary.build(t, "prefix_free")
        ranks = dct.encode_rows(v)
        c, l = dct.row_codes(ranks)
        col = build_vbp(pad_codes(c, l, a.width_bits), a.width_bits, "padded_encoding")
        out[f"pf{i}/planes"] = col.planes
        srt = np.sort(v)
        lits = []
        for k, (lo, hi) in enumerate(((0.1, 0.3), (0.5, 0.9), (0.0, 0.01))):
            p = dct.encode_literal(Predicate("c", Op.BETWEEN, int(srt[int(lo * n)]),
                                             int(srt[min(n - 1, int(hi * n))])))
            r, st = scan_vbp(col, p)
            out[f"pf{i}/q{k}/words"] = r.words
            for k2, vv in stats_dict(st).items():
                out[f"pf{i}/q{k}/st/{k2}"] = np.asarray(vv)
            padded, _ = lookup_vbp(col, r)
            out[f"pf{i}/q{k}/decoded"] = dct.decode_padded(padded)
            lits.append([p.op.name if p.op else None, p.code, p.length, p.code2, p.length2,
                         p.trivial])
        pf.append({"s": s, "d": d, "n": n, "preds": lits})
    meta["prefix_free"] = pf
    # store with every layout (forced) + one query
    n = 3000
    cols = {"a": rng.integers(0, 5000, n), "b": gen_zipf(ZipfSpec(1.2, 12, n, 970)),
            "c": rng.integers(-100, 100, n), "d": gen_zipf(ZipfSpec(0.8, 10, n, 971)),
            "e": rng.integers(0, 1 << 20, n)}
    layouts = {"a": "bitpacked", "b": "pevbp", "c": "vbp", "d": "ppvbs", "e": "byteslice"}
    with tempfile.TemporaryDirectory() as tmp:
        p = os.path.join(tmp, "c.csv")
        with open(p, "w") as fh:
            fh.write(",".join(cols) + "\n")
            for row in zip(*cols.values()):
                fh.write(",".join(str(int(x)) for x in row) + "\n")
        schema = Schema([ColumnSpec(k, ColumnKind.NUMERIC, layouts[k]) for k in cols])
        store, _ = ingest(p, schema, "forced")
        write_store(os.path.join(HERE, "baseline_store.byst"), store)
        sb = np.sort(cols["b"])
        q = [[Predicate("a", Op.LT, 2500), Predicate("b", Op.BETWEEN, int(sb[300]),
                                                     int(sb[2000])),
              Predicate("c", Op.NE, 0)], [Predicate("d", Op.EQ, int(cols["d"][0]))]]
        res = execute(store, Query(q, list(cols)))
        out["store/sel"] = res.selection.to_bools()
        for k in cols:
            out[f"store/col/{k}"] = cols[k]
            out[f"store/proj/{k}"] = np.asarray(res.columns[k])
    meta["store_layouts"] = layouts
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, "baseline.npz"), **out)
    print(len(out), "arrays;", os.path.getsize(os.path.join(HERE, "baseline.npz")), "bytes")


if __name__ == "__main__":
    main()
