"""Golden vectors for categorical and ordered-string columns, produced by the
REFERENCE itself (dictionary.py / engine.py / store.py).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_strings.py

Seeded string columns go through a temporary CSV into `engine.ingest`
(forced layouts, and the advisor in "bytes" cost mode); the store files are
written with `store.write_store`, and a set of queries is run with
`engine.execute`.  Outputs: tests/golden/strings_{forced,advised}.byst and
strings.npz (raw columns, ppe_categorical codes for several sizes, literal
resolutions, query selections and projected values).
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

from bytestore.datagen import ZipfSpec, gen_zipf  # noqa: E402
from bytestore.dictionary import (ColumnKind, Dictionary, build_frequency_table,  # noqa: E402
                                  ppe_categorical)
from bytestore.engine import ColumnSpec, Query, Schema, execute, ingest  # noqa: E402
from bytestore.predicate import Op, Predicate  # noqa: E402
from bytestore.store import write_store  # noqa: E402

KINDS = {"cat_a": ColumnKind.CATEGORICAL, "cat_b": ColumnKind.CATEGORICAL,
         "ostr": ColumnKind.ORDERED_STRING, "num": ColumnKind.NUMERIC}


def columns():
    n = 2500
    za = gen_zipf(ZipfSpec(1.3, 10, n, 910))
    zb = gen_zipf(ZipfSpec(0.6, 12, n, 911))
    zo = gen_zipf(ZipfSpec(1.0, 12, n, 912))
    rng = np.random.default_rng(913)
    return {
        "cat_a": np.array([f"k{v:04d}" for v in za]),
        "cat_b": np.array([("x" * (1 + v % 3)) + str(v) for v in zb]),
        "ostr": np.array([f"s{v:05d}" for v in zo]),
        "num": rng.integers(-1000, 1000, n),
    }


CASES = {
    "forced": {"cat_a": "ppvbs", "cat_b": "byteslice", "ostr": "ppvbs", "num": "byteslice"},
    "advised": {k: None for k in KINDS},
}


def queries(cols):
    ca = cols["cat_a"]
    u, c = np.unique(ca, return_counts=True)
    top, rare = str(u[np.argmax(c)]), str(u[np.argmin(c)])
    so = np.sort(cols["ostr"])
    return [
        [[Predicate("cat_a", Op.EQ, top)]],
        [[Predicate("cat_a", Op.NE, rare), Predicate("cat_b", Op.EQ, str(cols["cat_b"][7]))]],
        [[Predicate("cat_a", Op.EQ, "absent")], [Predicate("cat_b", Op.NE, "absent")]],
        [[Predicate("ostr", Op.BETWEEN, str(so[300]), str(so[1500]))]],
        [[Predicate("ostr", Op.LT, "s00005"), Predicate("num", Op.GE, 0)]],
        [[Predicate("ostr", Op.GE, "s00100"), Predicate("cat_b", Op.EQ, str(cols["cat_b"][3]))]],
    ]


def main():
    cols = columns()
    names = list(cols)
    out = {f"col/{k}": v for k, v in cols.items()}
    meta = {"cases": {}}
    # ppe_categorical codes for sizes that cross the 1-, 2- and 3-byte depths
    sizes = [1, 2, 254, 255, 256, 300, 65280, 65281, 70000]
    for i, n in enumerate(sizes):
        a = ppe_categorical(n)
        out[f"ppecat/{i}/codes"] = a.codes
        out[f"ppecat/{i}/lengths"] = a.lengths
    meta["ppecat_sizes"] = sizes
    # frequency tables + literal resolution
    lits = {}
    for k in ("cat_a", "cat_b", "ostr"):
        t = build_frequency_table(cols[k], KINDS[k])
        out[f"table/{k}/values"] = t.values.astype(str)
        out[f"table/{k}/weights"] = t.weights
        for scheme in ("fixed", "prefix_preserving"):
            d = Dictionary.build(t, scheme)
            probes = [str(t.values[0]), str(t.values[-1]), str(t.values[len(t.values) // 2]),
                      "absent", "k0000", "s00050"]
            ops = [Op.EQ, Op.NE] + ([Op.LT, Op.LE, Op.GT, Op.GE] if KINDS[k].ordered else [])
            res = []
            for v in probes:
                for op in ops:
                    r = d.encode_literal(Predicate(k, op, v))
                    res.append([v, op.name, r.op.name if r.op else None, r.code, r.length,
                                r.trivial])
            lits[f"{k}/{scheme}"] = res
    meta["literals"] = lits
    with tempfile.TemporaryDirectory() as tmp:
        csv_path = os.path.join(tmp, "cols.csv")
        with open(csv_path, "w") as fh:
            fh.write(",".join(names) + "\n")
            for row in zip(*(cols[k] for k in names)):
                fh.write(",".join(str(x) for x in row) + "\n")
        for case, layouts in CASES.items():
            schema = Schema([ColumnSpec(k, KINDS[k], layouts[k]) for k in names])
            policy = "forced" if all(v is not None for v in layouts.values()) else "advisor"
            store, _ = ingest(csv_path, schema, policy, advise_cost="bytes", advise_count=20)
            write_store(os.path.join(HERE, f"strings_{case}.byst"), store)
            qres = []
            for qi, groups in enumerate(queries(cols)):
                res = execute(store, Query(groups, ["cat_a", "ostr", "num"]))
                out[f"q/{case}/{qi}/sel"] = res.selection.to_bools()
                for c in ("cat_a", "ostr", "num"):
                    out[f"q/{case}/{qi}/{c}"] = np.asarray(res.columns[c]).astype(
                        str if c != "num" else np.int64)
                qres.append(int(res.n_selected))
            meta["cases"][case] = {"policy": policy, "layouts": layouts, "advise_count": 20,
                                   "n_selected": qres,
                                   "chosen": {e["name"]: e["layout"]
                                              for e in store.manifest["columns"]}}
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(HERE, "strings.npz"), **out)
    print(json.dumps({k: v for k, v in meta.items() if k != "literals"}, indent=1))


if __name__ == "__main__":
    main()
