"""Golden BYST store files written by the REFERENCE itself (store.py).

Run in the build container (the reference is mounted read-only there):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_store.py

Seeded numeric columns are written to a temporary CSV, ingested by the
reference (`engine.ingest`, forced layouts and the advisor in "bytes" cost
mode) and serialised with `store.write_store`; the resulting files and the raw
columns go to tests/golden/store_*.byst + store.npz.  tests/ checks that this
package writes the same bytes from the same columns and reads the reference's
files into device layouts that scan and look up identically.
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
from bytestore.dictionary import ColumnKind  # noqa: E402
from bytestore.engine import ColumnSpec, Schema, ingest  # noqa: E402
from bytestore.store import write_store  # noqa: E402


def columns():
    n = 3001
    rng = np.random.default_rng(900)
    return {
        "u12": rng.integers(0, 1 << 12, n),
        "neg": rng.integers(-50_000, 50_000, n),
        "z16": gen_zipf(ZipfSpec(1.1, 16, n, 901)),
        "z20": gen_zipf(ZipfSpec(0.9, 20, n, 902)),
        "const": np.full(n, 7, np.int64),
    }


CASES = {
    # forced layouts: each column in the layout named here
    "forced": {"u12": "byteslice", "neg": "ppvbs", "z16": "ppvbs", "z20": "byteslice",
               "const": "byteslice"},
    # advisor in bytes mode (deterministic), every column advised
    "advised": {"u12": None, "neg": None, "z16": None, "z20": None, "const": None},
}


def main():
    cols = columns()
    names = list(cols)
    with tempfile.TemporaryDirectory() as tmp:
        csv_path = os.path.join(tmp, "cols.csv")
        with open(csv_path, "w") as fh:
            fh.write(",".join(names) + "\n")
            for row in zip(*(cols[k] for k in names)):
                fh.write(",".join(str(int(x)) for x in row) + "\n")
        meta = {}
        for case, layouts in CASES.items():
            schema = Schema([ColumnSpec(k, ColumnKind.NUMERIC, layouts[k]) for k in names])
            policy = "forced" if all(v is not None for v in layouts.values()) else "advisor"
            store, _ = ingest(csv_path, schema, policy, advise_cost="bytes", advise_count=20)
            out = os.path.join(HERE, f"store_{case}.byst")
            write_store(out, store)
            meta[case] = {"policy": policy, "layouts": layouts, "advise_count": 20,
                          "size": os.path.getsize(out)}
    np.savez_compressed(os.path.join(HERE, "store.npz"),
                        **{f"col/{k}": v for k, v in cols.items()},
                        meta=np.array(json.dumps(meta)))
    print(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
