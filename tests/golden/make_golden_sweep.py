"""Deterministic columns of the reference's layout sweep (bench.py:59-107):
selectivity and bits per code for every layout, produced by the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_sweep.py
"""

import json
import os
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

from bytestore.bench import SweepSpec, run_sweep  # noqa: E402

if __name__ == "__main__":
    spec = SweepSpec(s_values=[0.5, 1.2], domain_bits=10, n_rows=20000, reps=1)
    rows = run_sweep(spec)
    keep = [{k: r[k] for k in ("layout", "s", "d", "n_rows", "selectivity", "bits_per_code")}
            for r in rows]
    with open(os.path.join(HERE, "sweep.json"), "w") as fh:
        json.dump({"spec": {"s_values": [0.5, 1.2], "domain_bits": 10, "n_rows": 20000},
                   "rows": keep}, fh, indent=1)
    print(json.dumps(keep[:3]))
