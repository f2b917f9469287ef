"""The README's usage example (run from the repo root: python tools/readme_example.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import paper_2209_00220_b200 as B
from paper_2209_00220_b200 import engine as E
from paper_2209_00220_b200.predicate import Op, Predicate

vals = B.gen_zipf(B.ZipfSpec(1.2, 20, 1 << 24, seed=42))      # reference datagen
store, _ = E.ingest_arrays({"v": vals, "u": np.arange(1 << 24)})  # advisor picks layouts
res = E.execute(store, E.Query.conjunction(
    [Predicate("v", Op.BETWEEN, 1000, 5000), Predicate("u", Op.GE, 10)], ["v", "u"]))
print(res.n_selected, res.columns["v"][:5])
B.write_store("/tmp/t.byst", store)   # byte-identical to the reference's write_store
print(B.read_store("/tmp/t.byst").n_rows)
