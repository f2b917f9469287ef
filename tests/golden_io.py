"""Loaders for the reference-generated golden fixtures (tests/golden/*.npz)."""

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)
    data = {k: z[k] for k in z.files}
    meta = json.loads(str(data.pop("meta"))) if "meta" in data else None
    return data, meta


def stats_of(data, key):
    misc = data[key + "misc"]
    return {
        "words_loaded": data[key + "words_loaded"],
        "bytes_loaded": data[key + "bytes_loaded"],
        "block_depth": data[key + "block_depth"],
        "levels": int(misc[0]), "blocks_total": int(misc[1]),
        "blocks_skipped": int(misc[2]), "mask_bytes": int(misc[3]),
        "total_bytes": int(misc[4]),
    }
