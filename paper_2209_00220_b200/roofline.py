"""Algorithmic-byte accounting for the roofline.

Scan algorithmic bytes are derived from the reference-identical ScanStats
block depths (the stats kernels reproduce stats.py bit-exactly), so they are
implementation independent and count each needed byte once, even for a fused
BETWEEN (merged depth = max over legs, stats.py:58):

  alg = sum_b sum_{j<=depth_b} bytes_j(b)          slice bytes the early stop must read
      + [PP-VBS] 4 * sum_{b: depth_b>=1} (min(depth_b+1, K) - 1)   existence words
      + 4 * nb                                        result bitvector write
      + 4 * nb * [input mask given]                   pipelined mask read

bytes_j(b) = 32 for level 1 and every ByteSlice level, popc(M_j[b]) for PP-VBS
levels j >= 2.
"""

from __future__ import annotations

import json
import os

import numpy as np

__all__ = ["scan_alg_bytes", "lookup_alg_bytes_rows", "hbm_peak"]

FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def hbm_peak(root: str | None = None):
    """(GB/s, source) from MEASURED_PEAKS.json, else the profiling guide fallback."""
    root = root or os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = os.path.join(root, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            v = float(json.load(fh)["hbm_gbs"])
        return v, "measured"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM_GBS, "fallback"


def scan_alg_bytes(depth: np.ndarray, layout: str, K: int, exist_words=None,
                   masked: bool = False) -> int:
    """Algorithmic bytes of one scan from its per-block depth (int8[nb])."""
    d = np.asarray(depth).astype(np.int64)
    nb = len(d)
    out = 4 * nb * (2 if masked else 1)
    if layout == "byteslice":
        return out + 32 * int(d.sum())
    out += 32 * int((d >= 1).sum())
    for j in range(2, K + 1):
        pop = np.bitwise_count(np.asarray(exist_words[j - 2], dtype=np.uint32)[:nb])
        out += int(pop.astype(np.int64)[d >= j].sum())
    live = d >= 1
    out += 4 * int((np.minimum(d[live] + 1, K) - 1).sum())
    return out


def lookup_alg_bytes_rows(rows: np.ndarray, K: int, layout: str, exist_words=None,
                          out_bytes: int = 4, id_bytes: int = 8, table_bytes: int = 0) -> int:
    """Distinct-32B-sector lower bound for a row-id lookup.

    ByteSlice: one sector per (plane, block).  PP-VBS: BS_1 sector per block,
    existence word sectors for every level tested, directory entry and deep
    byte sectors for levels the row has.  Plus ids in, values out, table once.
    """
    r = np.asarray(rows, dtype=np.int64)
    blocks = np.unique(r >> 5)
    total = r.size * (id_bytes + out_bytes) + table_bytes
    if layout == "byteslice":
        return total + 32 * K * blocks.size
    total += 32 * blocks.size  # BS_1
    alive = r
    for j in range(2, K + 1):
        w = np.asarray(exist_words[j - 2], dtype=np.uint32)
        b = alive >> 5
        total += 32 * np.unique(b >> 3).size          # 8 existence words per sector
        has = ((w[b] >> (alive & 31).astype(np.uint32)) & 1).astype(bool)
        alive = alive[has]
        if alive.size == 0:
            break
        total += 32 * np.unique((alive >> 5) >> 3).size   # u32 dir: 8 per sector
        total += 32 * np.unique(alive >> 5).size          # deep bytes of a block ~ 1 sector
    return int(total)
