"""Row-range sharding across the GPUs of one box.

Each rank owns a contiguous, tile-aligned row range [r0, r1) of every column
and scans it independently with the device kernels; the reference already
guarantees that any block-aligned partition concatenates bit-exactly
(SPEC.md:284, vbs.py:211-215, :317-323).  Per query exactly ONE collective
runs: an all_gather of the per-rank int64 match counts, from which every
rank derives the global count and its exclusive-prefix offset for compacted
global row ids.  Dictionaries are global (built from the all-gathered local
frequency tables) and replicated.

The exchange logic is device-agnostic: with NCCL the count tensor lives on
the GPU; the CPU tests drive the same code over gloo with the oracle as the
per-shard scan.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

__all__ = ["shard_range", "ShardResult", "exchange_counts", "sharded_scan",
           "global_row_ids", "merge_frequency_tables", "gather_row_ids", "global_sum",
           "owned_segments", "compact_segments", "global_nearest_rank_u32",
           "exclusive_offsets"]

TILE_ROWS = 1024
# A table larger than one kernel's comfortable row range is stored as fixed
# row-range segments (row groups) of this many rows; a rank owns a contiguous
# run of segments, so every segment boundary is also a tile boundary.
SEGMENT_ROWS = 1 << 29


def shard_range(n_total: int, world: int, rank: int, align: int = TILE_ROWS):
    """Contiguous [r0, r1) of rank, aligned to `align` rows (tiles never
    straddle GPUs, so result words never do either)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    per = -(-n_total // world)
    per = -(-per // align) * align
    r0 = min(n_total, rank * per)
    r1 = min(n_total, r0 + per)
    return r0, r1


def owned_segments(n_segments: int, world: int, rank: int) -> range:
    """Contiguous segments [lo, hi) of rank: the row-range partition at
    segment granularity (SPEC.md:284 -- any block-aligned partition
    concatenates bit-exactly).  Every rank owns at least one segment."""
    if world < 1 or not 0 <= rank < world or n_segments < world:
        raise ValueError("need 0 <= rank < world <= n_segments")
    return range(n_segments * rank // world, n_segments * (rank + 1) // world)


def exclusive_offsets(counts: torch.Tensor) -> torch.Tensor:
    """Exclusive prefix sum of int64 counts, on their device (no host sync)."""
    c = counts.reshape(-1).to(torch.int64)
    return torch.cumsum(c, 0) - c


def compact_segments(seg_words, seg_rows, seg_starts, seg_counts: torch.Tensor,
                     out: torch.Tensor, stream_ptr=None) -> None:
    """Global int64 row ids of several segments' matches, compacted into
    `out` in ascending row order without a host sync: segment s's ids
    (seg_starts[s] + local row) land at the exclusive prefix of seg_counts
    (device int64, one per segment) -- bitvector.py:71-72 per segment.
    `out` must hold the rank's total count."""
    from . import _lib
    from .device import stream as cur_stream
    lib = _lib.load()
    base = exclusive_offsets(seg_counts)
    sp = cur_stream() if stream_ptr is None else stream_ptr
    for s, (w, n, r0) in enumerate(zip(seg_words, seg_rows, seg_starts)):
        _lib.check(lib.bsb_bits_to_rows_at(w.data_ptr(), int(n), int(r0),
                                           base[s:].data_ptr(), out.data_ptr(), None, sp),
                   "compact_segments")
    return base


def global_nearest_rank_u32(chunks, fractions, n_total: int, group=None):
    """Exact nearest-rank quantiles sorted(v)[min(n-1, floor(x*n))] (the
    advisor's literal rule, advisor.py:56-59) of uint32 values spread over
    ranks and chunks (int64 tensors holding 0..2^32-1), by a two-level radix
    select: a 2^16-bin histogram of the high halves, all-reduced, picks each
    quantile's bin; a second histogram of the low halves inside that bin
    picks the value.  Two small all_reduces per quantile, no sort."""
    dev = chunks[0].device
    dist_on = dist.is_available() and dist.is_initialized()

    def hist(fn):
        h = torch.zeros(1 << 16, dtype=torch.int64, device=dev)
        for c in chunks:
            for p in torch.split(c, 1 << 27):
                v = fn(p)
                if v.numel():
                    h += torch.bincount(v, minlength=1 << 16)
        if dist_on:
            dist.all_reduce(h, group=group)
        return h

    hi = torch.cumsum(hist(lambda p: p >> 16), 0).cpu().numpy()
    out = []
    for x in fractions:
        k = min(n_total - 1, int(x * n_total))
        b = int(np.searchsorted(hi, k, side="right"))
        k2 = k - (int(hi[b - 1]) if b else 0)
        lo = torch.cumsum(hist(lambda p, b=b: (p[(p >> 16) == b] & 0xFFFF)), 0).cpu().numpy()
        out.append((b << 16) | int(np.searchsorted(lo, k2, side="right")))
    return out


@dataclass
class ShardResult:
    rank: int
    world: int
    r0: int
    r1: int
    local_bits: object        # DeviceBitVector (or host words for CPU tests)
    local_count: int
    global_count: int
    offset: int               # global position of this rank's first match
    counts: list


def exchange_counts(local_count, group=None):
    """ONE all_gather of int64 counts -> (counts per rank, global, offset).

    `local_count` is a 1-element int64 tensor on the collective's device
    (CUDA for NCCL, CPU for gloo) -- no host sync before the collective.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bufs = [torch.zeros_like(local_count) for _ in range(world)]
    dist.all_gather(bufs, local_count, group=group)
    counts = [int(b.item()) for b in bufs]
    return counts, sum(counts), sum(counts[:rank])


def sharded_scan(local_scan, n_total: int, group=None):
    """Run this rank's shard scan and combine counts.

    local_scan(r0, r1) -> (bits, count_tensor) scans rows [r0, r1) of this
    rank's columns (device: engine.conj_scan over the shard columns).
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    r0, r1 = shard_range(n_total, world, rank)
    bits, cnt = local_scan(r0, r1)
    counts, total, offset = exchange_counts(cnt.reshape(1).to(torch.int64), group)
    return ShardResult(rank, world, r0, r1, bits, counts[rank], total, offset, counts)


def global_row_ids(res: ShardResult) -> torch.Tensor:
    """This rank's matches as global int64 row ids (positions
    res.offset .. res.offset + local_count of the global id array)."""
    bits = res.local_bits
    if hasattr(bits, "row_ids"):
        return bits.row_ids(row_offset=res.r0)
    words = np.asarray(bits, dtype=np.uint32)
    flags = np.unpackbits(words.view(np.uint8), bitorder="little")[: res.r1 - res.r0]
    return torch.from_numpy(np.flatnonzero(flags).astype(np.int64) + res.r0)


def gather_row_ids(res: ShardResult, ids: torch.Tensor, group=None) -> torch.Tensor | None:
    """All ranks' global ids concatenated in rank order (== the unsharded
    ascending id list).  Uses an all_gather of padded tensors."""
    width = max(res.counts) if res.counts else 0
    pad = torch.full((max(width, 1),), -1, dtype=torch.int64, device=ids.device)
    pad[: ids.numel()] = ids
    bufs = [torch.empty_like(pad) for _ in range(res.world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:c] for b, c in zip(bufs, res.counts)])


def merge_frequency_tables(values: torch.Tensor, counts: torch.Tensor, group=None):
    """Global (values, counts) from every rank's local frequency table.

    Local tables are padded to the largest size, all_gathered, then merged
    by value with a segmented sum (setup path, not per query)."""
    world = dist.get_world_size(group)
    n = torch.tensor([values.numel()], dtype=torch.int64, device=values.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    width = max(sizes)
    pv = torch.zeros(width, dtype=torch.int64, device=values.device)
    pc = torch.zeros(width, dtype=torch.int64, device=values.device)
    pv[: values.numel()] = values
    pc[: counts.numel()] = counts
    gv = [torch.empty_like(pv) for _ in range(world)]
    gc = [torch.empty_like(pc) for _ in range(world)]
    dist.all_gather(gv, pv, group=group)
    dist.all_gather(gc, pc, group=group)
    allv = torch.cat([v[:s] for v, s in zip(gv, sizes)])
    allc = torch.cat([c[:s] for c, s in zip(gc, sizes)])
    uniq, inv = torch.unique(allv, sorted=True, return_inverse=True)
    tot = torch.zeros(uniq.numel(), dtype=torch.int64, device=values.device)
    tot.scatter_add_(0, inv, allc)
    return uniq, tot


def global_sum(local_sum: torch.Tensor, group=None) -> torch.Tensor:
    """a projected column's SUM over all shards -- each rank's
    local int64 sum, then one all_reduce (in place, on the collective's
    device)."""
    out = local_sum.reshape(1).to(torch.int64).clone()
    dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out

