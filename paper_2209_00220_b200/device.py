"""Device plumbing: the CUDA device, stream and tensor conversions.

PyTorch is used only for device memory, streams and host<->device copies;
every compute step goes through libbytestore_b200.so.  There is no CPU
fallback: without a CUDA device the device path raises.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

__all__ = ["device", "require_cuda", "to_dev_i64", "to_dev_u64", "to_dev_u8", "to_dev_u32",
           "host_u32", "host_u64", "stream"]


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2209_00220_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    _lib.load()


def device() -> torch.device:
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def stream():
    return _lib.stream_ptr()


_BIT_CARRIERS = {(torch.uint64, torch.int64), (torch.uint32, torch.int32),
                 (torch.int8, torch.uint8)}


def _to_dev(x, np_dtype, view_dtype, torch_dtype):
    """Integer data only: floating / bool / complex inputs raise TypeError
    (numpy fancy indexing rejects them too).  Integer dtypes convert by
    value; only the unsigned<->signed carrier pairs of the same width
    (uint64 codes in int64, uint32 words in int32) are reinterpreted."""
    if isinstance(x, torch.Tensor):
        t = x
        if t.dtype.is_floating_point or t.dtype.is_complex or t.dtype == torch.bool:
            raise TypeError(f"expected an integer tensor, got {t.dtype}")
        dev = device()
        if t.dtype != torch_dtype:
            if (t.dtype, torch_dtype) in _BIT_CARRIERS:
                t = t.view(torch_dtype)
            else:
                t = t.to(torch_dtype)
        return t.to(dev, non_blocking=True).contiguous()
    a = np.asarray(x)
    if a.dtype.kind not in "iu" and not (a.dtype == object or a.size == 0):
        raise TypeError(f"expected integer data, got {a.dtype}")
    a = np.ascontiguousarray(a.astype(np_dtype, copy=False))
    return torch.from_numpy(a.view(view_dtype)).to(device(), non_blocking=False)


def to_dev_i64(x) -> torch.Tensor:
    return _to_dev(x, np.int64, np.int64, torch.int64)


def to_dev_u64(x) -> torch.Tensor:
    """uint64 codes stored bit-for-bit in an int64 tensor."""
    if isinstance(x, torch.Tensor):
        return _to_dev(x, np.uint64, np.int64, torch.int64)
    a = np.asarray(x)
    if a.dtype.kind == "i" and (a < 0).any():
        raise ValueError("codes must be non-negative")
    return _to_dev(a.astype(np.uint64), np.uint64, np.int64, torch.int64)


def to_dev_u8(x) -> torch.Tensor:
    return _to_dev(x, np.uint8, np.uint8, torch.uint8)


def to_dev_u32(x) -> torch.Tensor:
    """uint32 words stored bit-for-bit in an int32 tensor."""
    return _to_dev(x, np.uint32, np.int32, torch.int32)


def host_u32(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint32)


def host_u64(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


# Row-id gathers: lists at least this long that are not ascending are sorted
# before the lookup and the output is scattered back (bsb_rows_sort).
SORT_GATHER_MIN = 1 << 16


def gather_order(rows: torch.Tensor, n_rows: int, order: str = "auto"):
    """(ids to gather, perm or None).  order="sort": an ascending list is
    gathered as it is, any other list of >= SORT_GATHER_MIN ids in row-bucket
    order with perm mapping back to input positions (bsb_rows_sort); "keep":
    as given.  The lookups choose per layout what "auto" means."""
    import ctypes

    if order not in ("sort", "keep"):
        raise ValueError(f"unknown order {order!r}")
    n = rows.numel()
    if order == "keep" or n < SORT_GATHER_MIN:
        return rows, None
    lib = _lib.load()
    srt = torch.empty_like(rows)
    perm = torch.empty_like(rows)
    was = ctypes.c_int32(1)
    _lib.check(lib.bsb_rows_sort(rows.data_ptr(), n, int(n_rows), srt.data_ptr(),
                                 perm.data_ptr(), ctypes.byref(was), stream()), "gather_order")
    return (rows, None) if was.value else (srt, perm)


# Row-id gathers over big columns: lists at least this long are partitioned
# into bucket-ordered (row, position) pairs (bsb_rows_bucket) unless ascending.
# Measured crossover on a 2^28-row, 3-slice column (tools/auto_probe.py):
# 2^20 ids 72 us as given vs 118 us bucketed, 2^22 ids 256 vs 232, 2^24 ids
# 1000 vs 620.
BUCKET_GATHER_MIN = 1 << 22
BUCKET_ROWS_MIN = 1 << 24
_PAIR_LIMIT = (1 << 32) - 1


def auto_gather(n_ids: int, n_rows: int) -> bool:
    """Whether order="auto" takes the *_lookup_rows_auto entry points (order
    check and bucket partition chosen on the device): long lists over big
    columns whose sizes fit the 32-bit pairs."""
    return (BUCKET_GATHER_MIN <= n_ids < _PAIR_LIMIT and BUCKET_ROWS_MIN <= n_rows < _PAIR_LIMIT)


def gather_pairs(rows: torch.Tensor, n_rows: int, check: bool = False):
    """(pairs, unsorted) for the *_lookup_pairs entry points: pairs =
    bucket-ordered row | position << 32 words (bsb_rows_bucket); unsorted =
    None, or with check=True the device word holding the sampled order
    check's verdict (0: the list looks ascending and pairs[] was not written;
    the pair lookups then gather the list as given).  One list can serve
    several columns of the same table.  Never synchronises."""
    n = rows.numel()
    if n >= _PAIR_LIMIT or n_rows >= _PAIR_LIMIT:
        raise ValueError("bucket-ordered pairs hold 32-bit rows and positions")
    lib = _lib.load()
    pairs = torch.empty(n, dtype=torch.int64, device=rows.device)
    uns = torch.empty(1, dtype=torch.int32, device=rows.device) if check else None
    _lib.check(lib.bsb_rows_bucket(rows.data_ptr(), n, int(n_rows), pairs.data_ptr(),
                                   _lib.ptr(uns), stream()), "gather_pairs")
    return pairs, uns


def row_gather_plan(rows: torch.Tensor, n_rows: int, order: str, auto_fn, pairs_fn, rows_fn):
    """(fn, ids, perm) for a row-id lookup under `order`: fn(desc, ids, n, ...)
    is the C entry point to call with the remaining arguments.  "auto": the
    *_auto entry for long lists over big columns, else as given; "bucket":
    bucket-ordered pairs (no order check); "sort": the sort + scatter-back
    path (gather_order); "keep": as given."""
    if order not in ("auto", "sort", "bucket", "keep"):
        raise ValueError(f"unknown order {order!r}")
    n = rows.numel()
    if order == "auto" and auto_gather(n, n_rows):
        return auto_fn, rows, None
    if order == "bucket" and 0 < n < _PAIR_LIMIT and n_rows < _PAIR_LIMIT:
        pairs, _ = gather_pairs(rows, n_rows)

        def fn(desc, ids, *rest):
            return pairs_fn(desc, ids, None, None, *rest)
        return fn, pairs, None
    g, perm = gather_order(rows, n_rows, "sort" if order == "sort" else "keep")
    return rows_fn, g, perm


def scatter_back(out: torch.Tensor, perm) -> torch.Tensor:
    """Output of a gather over sorted ids back in input order."""
    if perm is None:
        return out
    res = torch.empty_like(out)
    _lib.check(_lib.load().bsb_scatter(out.data_ptr(), perm.data_ptr(), out.numel(),
                                       out.element_size(), res.data_ptr(), stream()),
               "scatter_back")
    return res
