"""ByteSlice on the B200 (mirror of reference byteslice.py:34-169).

The device layout keeps the reference's byte planes (codes left-aligned,
plane j = byte j, MSB first) but stores each 32-row block swizzled (row r at
byte ((r & 7) << 2) | (r >> 3)) and pads planes to 1024-row tiles, so the scan
kernel reads one 256-bit sector per lane per plane.  ``slices`` exports the
reference layout for parity checks.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .bitvector import DeviceBitVector, as_device_bits
from .device import device, host_u64, row_gather_plan, scatter_back, stream, to_dev_i64, to_dev_u64
from .predicate import DEFAULT_LANES, LaneConfig, Op, ResolvedPredicate
from .stats import LazyScanStats, LookupStats, ScanStats

__all__ = ["ByteSliceColumn", "build_byteslice", "scan_byteslice", "lookup_byteslice",
           "lookup_byteslice_rows", "lookup_byteslice_bits", "byteslice_size_report"]


@dataclass
class ByteSliceColumn:
    """Device-resident ByteSlice column."""

    n_rows: int
    width_bits: int
    lanes: LaneConfig
    stride: int
    planes: torch.Tensor            # uint8 [n_slices * stride], swizzled blocks
    _desc: _lib.BsbByteSlice = field(default=None, repr=False)

    def __post_init__(self):
        d = _lib.BsbByteSlice()
        d.n_rows = self.n_rows
        d.stride = self.stride
        d.width_bits = self.width_bits
        d.n_slices = self.n_slices
        d.slices = self.planes.data_ptr()
        self._desc = d

    @property
    def n_slices(self) -> int:
        return -(-self.width_bits // 8)

    @property
    def n_blocks(self) -> int:
        return -(-self.n_rows // 32)

    @property
    def slices(self) -> np.ndarray:
        """Reference layout (n_slices, n_blocks*32) uint8, copied to the host."""
        out = torch.empty(self.n_slices * self.n_blocks * 32, dtype=torch.uint8,
                          device=self.planes.device)
        _lib.check(_lib.load().bsb_byteslice_export(ctypes.byref(self._desc), out.data_ptr(),
                                                    stream()), "export")
        return out.cpu().numpy().reshape(self.n_slices, -1)

    @property
    def desc_ref(self):
        return ctypes.byref(self._desc)


def build_byteslice(codes, width_bits: int, lanes: LaneConfig = DEFAULT_LANES
                    ) -> ByteSliceColumn:
    """byteslice.py:56-73 on the device.  ``codes``: numpy/list/torch, any device."""
    lanes.require_device()
    if not 1 <= int(width_bits) <= 64:
        raise ValueError("width must be 1..64 bits")
    is_ranks = isinstance(codes, torch.Tensor) and codes.dtype == torch.int64
    if isinstance(codes, torch.Tensor):
        n = codes.numel()
    else:
        codes = np.asarray(codes)
        n = len(codes)
        if codes.dtype.kind == "i" and codes.size and codes.min() >= 0:
            is_ranks = True
            codes = codes.astype(np.int64)
    if n == 0:
        raise ValueError("empty column")
    lib = _lib.load()
    K = -(-int(width_bits) // 8)
    stride = int(lib.bsb_stride_for(n))
    planes = torch.empty(K * stride, dtype=torch.uint8, device=device())
    if is_ranks:
        dc = to_dev_i64(codes)
        rc = lib.bsb_byteslice_build_ranks(dc.data_ptr(), n, int(width_bits), planes.data_ptr(),
                                           stride, stream())
    else:
        dc = to_dev_u64(codes)
        rc = lib.bsb_byteslice_build(dc.data_ptr(), n, int(width_bits), planes.data_ptr(),
                                     stride, stream())
    _lib.check(rc, "build_byteslice")
    return ByteSliceColumn(n, int(width_bits), lanes, stride, planes)


def _scan_stats(col: ByteSliceColumn, pred: ResolvedPredicate, mask,
                with_depth: bool = True) -> ScanStats:
    lib = _lib.load()
    nb = col.n_blocks
    dev = col.planes.device
    st = torch.zeros(_lib.STATS_WORDS, dtype=torch.int64, device=dev)
    depth = torch.zeros(max(nb, 1), dtype=torch.int8, device=dev) if with_depth else None
    out = torch.empty(nb, dtype=torch.int32, device=dev)
    cnt = torch.empty(1, dtype=torch.int64, device=dev)
    cp = pred.to_c()
    _lib.check(lib.bsb_byteslice_scan(col.desc_ref, ctypes.byref(cp),
                                      None if mask is None else mask.dwords.data_ptr(),
                                      out.data_ptr(), cnt.data_ptr(), st.data_ptr(),
                                      _lib.ptr(depth), stream()), "scan_byteslice(stats)")
    h = st.cpu().numpy()
    K = col.n_slices
    skipped = int(h[17])
    if pred.op is Op.BETWEEN:
        skipped = min(int(h[17]), int(h[19]))
    return ScanStats(levels=K, blocks_total=nb, blocks_skipped=skipped,
                     words_loaded=h[0:K].copy(), bytes_loaded=h[8:8 + K].copy(),
                     mask_bytes=0,
                     block_depth=None if depth is None else depth[:nb].cpu().numpy())


def scan_byteslice(col: ByteSliceColumn, pred: ResolvedPredicate, mask=None,
                   threads: int = 1):
    """byteslice.py:109-140: early-stopping scan of one resolved predicate.

    Returns (DeviceBitVector, ScanStats).  The stats are computed lazily (a
    second pass through the stats kernels) only if a field is read.
    ``threads`` is accepted for signature compatibility and ignored.
    """
    m = None
    if mask is not None:
        m = as_device_bits(mask)
        if m.n_rows != col.n_rows:
            raise ValueError("input mask length mismatch")
    lib = _lib.load()
    out = torch.empty(col.n_blocks, dtype=torch.int32, device=col.planes.device)
    cnt = torch.empty(1, dtype=torch.int64, device=col.planes.device)
    cp = pred.to_c()
    _lib.check(lib.bsb_byteslice_scan(col.desc_ref, ctypes.byref(cp),
                                      None if m is None else m.dwords.data_ptr(),
                                      out.data_ptr(), cnt.data_ptr(), None, None, stream()),
               "scan_byteslice")
    return DeviceBitVector(col.n_rows, out, cnt), LazyScanStats(
        lambda with_depth: _scan_stats(col, pred, m, with_depth))


def lookup_byteslice_rows(col: ByteSliceColumn, rows: torch.Tensor, rank_values=None,
                          out_dtype=torch.int64, order: str = "auto", err=None):
    """Device lookup of a row-id list (any order, duplicates allowed; output
    in input order).  Returns codes, or decoded values rank_values[code] when
    a device value table is given.  order="auto": a long list over a big
    column is partitioned into bucket-ordered (row, position) pairs first
    (bsb_rows_bucket: ids of one bucket share sectors and DRAM pages) unless
    a sampled check on the device finds it ascending, the results go back to
    their positions, and nothing synchronises; "bucket" skips the check, "keep" gathers the list as given, "sort"
    is the older sort + scatter-back path (device.gather_order).
    rank_values None + out_dtype int32: the codes as int32.  An id outside
    [0, n_rows) raises IndexError (synchronises), unless `err` (a zeroed
    device int32 word) is given: then the call stays asynchronous and
    _lib.ERR_INDEX is OR-ed into it."""
    lib = _lib.load()
    rows = to_dev_i64(rows)
    n = rows.numel()
    fn, g, perm = row_gather_plan(rows, col.n_rows, order, lib.bsb_byteslice_lookup_rows_auto,
                                  lib.bsb_byteslice_lookup_pairs, lib.bsb_byteslice_lookup_rows)
    if rank_values is None:
        if out_dtype == torch.int32:  # codes as int32 (identity dictionaries)
            out = torch.empty(n, dtype=torch.int32, device=rows.device)
            _lib.check(fn(col.desc_ref, g.data_ptr(), n, None, None, None, out.data_ptr(),
                          _lib.ptr(err), stream()), "lookup_byteslice")
            return scatter_back(out, perm)
        out = torch.empty(n, dtype=torch.int64, device=rows.device)
        _lib.check(fn(col.desc_ref, g.data_ptr(), n, out.data_ptr(), None, None, None,
                      _lib.ptr(err), stream()), "lookup_byteslice")
        return scatter_back(out, perm)
    out = torch.empty(n, dtype=out_dtype, device=rows.device)
    p64 = out.data_ptr() if out_dtype == torch.int64 else None
    p32 = out.data_ptr() if out_dtype == torch.int32 else None
    _lib.check(fn(col.desc_ref, g.data_ptr(), n, None, rank_values.data_ptr(), p64, p32,
                  _lib.ptr(err), stream()), "lookup_byteslice")
    return scatter_back(out, perm)


def lookup_byteslice_bits(col: ByteSliceColumn, selection, decoder=None,
                          out_dtype=torch.int64):
    """Fused selection -> codes (or decoded values with a rank-table
    decoder), ascending row order, no row-id array materialised."""
    sel = as_device_bits(selection)
    if sel.n_rows != col.n_rows:
        raise ValueError("selection length mismatch")
    n = sel.count()
    dev = col.planes.device
    cnt = torch.empty(1, dtype=torch.int64, device=dev)
    lib = _lib.load()
    out = torch.empty(max(n, 1), dtype=torch.int64 if decoder is None else out_dtype,
                      device=dev)
    if decoder is None:
        _lib.check(lib.bsb_byteslice_lookup_bits(col.desc_ref, sel.dwords.data_ptr(), None,
                                                 out.data_ptr(), None, None, cnt.data_ptr(),
                                                 stream()), "lookup_byteslice")
        return out[:n]
    p64 = out.data_ptr() if out_dtype == torch.int64 else None
    p32 = out.data_ptr() if out_dtype == torch.int32 else None
    _lib.check(lib.bsb_byteslice_lookup_bits(col.desc_ref, sel.dwords.data_ptr(),
                                             ctypes.byref(decoder), None, p64, p32,
                                             cnt.data_ptr(), stream()), "lookup_byteslice")
    if int(cnt.item()) == -1:
        raise LookupError("lookup_byteslice: code not in dictionary")
    return out[:n]


def lookup_byteslice(col: ByteSliceColumn, selection):
    """byteslice.py:143-158: codes of the selected rows, ascending row order."""
    if selection.n_rows != col.n_rows:
        raise ValueError("selection length mismatch")
    rows = as_device_bits(selection).row_ids()
    n = rows.numel()
    if n == 0:
        return np.zeros(0, np.uint64), LookupStats()
    codes = lookup_byteslice_rows(col, rows)
    st = LookupStats(levels_touched=col.n_slices, bytes_loaded=n * col.n_slices)
    return host_u64(codes), st


def byteslice_size_report(col: ByteSliceColumn) -> dict:
    """byteslice.py:161-169."""
    data = col.n_slices * col.n_rows
    return {"slice_bytes": [col.n_rows] * col.n_slices, "mask_bytes": 0,
            "directory_bytes": 0, "total_bytes": data,
            "avg_bits_per_code": 8.0 * data / col.n_rows}
