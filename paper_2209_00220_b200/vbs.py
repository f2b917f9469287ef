"""PP-VBS (variable byte slices) on the B200 (mirror of reference vbs.py:42-517).

Device layout = the reference's arrays: BS_1 (swizzled per 32-row block like
ByteSlice, padded to 1024-row tiles), packed deep slices BS_j in row order,
one uint32 existence word per block per deep slice, and the int64 block
directory.  Scans use a per-tile warp prefix over existence popcounts instead
of reading the directory; lookups read the directory.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .bitvector import DeviceBitVector, as_device_bits
from .device import (auto_gather, device, gather_order, host_u32, row_gather_plan, host_u64, scatter_back, stream, to_dev_i64,
                     to_dev_u8, to_dev_u64)
from .predicate import DEFAULT_LANES, LaneConfig, Op, ResolvedPredicate
from .stats import LazyScanStats, LookupStats, ScanStats

__all__ = ["VbsColumn", "build_vbs", "scan_vbs", "lookup_vbs", "lookup_vbs_rows",
           "lookup_vbs_rows_dec", "lookup_vbs_bits", "vbs_size_report", "scan_serial",
           "lookup_serial"]

DEEP_PAD = 64


@dataclass
class VbsColumn:
    """Device-resident PP-VBS column."""

    n_rows: int
    max_len: int
    lanes: LaneConfig
    stride: int
    bs1: torch.Tensor                     # uint8 [stride], swizzled blocks
    deep: list                            # deep[j] (j=1..K-1): uint8 packed slice j+1
    exist: list                           # exist[j]: int32 [stride/32] words of slice j+1
    block_dir: list                       # block_dir[j]: int64 [stride/32 + 1]
    level_rows: list                      # rows owning byte j (j = 1..K), reference counts
    deep_mode: int = _lib.DEEP_PACKED     # DEEP_PACKED / DEEP_SLICED (header)
    rexist: list = None                   # SLICED: deep-row bitmaps of byte j+1 (j>=2)
    deep1_range: tuple = (1, 0)           # (min, max) first byte of the deep rows; (1, 0) unknown
    _desc: _lib.BsbVbs = field(default=None, repr=False)

    def __post_init__(self):
        d = _lib.BsbVbs()
        d.n_rows = self.n_rows
        d.stride = self.stride
        d.max_len = self.max_len
        d.deep_mode = self.deep_mode
        d.bs1 = self.bs1.data_ptr()
        lo, hi = self.deep1_range
        d.deep1_shared = lo + 1 if lo == hi else 0  # zone map: shared first byte + 1
        if self.deep and self.deep[0] is not None:  # SLICED: deep rows' first byte
            d.deep[0] = self.deep[0].data_ptr()
            d.deep_len[0] = self.deep[0].numel() - DEEP_PAD
        for j in range(1, self.max_len):
            if self.deep[j] is not None:
                d.deep[j] = self.deep[j].data_ptr()
                d.deep_len[j] = self.deep[j].numel() * self.deep[j].element_size() - DEEP_PAD
            d.exist[j] = self.exist[j].data_ptr()
            if self.block_dir[j] is not None:
                d.block_dir[j] = self.block_dir[j].data_ptr()
            if self.rexist is not None and self.rexist[j] is not None:
                d.rexist[j] = self.rexist[j].data_ptr()
        self._desc = d

    @property
    def desc_ref(self):
        return ctypes.byref(self._desc)

    @property
    def n_blocks(self) -> int:
        return -(-self.n_rows // 32)

    def slice_len(self, j: int) -> int:
        return self.n_rows if j == 1 else int(self.level_rows[j - 1])

    # reference-layout views (host copies) --------------------------------
    @property
    def slices(self) -> list:
        npad = self.n_blocks * 32
        first = torch.empty(npad, dtype=torch.uint8, device=self.bs1.device)
        _lib.check(_lib.load().bsb_vbs_export_bs1(self.desc_ref, first.data_ptr(), stream()),
                   "export")
        out = [first.cpu().numpy()]
        for j in range(2, self.max_len + 1):
            out.append(self._export_level(j)[0])
        return out

    def _export_level(self, j: int):
        """Reference packing (bytes, block_dir) of slice j, from either mode."""
        nb = self.n_blocks
        by = torch.empty(max(self.level_rows[j - 1], 1), dtype=torch.uint8, device=self.bs1.device)
        dr = torch.empty(nb + 1, dtype=torch.int64, device=self.bs1.device)
        _lib.check(_lib.load().bsb_vbs_export_level(self.desc_ref, j, by.data_ptr(),
                                                    dr.data_ptr(), stream()), "export")
        return by[: self.level_rows[j - 1]].cpu().numpy(), dr.cpu().numpy()

    def mask_words(self, j: int) -> np.ndarray:
        """Existence words of slice j (j >= 2), one per block (vbs.py:58-61)."""
        return host_u32(self.exist[j - 1][: self.n_blocks])

    @property
    def exist_bits(self) -> list:
        return [self.mask_words(j).view(np.uint8) for j in range(2, self.max_len + 1)]

    @property
    def block_dir_host(self) -> np.ndarray:
        """Reference block directory (K-1, nb+1) int64 (vbs.py:95, :105-106)."""
        nb = self.n_blocks
        rows = [self._export_level(j)[1] for j in range(2, self.max_len + 1)]
        return np.stack(rows) if rows else np.zeros((0, nb + 1), np.int64)


SLICED_MAX_OVERHEAD = 1.30


def choose_deep_mode(level_rows, K: int) -> int:
    """SLICED (deep rows as their own swizzled ByteSlice column; the fastest
    scan, measured on B200) when its pad bytes cost <= 30% over the reference
    packing -- true for PPE dictionaries, whose deep codes are mostly full
    length -- else the reference packing."""
    if K < 2:
        return _lib.DEEP_PACKED
    exact = sum(int(level_rows[j]) for j in range(1, K))
    cnt2 = int(level_rows[1])
    if (K - 1) * (-(-cnt2 // 32) * 32) <= SLICED_MAX_OVERHEAD * exact:
        return _lib.DEEP_SLICED
    return _lib.DEEP_PACKED


def build_vbs(row_codes, row_lengths, lanes: LaneConfig = DEFAULT_LANES,
              deep_mode: str = "auto") -> VbsColumn:
    """vbs.py:68-114 on the device: plan (validate, K, level sizes) + build.

    deep_mode: "auto" | "packed" (reference packing) | "sliced" (the deep
    rows as their own swizzled byte-plane column); see
    include/bytestore_b200.h."""
    lanes.require_device()
    codes = row_codes if isinstance(row_codes, torch.Tensor) else np.asarray(row_codes)
    lens = row_lengths if isinstance(row_lengths, torch.Tensor) else np.asarray(row_lengths)
    n = codes.numel() if isinstance(codes, torch.Tensor) else len(codes)
    nl = lens.numel() if isinstance(lens, torch.Tensor) else len(lens)
    if n == 0:
        raise ValueError("empty column")
    if nl != n:
        raise ValueError("codes and lengths differ in length")
    if not isinstance(lens, torch.Tensor):
        if lens.min() < 1 or lens.max() > 8:
            raise ValueError("code lengths must be 1..8 bytes")
    lib = _lib.load()
    dc = to_dev_u64(codes)
    dl = to_dev_u8(lens)
    K = ctypes.c_int32(0)
    lr = (ctypes.c_int64 * _lib.MAX_LEVELS)()
    _lib.check(lib.bsb_vbs_plan(dc.data_ptr(), dl.data_ptr(), n, ctypes.byref(K), lr,
                                stream()), "build_vbs")
    K = int(K.value)
    stride = int(lib.bsb_stride_for(n))
    nbpad = stride // 32
    dev = device()
    level_rows = [int(x) for x in lr[:K]]
    modes = {"packed": _lib.DEEP_PACKED, "sliced": _lib.DEEP_SLICED}
    if deep_mode == "auto":
        mode = choose_deep_mode(level_rows, K)
    elif deep_mode in modes:
        mode = modes[deep_mode] if K >= 2 else _lib.DEEP_PACKED
    else:
        raise ValueError(f"unknown deep_mode {deep_mode!r}")
    bs1 = torch.empty(stride, dtype=torch.uint8, device=dev)
    deep, exist, bdir, rex = [None], [None], [None], [None]
    cnt2 = level_rows[1] if K >= 2 else 0
    d1 = (1, 0)
    if mode == _lib.DEEP_SLICED and cnt2 > 0:
        # zone map of the deep rows' first byte: when they all share it the
        # deep-space scan settles their level 1 without reading any bytes
        lt = dl.to(torch.int64)
        first = ((dc >> (8 * (lt - 1))) & 0xFF)[lt >= 2]
        d1 = (int(first.min().item()), int(first.max().item()))
        del lt, first
    if mode == _lib.DEEP_SLICED and d1[0] != d1[1]:
        # level 1 of the deep rows in deep-row space (deep-space scan kernel)
        deep[0] = torch.zeros(-(-cnt2 // 32) * 32 + DEEP_PAD, dtype=torch.uint8, device=dev)
    for j in range(1, K):
        if mode == _lib.DEEP_SLICED:
            # byte j+1 of every deep row, swizzled 32-deep-row blocks
            deep.append(torch.zeros(-(-cnt2 // 32) * 32 + DEEP_PAD, dtype=torch.uint8,
                                    device=dev))
            rex.append(torch.zeros(cnt2 // 32 + 2, dtype=torch.int32, device=dev)
                       if j >= 2 else None)
        else:
            deep.append(torch.empty(level_rows[j] + DEEP_PAD, dtype=torch.uint8, device=dev))
            rex.append(None)
        exist.append(torch.empty(nbpad, dtype=torch.int32, device=dev))
        need_dir = mode == _lib.DEEP_PACKED or j == 1
        bdir.append(torch.empty(nbpad + 1, dtype=torch.int64, device=dev) if need_dir else None)
    col = VbsColumn(n, K, lanes, stride, bs1, deep, exist, bdir, level_rows, mode, rex, d1)
    _lib.check(lib.bsb_vbs_build(dc.data_ptr(), dl.data_ptr(), col.desc_ref, stream()),
               "build_vbs")
    return col


def _mask_bytes(col: VbsColumn, live: int, length: int) -> int:
    """vbs.py:286-287: existence words charged per live block."""
    return live * 4 * (min(length + 1, col.max_len) - 1)


def _scan_stats(col: VbsColumn, pred: ResolvedPredicate, mask,
                with_depth: bool = True) -> ScanStats:
    lib = _lib.load()
    nb = col.n_blocks
    dev = col.bs1.device
    st = torch.zeros(_lib.STATS_WORDS, dtype=torch.int64, device=dev)
    depth = torch.zeros(max(nb, 1), dtype=torch.int8, device=dev) if with_depth else None
    out = torch.empty(nb, dtype=torch.int32, device=dev)
    cnt = torch.empty(1, dtype=torch.int64, device=dev)
    cp = pred.to_c()
    _lib.check(lib.bsb_vbs_scan(col.desc_ref, ctypes.byref(cp),
                                None if mask is None else mask.dwords.data_ptr(),
                                out.data_ptr(), cnt.data_ptr(), st.data_ptr(), _lib.ptr(depth),
                                stream()), "scan_vbs(stats)")
    h = st.cpu().numpy()
    K = col.max_len
    if pred.is_trivial:
        skipped, mb = nb, 0
    elif pred.op is Op.BETWEEN:
        s1, s2 = int(h[17]), int(h[19])
        skipped = min(s1, s2)
        mb = _mask_bytes(col, nb - s1, pred.length) + _mask_bytes(col, nb - s2, pred.length2)
    else:
        skipped = int(h[17])
        mb = _mask_bytes(col, nb - skipped, pred.length)
    return ScanStats(levels=K, blocks_total=nb, blocks_skipped=skipped,
                     words_loaded=h[0:K].copy(), bytes_loaded=h[8:8 + K].copy(),
                     mask_bytes=mb,
                     block_depth=None if depth is None else depth[:nb].cpu().numpy())


def scan_vbs(col: VbsColumn, pred: ResolvedPredicate, mask=None, threads: int = 1):
    """vbs.py:292-324: Alg. 3 on the device.  Returns (DeviceBitVector, ScanStats).

    A literal longer than the column's longest code raises ValueError (the
    reference fails with IndexError at vbs.py:274).  ``threads`` is ignored.
    """
    m = None
    if mask is not None:
        m = as_device_bits(mask)
        if m.n_rows != col.n_rows:
            raise ValueError("input mask length mismatch")
    lib = _lib.load()
    out = torch.empty(col.n_blocks, dtype=torch.int32, device=col.bs1.device)
    cnt = torch.empty(1, dtype=torch.int64, device=col.bs1.device)
    cp = pred.to_c()
    _lib.check(lib.bsb_vbs_scan(col.desc_ref, ctypes.byref(cp),
                                None if m is None else m.dwords.data_ptr(), out.data_ptr(),
                                cnt.data_ptr(), None, None, stream()), "scan_vbs")
    return DeviceBitVector(col.n_rows, out, cnt), LazyScanStats(
        lambda with_depth: _scan_stats(col, pred, m, with_depth))


def _vbs_order(col: VbsColumn, order: str) -> str:
    if order == "auto":
        return "sort" if col.max_len >= 3 else "keep"
    return order


def lookup_vbs_rows(col: VbsColumn, rows, sorted_padded=None, dict_values=None,
                    out_dtype=torch.int64, level_counts=None, order: str = "auto", err=None):
    """Device lookup of a row-id list (any order, output in input order):
    padded codes, or decoded values when the dictionary's sorted padded codes
    / values are given.  order: see lookup_byteslice_rows (a deep row costs up
    to ~2K random sectors: bs1, existence words, directory, deep bytes, so
    locality matters more here); with a binary-search dictionary or
    level_counts the long unsorted lists take the sort + scatter-back path.
    Ids outside [0, n_rows) raise IndexError; `err` as in
    lookup_byteslice_rows."""
    lib = _lib.load()
    rows = to_dev_i64(rows)
    n = rows.numel()
    lc = None if level_counts is None else level_counts.data_ptr()
    if sorted_padded is None:
        out = torch.empty(n, dtype=torch.int64, device=rows.device)
        if lc is None and order != "sort" and (order == "bucket" or (
                order == "auto" and auto_gather(n, col.n_rows))):
            fn, g, _ = row_gather_plan(rows, col.n_rows, order, lib.bsb_vbs_lookup_rows_dec_auto,
                                       lib.bsb_vbs_lookup_pairs_dec, lib.bsb_vbs_lookup_rows_dec)
            _lib.check(fn(col.desc_ref, g.data_ptr(), n, None, out.data_ptr(), None, None,
                          _lib.ptr(err), stream()), "lookup_vbs")
            return out
        g, perm = gather_order(rows, col.n_rows, _vbs_order(col, order) if order in
                               ("auto", "sort") else "keep")
        _lib.check(lib.bsb_vbs_lookup_rows(col.desc_ref, g.data_ptr(), n, out.data_ptr(),
                                           None, None, 0, None, None, lc, _lib.ptr(err), stream()),
                   "lookup_vbs")
        return scatter_back(out, perm)
    g, perm = gather_order(rows, col.n_rows, _vbs_order(col, order) if order in
                           ("auto", "sort") else "keep")
    out = torch.empty(n, dtype=out_dtype, device=rows.device)
    p64 = out.data_ptr() if out_dtype == torch.int64 else None
    p32 = out.data_ptr() if out_dtype == torch.int32 else None
    _lib.check(lib.bsb_vbs_lookup_rows(col.desc_ref, g.data_ptr(), n, None,
                                       sorted_padded.data_ptr(), dict_values.data_ptr(),
                                       sorted_padded.numel(), p64, p32, lc, _lib.ptr(err), stream()),
               "lookup_vbs")
    return scatter_back(out, perm)


def lookup_vbs_rows_dec(col: VbsColumn, rows, decoder, out_dtype=torch.int64,
                        order: str = "auto", err=None):
    """Row-id lookup decoded through a C-ABI decoder (Dictionary.dev_decoder).
    order / err: see lookup_vbs_rows."""
    lib = _lib.load()
    rows = to_dev_i64(rows)
    n = rows.numel()
    fn, g, perm = row_gather_plan(rows, col.n_rows, order, lib.bsb_vbs_lookup_rows_dec_auto,
                                  lib.bsb_vbs_lookup_pairs_dec, lib.bsb_vbs_lookup_rows_dec)
    out = torch.empty(n, dtype=out_dtype, device=rows.device)
    p64 = out.data_ptr() if out_dtype == torch.int64 else None
    p32 = out.data_ptr() if out_dtype == torch.int32 else None
    _lib.check(fn(col.desc_ref, g.data_ptr(), n, ctypes.byref(decoder), None, p64, p32,
                  _lib.ptr(err), stream()), "lookup_vbs")
    return scatter_back(out, perm)


def lookup_vbs_bits(col: VbsColumn, selection, decoder=None, out_dtype=torch.int64):
    """Fused selection -> values (or padded codes without a decoder), in
    ascending row order; no row-id array is materialised."""
    sel = as_device_bits(selection)
    if sel.n_rows != col.n_rows:
        raise ValueError("selection length mismatch")
    n = sel.count()
    dev = col.bs1.device
    cnt = torch.empty(1, dtype=torch.int64, device=dev)
    lib = _lib.load()
    if decoder is None:
        out = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        _lib.check(lib.bsb_vbs_lookup_bits(col.desc_ref, sel.dwords.data_ptr(), None,
                                           out.data_ptr(), None, None, cnt.data_ptr(),
                                           stream()), "lookup_vbs")
        return out[:n]
    out = torch.empty(max(n, 1), dtype=out_dtype, device=dev)
    p64 = out.data_ptr() if out_dtype == torch.int64 else None
    p32 = out.data_ptr() if out_dtype == torch.int32 else None
    _lib.check(lib.bsb_vbs_lookup_bits(col.desc_ref, sel.dwords.data_ptr(),
                                       ctypes.byref(decoder), None, p64, p32, cnt.data_ptr(),
                                       stream()), "lookup_vbs")
    _check_count(cnt, "lookup_vbs")
    return out[:n]


def _check_count(cnt: torch.Tensor, where: str):
    """UINT64_MAX in the async count = a code not in the dictionary."""
    if int(cnt.item()) == -1:
        raise LookupError(f"{where}: padded code not in dictionary")


def lookup_vbs(col: VbsColumn, selection):
    """vbs.py:331-371: padded codes of the selected rows, ascending row order."""
    if selection.n_rows != col.n_rows:
        raise ValueError("selection length mismatch")
    sel = as_device_bits(selection)
    rows = sel.row_ids()
    n = rows.numel()
    if n == 0:
        return np.zeros(0, np.uint64), LookupStats()
    lc = torch.zeros(_lib.MAX_LEVELS, dtype=torch.int64, device=rows.device)
    codes = lookup_vbs_rows(col, rows, level_counts=lc)
    counts = lc.cpu().numpy()
    levels = int(np.flatnonzero(counts)[-1]) + 1
    nz_words = int((sel.dwords != 0).sum().item())
    st = LookupStats(levels_touched=levels, bytes_loaded=int(counts.sum()),
                     mask_bytes=nz_words * (col.max_len - 1) * 4)
    return host_u64(codes), st


def scan_serial(col: VbsColumn, pred: ResolvedPredicate, mask=None):
    """vbs.py:378-462, the reference's block-at-a-time scan.  Its results and
    stats equal scan_vbs's by contract (tests/test_vbs.py:198-209); on the
    device both are the same Alg. 3 kernels, here with the ScanStats
    materialised eagerly as the serial form returns them."""
    bv, st = scan_vbs(col, pred, mask)
    return bv, st.materialize()


def lookup_serial(col: VbsColumn, selection) -> np.ndarray:
    """vbs.py:465-498 (Alg. 4): padded codes of the selected rows in
    ascending row order, as uint64.  Same errors as the reference: a
    selection of another length is ValueError; lanes other than 32 cannot
    reach the device path (LaneConfig.require_device)."""
    if selection.n_rows != col.n_rows:
        raise ValueError("selection length mismatch")
    if col.lanes.lane_count != 32:
        raise NotImplementedError("reference lookup assumes 32-code blocks")
    codes, _ = lookup_vbs(col, selection)
    return codes


def vbs_size_report(col: VbsColumn) -> dict:
    """vbs.py:505-517."""
    sb = [col.slice_len(j) for j in range(1, col.max_len + 1)]
    mb = ((col.n_rows + 7) // 8) * (col.max_len - 1)
    db = col.n_blocks * (col.max_len - 1) * 4
    data = sum(sb) + mb
    return {"slice_bytes": sb, "mask_bytes": mb, "directory_bytes": db,
            "total_bytes": data + db, "avg_bits_per_code": 8.0 * data / col.n_rows}
