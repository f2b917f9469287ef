"""VBP / PE-VBP baseline layouts on the device (mirror of reference vbp.py).

Plane j holds the j-th most significant bit of every code, one uint32 per
32-row block (vbp.py:31-37); scans walk planes top down per block with the
reference's greater / still-equal masks and stop when nothing is still equal.
The padded-encoding variant stores prefix-free codes zero-padded to w_max
bits (vbp.py:40-48).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .bitvector import DeviceBitVector, as_device_bits
from .device import device, host_u64, stream, to_dev_u64
from .predicate import Op, ResolvedPredicate
from .stats import LazyScanStats, LookupStats, ScanStats

__all__ = ["VbpColumn", "build_vbp", "pad_codes", "scan_vbp", "lookup_vbp", "lookup_vbp_bits",
           "vbp_size_report"]

_KINDS = {"plain": _lib.VBP_PLAIN, "padded_encoding": _lib.VBP_PADDED}


@dataclass
class VbpColumn:
    n_rows: int
    w_max: int
    kind: str                    # "plain" | "padded_encoding"
    dplanes: torch.Tensor        # int32 [w_max * n_words]
    _desc: _lib.BsbVbp = field(default=None, repr=False)

    def __post_init__(self):
        d = _lib.BsbVbp()
        d.n_rows, d.w_max, d.kind = self.n_rows, self.w_max, _KINDS[self.kind]
        d.planes = self.dplanes.data_ptr()
        self._desc = d

    @property
    def desc_ref(self):
        return ctypes.byref(self._desc)

    @property
    def n_words(self) -> int:
        return -(-self.n_rows // 32)

    @property
    def planes(self) -> np.ndarray:
        """Reference planes (w_max, n_words) uint32, host copy."""
        return self.dplanes.cpu().numpy().view(np.uint32).reshape(self.w_max, self.n_words)


def pad_codes(codes, lengths, w_max: int) -> np.ndarray:
    """vbp.py:40-46: zero-pad variable bit-length codes up to w_max bits."""
    arr = np.ascontiguousarray(codes, dtype=np.uint64)
    lens = np.ascontiguousarray(lengths, dtype=np.uint64)
    if lens.max(initial=0) > w_max:
        raise ValueError("code longer than padded width")
    return arr << (np.uint64(w_max) - lens)


def build_vbp(codes, w_max: int, kind: str = "plain") -> VbpColumn:
    """vbp.py:49-68."""
    if kind not in _KINDS:
        raise ValueError(f"unknown vbp kind {kind!r}")
    if not 1 <= int(w_max) <= 32:
        raise ValueError("plane count must be 1..32")
    c = to_dev_u64(codes)
    n = c.numel()
    if n == 0:
        raise ValueError("empty column")
    nw = -(-n // 32)
    planes = torch.empty(int(w_max) * nw, dtype=torch.int32, device=device())
    _lib.check(_lib.load().bsb_vbp_build(c.data_ptr(), n, int(w_max), planes.data_ptr(),
                                         stream()), "build_vbp")
    return VbpColumn(n, int(w_max), kind, planes)


def _scan(col: VbpColumn, pred: ResolvedPredicate, m, stats: bool):
    lib = _lib.load()
    dev = col.dplanes.device
    out = torch.empty(col.n_words, dtype=torch.int32, device=dev)
    cnt = torch.empty(1, dtype=torch.int64, device=dev)
    st = torch.zeros(_lib.VBP_STATS_WORDS, dtype=torch.int64, device=dev) if stats else None
    depth = torch.zeros(max(col.n_words, 1), dtype=torch.int8, device=dev) if stats else None
    cp = pred.to_c()
    _lib.check(lib.bsb_vbp_scan(col.desc_ref, ctypes.byref(cp),
                                None if m is None else m.dwords.data_ptr(), out.data_ptr(),
                                cnt.data_ptr(), None if st is None else st.data_ptr(),
                                None if depth is None else depth.data_ptr(), stream()),
               "scan_vbp")
    return DeviceBitVector(col.n_rows, out, cnt), st, depth


def _stats(col: VbpColumn, pred: ResolvedPredicate, m) -> ScanStats:
    _, st, depth = _scan(col, pred, m, True)
    h = st.cpu().numpy()
    L = col.w_max
    skipped = int(h[64])
    if pred.op is Op.BETWEEN and not pred.is_trivial:
        skipped = min(skipped, int(h[65]))
    words = h[:L].copy()
    return ScanStats(levels=L, blocks_total=col.n_words, blocks_skipped=skipped,
                     words_loaded=words, bytes_loaded=4 * words, mask_bytes=0,
                     block_depth=depth[: col.n_words].cpu().numpy())


def scan_vbp(col: VbpColumn, pred: ResolvedPredicate, mask=None, threads: int = 1):
    """vbp.py:144-194: (DeviceBitVector, ScanStats) -- stats materialised on
    first access through the stats kernel variant."""
    m = None
    if mask is not None:
        m = as_device_bits(mask)
        if m.n_rows != col.n_rows:
            raise ValueError("input mask length mismatch")
    bv, _, _ = _scan(col, pred, m, False)
    return bv, LazyScanStats(lambda with_depth: _stats(col, pred, m))


def lookup_vbp_bits(col: VbpColumn, selection, decoder=None,
                    out_dtype=torch.int64) -> torch.Tensor:
    sel = as_device_bits(selection)
    if sel.n_rows != col.n_rows:
        raise ValueError("selection length mismatch")
    n = sel.count()
    out = torch.empty(max(n, 1), dtype=torch.int64 if decoder is None else out_dtype,
                      device=col.dplanes.device)
    p64 = out.data_ptr() if (decoder is not None and out_dtype == torch.int64) else None
    p32 = out.data_ptr() if (decoder is not None and out_dtype == torch.int32) else None
    _lib.check(_lib.load().bsb_vbp_lookup_bits(
        col.desc_ref, sel.dwords.data_ptr(), None if decoder is None else ctypes.byref(decoder),
        out.data_ptr() if decoder is None else None, p64, p32, None, stream()), "lookup_vbp")
    return out[:n]


def lookup_vbp(col: VbpColumn, selection):
    """vbp.py:197-212: padded codes of the selected rows + LookupStats."""
    if selection.n_rows != col.n_rows:
        raise ValueError("selection length mismatch")
    codes = host_u64(lookup_vbp_bits(col, selection))
    st = LookupStats()
    if len(codes):
        st.levels_touched = col.w_max
        st.bytes_loaded = len(codes) * col.w_max * 4
    return codes, st


def vbp_size_report(col: VbpColumn) -> dict:
    data = col.w_max * col.n_words * 4
    return {"total_bytes": data, "avg_bits_per_code": 8.0 * data / col.n_rows}
