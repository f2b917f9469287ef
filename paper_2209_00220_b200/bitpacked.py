"""Bit-Packed baseline layout on the device (mirror of reference bitpacked.py).

Code i occupies stream bits [i*w, (i+1)*w), most significant bit first
(bitpacked.py:1-6).  The device buffer's bytes are the reference stream
(`bits`), padded to whole 32-row groups.  Scans unpack and compare every
code -- no early stop and no ScanStats, exactly like the reference.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .bitvector import DeviceBitVector, as_device_bits
from .device import device, host_u64, stream, to_dev_i64
from .predicate import ResolvedPredicate

__all__ = ["BitPackedColumn", "build_bitpacked", "scan_bitpacked", "lookup_bitpacked",
           "lookup_bitpacked_bits", "byte_span", "bitpacked_size_report"]


@dataclass
class BitPackedColumn:
    n_rows: int
    w: int
    words: torch.Tensor          # int32 view of the padded stream
    _desc: _lib.BsbBitPacked = field(default=None, repr=False)

    def __post_init__(self):
        d = _lib.BsbBitPacked()
        d.n_rows, d.width_bits, d.words = self.n_rows, self.w, self.words.data_ptr()
        self._desc = d

    @property
    def desc_ref(self):
        return ctypes.byref(self._desc)

    @property
    def total_bits(self) -> int:
        return self.n_rows * self.w

    @property
    def bits(self) -> np.ndarray:
        """The reference packed stream (uint8, ceil(n*w/8) bytes)."""
        raw = self.words.cpu().numpy().view(np.uint8)
        return raw[: (self.n_rows * self.w + 7) // 8].copy()


def build_bitpacked(codes, w: int) -> BitPackedColumn:
    """bitpacked.py:36-52."""
    if not 1 <= int(w) <= 32:
        raise ValueError("width must be 1..32 bits")
    c = to_dev_i64(codes if isinstance(codes, torch.Tensor) else
                   np.asarray(codes, dtype=np.uint64).astype(np.int64))
    n = c.numel()
    if n == 0:
        raise ValueError("empty column")
    lib = _lib.load()
    words = torch.empty(int(lib.bsb_bitpacked_words_for(n, int(w))), dtype=torch.int32,
                        device=device())
    _lib.check(lib.bsb_bitpacked_build(c.data_ptr(), n, int(w), words.data_ptr(), stream()),
               "build_bitpacked")
    return BitPackedColumn(n, int(w), words)


def scan_bitpacked(col: BitPackedColumn, pred: ResolvedPredicate, mask=None,
                   threads: int = 1) -> DeviceBitVector:
    """bitpacked.py:94-118: every code unpacked and compared; mask post-AND."""
    m = None
    if mask is not None:
        m = as_device_bits(mask)
        if m.n_rows != col.n_rows:
            raise ValueError("input mask length mismatch")
    nb = -(-col.n_rows // 32)
    out = torch.empty(nb, dtype=torch.int32, device=col.words.device)
    cnt = torch.empty(1, dtype=torch.int64, device=col.words.device)
    cp = pred.to_c()
    _lib.check(_lib.load().bsb_bitpacked_scan(col.desc_ref, ctypes.byref(cp),
                                              None if m is None else m.dwords.data_ptr(),
                                              out.data_ptr(), cnt.data_ptr(), stream()),
               "scan_bitpacked")
    return DeviceBitVector(col.n_rows, out, cnt)


def lookup_bitpacked_bits(col: BitPackedColumn, selection, decoder=None,
                          out_dtype=torch.int64) -> torch.Tensor:
    """Selected rows (ascending) -> codes, or values through a rank decoder."""
    sel = as_device_bits(selection)
    if sel.n_rows != col.n_rows:
        raise ValueError("selection length mismatch")
    n = sel.count()
    dev = col.words.device
    out = torch.empty(max(n, 1), dtype=torch.int64 if decoder is None else out_dtype,
                      device=dev)
    p64 = out.data_ptr() if (decoder is not None and out_dtype == torch.int64) else None
    p32 = out.data_ptr() if (decoder is not None and out_dtype == torch.int32) else None
    _lib.check(_lib.load().bsb_bitpacked_lookup_bits(
        col.desc_ref, sel.dwords.data_ptr(), None if decoder is None else ctypes.byref(decoder),
        out.data_ptr() if decoder is None else None, p64, p32, None, stream()),
        "lookup_bitpacked")
    return out[:n]


def lookup_bitpacked(col: BitPackedColumn, selection) -> np.ndarray:
    """bitpacked.py:127-143: codes of the selected rows, ascending row order."""
    if selection.n_rows != col.n_rows:
        raise ValueError("selection length mismatch")
    return host_u64(lookup_bitpacked_bits(col, selection))


def byte_span(col: BitPackedColumn, row: int) -> tuple[int, int]:
    """bitpacked.py:121-124."""
    start = row * col.w
    return start >> 3, (start + col.w - 1) >> 3


def bitpacked_size_report(col: BitPackedColumn) -> dict:
    return {"total_bytes": (col.n_rows * col.w + 7) // 8, "avg_bits_per_code": col.w}
