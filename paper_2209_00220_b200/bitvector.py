"""Result bitvectors (mirror of reference bitvector.py:19-125).

``ResultBitVector`` is the host type with the reference's exact API and
layout (uint32 words, LSB first, tail bits zero).  Scans return
``DeviceBitVector``: the same API over device-resident words, with
combinators and popcount running as CUDA kernels and host copies made only
when host data is asked for (``words``, ``to_bools``...).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .device import device, host_u32, stream, to_dev_u32

__all__ = ["ResultBitVector", "DeviceBitVector", "bitvector_and", "bitvector_or",
           "popcount_vector", "as_device_bits"]


def _n_words(n_rows: int) -> int:
    return (n_rows + 31) // 32


class ResultBitVector:
    """Fixed-length host bit sequence over the rows of one column."""

    __slots__ = ("n_rows", "words")

    def __init__(self, n_rows: int, words):
        if n_rows < 0:
            raise ValueError("n_rows must be nonnegative")
        # copy: the reference clears the tail of an aliased caller array in
        # place (bitvector.py:27-37); we never mutate caller memory
        w = np.array(words, dtype=np.uint32, copy=True).reshape(-1)
        if w.shape != (_n_words(n_rows),):
            raise ValueError("word count does not match row count")
        if n_rows % 32 and len(w):
            w[-1] &= np.uint32((1 << (n_rows % 32)) - 1)
        self.n_rows = n_rows
        self.words = w

    @classmethod
    def zeros(cls, n_rows: int) -> "ResultBitVector":
        return cls(n_rows, np.zeros(_n_words(n_rows), np.uint32))

    @classmethod
    def ones(cls, n_rows: int) -> "ResultBitVector":
        return cls(n_rows, np.full(_n_words(n_rows), 0xFFFFFFFF, np.uint32))

    @classmethod
    def from_bools(cls, flags) -> "ResultBitVector":
        f = np.asarray(flags, dtype=bool)
        buf = np.zeros(_n_words(len(f)) * 4, np.uint8)
        p = np.packbits(f, bitorder="little")
        buf[: len(p)] = p
        return cls(len(f), buf.view(np.uint32))

    @classmethod
    def from_indices(cls, n_rows: int, indices) -> "ResultBitVector":
        f = np.zeros(n_rows, bool)
        f[np.asarray(indices, dtype=np.int64)] = True
        return cls.from_bools(f)

    def to_bools(self) -> np.ndarray:
        return np.unpackbits(self.words.view(np.uint8), bitorder="little")[: self.n_rows] \
            .astype(bool)

    def to_indices(self) -> np.ndarray:
        return np.flatnonzero(self.to_bools()).astype(np.int64)

    def count(self) -> int:
        return int(np.bitwise_count(self.words).sum())

    def get(self, i: int) -> bool:
        if not 0 <= i < self.n_rows:
            raise IndexError(i)
        return bool((int(self.words[i >> 5]) >> (i & 31)) & 1)

    def _check(self, other):
        if self.n_rows != other.n_rows:
            raise ValueError("bitvector lengths differ")

    def __and__(self, other):
        self._check(other)
        return ResultBitVector(self.n_rows, self.words & _host_words(other))

    def __or__(self, other):
        self._check(other)
        return ResultBitVector(self.n_rows, self.words | _host_words(other))

    def __invert__(self):
        return ResultBitVector(self.n_rows, ~self.words)

    def __eq__(self, other):
        if not isinstance(other, (ResultBitVector, DeviceBitVector)):
            return NotImplemented
        return self.n_rows == other.n_rows and bool(
            np.array_equal(self.words, _host_words(other)))

    def __hash__(self):
        raise TypeError("ResultBitVector is mutable, not hashable")

    def __len__(self):
        return self.n_rows

    def to_device(self) -> "DeviceBitVector":
        return DeviceBitVector(self.n_rows, to_dev_u32(self.words))

    def __repr__(self):
        return f"ResultBitVector(n_rows={self.n_rows}, set={self.count()})"


def _host_words(bv) -> np.ndarray:
    return bv.words if isinstance(bv, ResultBitVector) else bv.host().words


class DeviceBitVector:
    """Device-resident result bitvector (same API as ResultBitVector).

    ``dwords`` is an int32 CUDA tensor holding the uint32 words bit for bit.
    ``_count`` optionally caches a device uint64 popcount produced by a scan.
    """

    __slots__ = ("n_rows", "dwords", "_count", "_host")

    def __init__(self, n_rows: int, dwords: torch.Tensor, count_dev: torch.Tensor | None = None):
        if dwords.numel() != _n_words(n_rows):
            raise ValueError("word count does not match row count")
        self.n_rows = n_rows
        self.dwords = dwords
        self._count = count_dev
        self._host = None

    @classmethod
    def empty(cls, n_rows: int) -> "DeviceBitVector":
        return cls(n_rows, torch.empty(_n_words(n_rows), dtype=torch.int32, device=device()))

    @classmethod
    def zeros(cls, n_rows: int) -> "DeviceBitVector":
        return cls(n_rows, torch.zeros(_n_words(n_rows), dtype=torch.int32, device=device()))

    @classmethod
    def ones(cls, n_rows: int) -> "DeviceBitVector":
        z = cls.zeros(n_rows)
        return ~z

    def host(self) -> ResultBitVector:
        if self._host is None:
            self._host = ResultBitVector(self.n_rows, host_u32(self.dwords))
        return self._host

    to_host = host

    @property
    def words(self) -> np.ndarray:
        return self.host().words

    def count_device(self) -> torch.Tensor:
        """uint64 popcount as a 1-element device tensor (no host sync)."""
        if self._count is None:
            c = torch.empty(1, dtype=torch.int64, device=self.dwords.device)
            _lib.check(_lib.load().bsb_bits_popcount(self.dwords.data_ptr(), self.n_rows,
                                                     c.data_ptr(), stream()), "popcount")
            self._count = c
        return self._count

    def count(self) -> int:
        return int(self.count_device().item())

    def to_bools(self) -> np.ndarray:
        return self.host().to_bools()

    def to_indices(self) -> np.ndarray:
        return self.row_ids().cpu().numpy()

    def row_ids(self, row_offset: int = 0) -> torch.Tensor:
        """Ascending int64 row ids on the device (bitvector.py:71-72)."""
        lib = _lib.load()
        n = self.count()
        out = torch.empty(max(n, 1), dtype=torch.int64, device=self.dwords.device)
        if n:
            cnt = torch.empty(1, dtype=torch.int64, device=self.dwords.device)
            _lib.check(lib.bsb_bits_to_rows_async(self.dwords.data_ptr(), self.n_rows,
                                                  int(row_offset), out.data_ptr(),
                                                  cnt.data_ptr(), stream()), "to_indices")
        return out[:n]

    def get(self, i: int) -> bool:
        if not 0 <= i < self.n_rows:
            raise IndexError(i)
        return bool((int(self.dwords[i >> 5].item()) >> (i & 31)) & 1)

    def _combine(self, op: int, other):
        if other is not None:
            if self.n_rows != other.n_rows:
                raise ValueError("bitvector lengths differ")
            o = as_device_bits(other).dwords
        else:
            o = None
        out = torch.empty_like(self.dwords)
        _lib.check(_lib.load().bsb_bits_combine(op, self.dwords.data_ptr(),
                                                None if o is None else o.data_ptr(),
                                                out.data_ptr(), self.n_rows, stream()),
                   "bitvector op")
        return DeviceBitVector(self.n_rows, out)

    def __and__(self, other):
        return self._combine(0, other)

    def __or__(self, other):
        return self._combine(1, other)

    def __invert__(self):
        return self._combine(2, None)

    def andnot(self, other):
        return self._combine(3, other)

    def __eq__(self, other):
        if isinstance(other, DeviceBitVector):
            return self.n_rows == other.n_rows and bool(torch.equal(self.dwords, other.dwords))
        if isinstance(other, ResultBitVector):
            return other == self
        return NotImplemented

    def __hash__(self):
        raise TypeError("bitvectors are mutable, not hashable")

    def __len__(self):
        return self.n_rows

    def __repr__(self):
        return f"DeviceBitVector(n_rows={self.n_rows}, set={self.count()})"


def as_device_bits(bv) -> DeviceBitVector:
    if isinstance(bv, DeviceBitVector):
        return bv
    if isinstance(bv, ResultBitVector):
        return bv.to_device()
    raise TypeError(f"expected a bitvector, got {type(bv).__name__}")


def bitvector_and(a, b):
    return a & b


def bitvector_or(a, b):
    return a | b


def popcount_vector(v) -> int:
    return v.count()
