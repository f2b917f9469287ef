"""Dictionary encoders (mirror of reference dictionary.py).

Numeric columns: the frequency table + row ranks come from one radix sort on
the GPU (bsb_freq_table); encode_rows is a device binary search; row codes
are a device gather.  Host work (O(distinct)): ppe_numerical in C++
(bsb_ppe_numerical_host), literal resolution (scalar searchsorted) and the
decode tables handed to the lookup kernels.

Categorical and ordered-string columns: strings do
not live on the device, so their frequency tables, ranks and ppe_categorical
codes (Alg. 2) are built on the host exactly as the reference does; the
codes then go through the same device layouts, scans and lookups, and
looked-up ranks are mapped back to strings on the host.  Prefix-free
(PE-VBP) codes stay outside the device path and raise ValueError.
"""

from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass
from functools import cached_property

import numpy as np
import torch

from . import _lib
from .device import device, stream, to_dev_i64
from .predicate import Op, Predicate, ResolvedPredicate

__all__ = ["ColumnKind", "FrequencyTable", "build_frequency_table", "CodeAssignment",
           "ppe_numerical", "ppe_categorical", "fixed_assignment", "prefix_free_assignment",
           "Dictionary",
           "compare_codes", "freq_table_and_ranks"]

MAX_CODE_BYTES = 8
MAX_FIXED_BITS = 32


class ColumnKind(enum.Enum):
    NUMERIC = "numeric"
    CATEGORICAL = "categorical"
    ORDERED_STRING = "ordered_string"

    @property
    def ordered(self) -> bool:
        return self is not ColumnKind.CATEGORICAL


def _string_array(values) -> np.ndarray:
    """dictionary.py:72-98 for the string kinds: str array, no NULL/empty."""
    arr = np.asarray(values)
    if arr.ndim != 1 or arr.size == 0:
        raise ValueError("column must be a nonempty 1-d sequence")
    if arr.dtype == object and any(v is None for v in arr):
        raise ValueError("NULL value in column")
    arr = arr.astype(str)
    if (np.char.str_len(arr) == 0).any():
        raise ValueError("NULL (empty) value in string column")
    return arr


def _host_table(arr: np.ndarray, kind: ColumnKind):
    """dictionary.py:101-109 on the host: ordered kinds ascending; categorical
    by descending count, ties by first appearance.  Also returns the rank of
    every row."""
    if kind.ordered:
        uniq, inv, counts = np.unique(arr, return_inverse=True, return_counts=True)
        return uniq, counts.astype(np.int64), inv.astype(np.int64)
    uniq, first, inv, counts = np.unique(arr, return_index=True, return_inverse=True,
                                         return_counts=True)
    order = np.lexsort((first, -counts))
    rank_of = np.empty(len(order), np.int64)
    rank_of[order] = np.arange(len(order))
    return uniq[order], counts[order].astype(np.int64), rank_of[inv]


@dataclass(frozen=True)
class FrequencyTable:
    """Distinct values (ascending) and their counts (dictionary.py:57-82)."""

    values: np.ndarray
    weights: np.ndarray
    kind: ColumnKind

    def __post_init__(self):
        if len(self.values) == 0:
            raise ValueError("empty column")
        if len(self.values) != len(self.weights):
            raise ValueError("values and weights differ in length")

    @property
    def n(self) -> int:
        return len(self.values)


def _values_tensor(values) -> torch.Tensor:
    if isinstance(values, torch.Tensor):
        if values.dtype.is_floating_point or values.dtype == torch.bool:
            raise ValueError("numeric column holds a non-integer")
        if values.ndim != 1 or values.numel() == 0:
            raise ValueError("column must be a nonempty 1-d sequence")
        return to_dev_i64(values)
    arr = np.asarray(values)
    if arr.ndim != 1 or arr.size == 0:
        raise ValueError("column must be a nonempty 1-d sequence")
    if arr.dtype.kind not in "iu":
        if arr.dtype == object and all(isinstance(v, (int, np.integer)) and
                                       not isinstance(v, bool) for v in arr):
            arr = arr.astype(np.int64)
        else:
            raise ValueError("numeric column holds a non-integer")
    return to_dev_i64(arr.astype(np.int64))


def freq_table_and_ranks(values):
    """Device sort -> (sorted distinct values, counts, per-row ranks) tensors.

    One pass gives build_frequency_table (dictionary.py:101-106) and
    encode_rows (dictionary.py:381-397) for the same column.
    """
    v = _values_tensor(values)
    n = v.numel()
    lib = _lib.load()
    uniq = torch.empty(n, dtype=torch.int64, device=v.device)
    cnts = torch.empty(n, dtype=torch.int64, device=v.device)
    ranks = torch.empty(n, dtype=torch.int64, device=v.device)
    D = ctypes.c_int64(0)
    _lib.check(lib.bsb_freq_table(v.data_ptr(), n, uniq.data_ptr(), cnts.data_ptr(),
                                  ranks.data_ptr(), ctypes.byref(D), stream()), "freq_table")
    D = int(D.value)
    return uniq[:D], cnts[:D], ranks


def build_frequency_table(values, kind: ColumnKind) -> FrequencyTable:
    """dictionary.py:101-109: numeric columns by a device radix sort, string
    kinds on the host."""
    if kind is not ColumnKind.NUMERIC:
        u, c, _ = _host_table(_string_array(values), kind)
        return FrequencyTable(u, c, kind)
    u, c, _ = freq_table_and_ranks(values)
    return FrequencyTable(u.cpu().numpy(), c.cpu().numpy(), kind)


def table_and_ranks(values, kind: ColumnKind):
    """(FrequencyTable, device int64 ranks) for any kind (ingest / advisor)."""
    if kind is ColumnKind.NUMERIC:
        u, c, r = freq_table_and_ranks(values)
        return FrequencyTable(u.cpu().numpy(), c.cpu().numpy(), kind), r
    u, c, r = _host_table(_string_array(values), kind)
    return FrequencyTable(u, c, kind), to_dev_i64(r)


@dataclass(frozen=True)
class CodeAssignment:
    """dictionary.py:115-140."""

    codes: np.ndarray
    lengths: np.ndarray
    scheme: str
    width_bits: int = 0

    @property
    def n(self) -> int:
        return len(self.codes)

    @property
    def max_len(self) -> int:
        return int(self.lengths.max())

    @property
    def bit_granular(self) -> bool:
        return self.scheme == "prefix_free"


def ppe_numerical(weights) -> CodeAssignment:
    """Alg. 1 (dictionary.py:148-196), native host implementation."""
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.int64))
    n = len(w)
    if n == 0:
        raise ValueError("empty weight table")
    if (w < 0).any():
        raise ValueError("negative weight")
    codes = np.zeros(n, np.uint64)
    lens = np.zeros(n, np.uint8)
    _lib.check(_lib.load().bsb_ppe_numerical_host(w.ctypes.data, n, codes.ctypes.data,
                                                  lens.ctypes.data), "ppe_numerical")
    return CodeAssignment(codes, lens, "ppe_numerical")


def ppe_categorical(n: int) -> CodeAssignment:
    """Alg. 2 (dictionary.py:199-230): byte codes for n values ranked by
    descending weight.  With depth B = ceil(log256(n+1)), depths 1..B-1 are
    filled densely (255 slots under each of 256^(b-1) nodes, code = node << 8 |
    slot); the remaining values are dealt round-robin over the 256^(B-1)
    last-level nodes, slot by slot."""
    if n <= 0:
        raise ValueError("need at least one value")
    depth, cap = 1, 255
    while cap < n:  # smallest B with 256^B - 1 >= n
        depth += 1
        cap = (1 << (8 * depth)) - 1
    codes, lens = [], []
    placed = 0
    for b in range(1, depth):
        m = 255 * (1 << (8 * (b - 1)))
        i = np.arange(m, dtype=np.uint64)
        codes.append(((i // np.uint64(255)) << np.uint64(8)) + i % np.uint64(255) + np.uint64(1))
        lens.append(np.full(m, b, np.uint8))
        placed += m
    rest = n - placed
    nodes = np.uint64(1 << (8 * (depth - 1)))
    i = np.arange(rest, dtype=np.uint64)
    codes.append(((i % nodes) << np.uint64(8)) + i // nodes + np.uint64(1))
    lens.append(np.full(rest, depth, np.uint8))
    return CodeAssignment(np.concatenate(codes), np.concatenate(lens), "ppe_categorical")


def prefix_free_assignment(weights) -> CodeAssignment:
    """Order-preserving prefix-free bit codes by weighted bisection
    (dictionary.py:245-290; PE-VBP baseline layout).  A value range [s, e)
    splits at the cut k whose heavier side is lightest (the float64 prefix
    sum's midpoint, then k-1 / k+1 tried), clamped so no code exceeds
    ceil(log2 n) + 4 bits; the left part appends bit 0, the right bit 1."""
    w = np.asarray(weights, dtype=np.float64)
    n = len(w)
    if n == 0:
        raise ValueError("empty weight table")
    codes = np.zeros(n, np.uint64)
    nbits = np.zeros(n, np.uint8)
    if n == 1:
        nbits[0] = 1
        return CodeAssignment(codes, nbits, "prefix_free", width_bits=1)
    limit = (n - 1).bit_length() + 4
    pre = np.concatenate(([0.0], np.cumsum(w)))
    todo = [(0, n, 0, 0)]
    while todo:
        s, e, code, depth = todo.pop()
        if e - s == 1:
            codes[s], nbits[s] = code, depth
            continue
        reach = 1 << (limit - depth - 1)  # leaves a subtree of this depth may hold
        lo, hi = max(s + 1, e - reach), min(e - 1, s + reach)
        k = int(np.searchsorted(pre, (pre[s] + pre[e]) / 2.0, side="left"))
        k = min(max(k, lo), hi)

        def heavier(c):
            return max(pre[c] - pre[s], pre[e] - pre[c])

        best = k
        for c in (k - 1, k + 1):
            if lo <= c <= hi and heavier(c) < heavier(best):
                best = c
        todo.append((best, e, (code << 1) | 1, depth + 1))
        todo.append((s, best, code << 1, depth + 1))
    return CodeAssignment(codes, nbits, "prefix_free", width_bits=int(nbits.max()))


def fixed_assignment(n: int) -> CodeAssignment:
    """Rank codes at w = max(1, ceil(log2 n)) bits (dictionary.py:233-242)."""
    if n <= 0:
        raise ValueError("need at least one value")
    width = max(1, (n - 1).bit_length())
    if width > MAX_FIXED_BITS:
        raise ValueError("dictionary width overflow (more than 2**32 values)")
    return CodeAssignment(np.arange(n, dtype=np.uint64),
                          np.full(n, (width + 7) // 8, np.uint8), "fixed", width_bits=width)


def compare_codes(code1: int, len1: int, code2: int, len2: int):
    """Lemma 1 comparator (dictionary.py:293-309): (sign, bytes examined)."""
    m = min(len1, len2)
    for k in range(1, m + 1):
        a = (code1 >> (8 * (len1 - k))) & 0xFF
        b = (code2 >> (8 * (len2 - k))) & 0xFF
        if a != b:
            return (1 if a > b else -1), k
    if len1 == len2:
        return 0, m
    return (1 if len1 > len2 else -1), m


def ppe_decode_tree(codes, lens):
    """Two-level tables decoding ppe_numerical codes (include/bytestore_b200.h
    bsb_decode kind 3).

    ppe_numerical builds a 256-ary tree whose internal nodes sit at depth 0
    and 1 only and whose depth-2 nodes are leaves enumerating a contiguous
    rank range (dictionary.py:170-195); a node can be a code and a parent at
    once.  So, with -1 for "absent" in every field:
      e1[b1]            = child c (low 32 bits) | rank of 1-byte code b1 << 32
      e2[2*(c*256+b2)]  = rank of the 2-byte code (b1, b2)
      e2[2*(c*256+b2)+1]= leaf start | size << 32 | beta << 56: the codes of
                          length beta + 2 below (b1, b2), rank = start +
                          suffix - 1 for 1 <= suffix <= size.
    Every code is decoded through the tables before they are accepted;
    returns None when the codes do not have that shape (the caller then
    decodes by binary search over the sorted padded codes).
    """
    cd = np.asarray(codes, dtype=np.uint64)
    L = np.asarray(lens).astype(np.int64)
    D = len(cd)
    if D == 0 or L.max() > 8 or D >= (1 << 31) - 1:
        return None
    ranks = np.arange(D, dtype=np.int64)
    b1 = ((cd >> (np.uint64(8) * (L - 1).astype(np.uint64))) & np.uint64(0xFF)).astype(np.int64)
    b2 = ((cd >> (np.uint64(8) * np.maximum(L - 2, 0).astype(np.uint64)))
          & np.uint64(0xFF)).astype(np.int64)
    one, two, deep = L == 1, L == 2, L >= 3
    M32 = 0xFFFFFFFF
    r1 = np.full(256, M32, np.int64)
    r1[b1[one]] = ranks[one]
    ch = np.full(256, M32, np.int64)
    ub1 = np.unique(b1[~one])
    ch[ub1] = np.arange(len(ub1))
    e1 = (ch | (r1 << 32)).astype(np.uint64).view(np.int64)
    nk = max(len(ub1), 1) * 256
    e2 = np.full(2 * nk, -1, np.int64)
    key = ch[b1] * 256 + b2          # valid where L >= 2
    e2[2 * key[two]] = ranks[two]
    if deep.any():
        rk, Ld = ranks[deep], L[deep]
        ukey, inv = np.unique(key[deep], return_inverse=True)
        start = np.full(len(ukey), np.iinfo(np.int64).max)
        np.minimum.at(start, inv, rk)
        size = np.bincount(inv, minlength=len(ukey)).astype(np.int64)
        beta = np.zeros(len(ukey), np.int64)
        beta[inv] = Ld - 2
        if (beta[inv] != Ld - 2).any() or size.max() >= (1 << 24):
            return None
        e2[2 * ukey + 1] = start | (size << 32) | (beta << 56)
    # decode every code through the tables and require the identity
    got = np.full(D, -1, np.int64)
    e1u = e1.view(np.uint64)
    r1g = (e1u[b1[one]] >> np.uint64(32)).astype(np.int64)
    got[one] = np.where(r1g == M32, -1, r1g)
    c = (e1u[b1] & np.uint64(M32)).astype(np.int64)
    kk = c * 256 + b2
    okc = c != M32
    if two.any():
        got[two] = np.where(okc[two], e2[2 * np.where(okc[two], kk[two], 0)], -1)
    if deep.any():
        ent = np.where(okc[deep], e2[2 * np.where(okc[deep], kk[deep], 0) + 1], -1)
        st, sz, bt = ent & M32, (ent >> 32) & 0xFFFFFF, ent >> 56
        Ld = L[deep]
        sh = (np.uint64(8) * (Ld - 2).astype(np.uint64))
        sfx = (cd[deep] & ((np.uint64(1) << sh) - np.uint64(1))).astype(np.int64)
        ok = (ent >= 0) & (bt == Ld - 2) & (sfx >= 1) & (sfx <= sz)
        got[deep] = np.where(ok, st + sfx - 1, -1)
    if not np.array_equal(got, ranks):
        return None
    return {"e1": e1, "e2": e2}


class Dictionary:
    """Value table plus one code assignment (dictionary.py:316-485)."""

    def __init__(self, table: FrequencyTable, assignment: CodeAssignment):
        if assignment.n != table.n:
            raise ValueError("assignment size does not match table")
        self.table = table
        self.assignment = assignment

    @classmethod
    def build(cls, table: FrequencyTable, scheme: str) -> "Dictionary":
        """dictionary.py:328-344."""
        if scheme == "fixed":
            return cls(table, fixed_assignment(table.n))
        if scheme == "prefix_preserving":
            a = (ppe_numerical(table.weights) if table.kind.ordered
                 else ppe_categorical(table.n))
            if a.max_len > MAX_CODE_BYTES:
                raise ValueError("code length overflow")
            return cls(table, a)
        if scheme == "prefix_free":
            return cls(table, prefix_free_assignment(table.weights))
        raise ValueError(f"unknown scheme {scheme!r}")

    @property
    def kind(self) -> ColumnKind:
        return self.table.kind

    @property
    def n(self) -> int:
        return self.table.n

    @property
    def max_len(self) -> int:
        return self.assignment.max_len

    @cached_property
    def padded(self) -> np.ndarray:
        """Codes with the padding zeros in the low bits (dictionary.py:360-368):
        code << 8*(K - len) for byte codes, code << (w_max - len) for
        prefix-free bit codes."""
        a = self.assignment
        if a.bit_granular:
            shift = np.uint64(a.width_bits) - a.lengths.astype(np.uint64)
        else:
            shift = np.uint64(8) * (np.uint64(a.max_len) - a.lengths.astype(np.uint64))
        return a.codes << shift

    @cached_property
    def _padded_order(self):
        order = np.argsort(self.padded, kind="stable")
        return self.padded[order], order

    # device-side tables ------------------------------------------------
    @property
    def numeric(self) -> bool:
        return self.table.kind is ColumnKind.NUMERIC

    @cached_property
    def dev_values(self) -> torch.Tensor:
        """rank -> value on the device; for string kinds rank -> rank (the
        lookups then return ranks, mapped to strings on the host)."""
        if not self.numeric:
            return torch.arange(self.n, dtype=torch.int64, device=device())
        return to_dev_i64(self.table.values)

    @cached_property
    def _rank_of_value(self) -> dict:
        return {v: i for i, v in enumerate(self.table.values.tolist())}

    @cached_property
    def dev_decode(self):
        """(sorted padded codes, values in that order) for lookup decode."""
        srt, order = self._padded_order
        vals = self.table.values[order] if self.numeric else order  # strings: ranks
        return torch.from_numpy(srt.view(np.int64)).to(device()), to_dev_i64(vals)

    @cached_property
    def dev_codes(self):
        a = self.assignment
        return (torch.from_numpy(a.codes.view(np.int64)).to(device()),
                torch.from_numpy(a.lengths).to(device()))

    @cached_property
    def dev_decoder(self):
        """C-ABI decoder for the lookup kernels (include/bytestore_b200.h):
        rank table for fixed codes, the PPE tree for ppe_numerical codes
        (checked against every code on build), else sorted padded codes."""
        dec = _lib.BsbDecode()
        keep = {}
        if self.assignment.scheme == "fixed":
            keep["values"] = self.dev_values
            dec.kind = 1
            dec.values = keep["values"].data_ptr()
        else:
            tree = (None if self.assignment.bit_granular else
                    ppe_decode_tree(self.assignment.codes, self.assignment.lengths))
            if tree is not None:
                dev = device()
                for k, v in tree.items():
                    keep[k] = torch.from_numpy(np.ascontiguousarray(v)).to(dev)
                keep["values"] = self.dev_values
                dec.kind = 3
                dec.values = keep["values"].data_ptr()
                dec.e1 = keep["e1"].data_ptr()
                dec.e2 = keep["e2"].data_ptr()
            else:
                sp, vals = self.dev_decode
                keep["sp"], keep["vals"] = sp, vals
                dec.kind = 2
                dec.values = vals.data_ptr()
                dec.sorted_padded = sp.data_ptr()
                dec.n_dict = sp.numel()
        dec.n_dict = dec.n_dict or self.n
        self._decoder_keep = keep
        return dec

    @property
    def dev_decoder_bytes(self) -> int:
        """Device bytes of the decoder tables (roofline: read once per launch)."""
        self.dev_decoder
        return sum(t.numel() * t.element_size() for t in self._decoder_keep.values())

    # row encoding / decoding -------------------------------------------
    def encode_rows_device(self, values) -> torch.Tensor:
        if not self.numeric:
            return to_dev_i64(self.encode_rows(values))
        v = _values_tensor(values)
        ranks = torch.empty_like(v)
        _lib.check(_lib.load().bsb_encode_rows(v.data_ptr(), v.numel(),
                                               self.dev_values.data_ptr(), self.n,
                                               ranks.data_ptr(), stream()), "encode_rows")
        return ranks

    def encode_rows(self, values) -> np.ndarray:
        """dictionary.py:381-397: ranks of raw values (KeyError if absent)."""
        if not self.numeric:
            arr = _string_array(values)
            uniq, inv = np.unique(arr, return_inverse=True)
            if self.kind.ordered:
                pos = np.searchsorted(self.table.values, uniq)
                if (pos >= self.n).any() or not (self.table.values[pos] == uniq).all():
                    raise KeyError("value missing from dictionary")
            else:
                lut = self._rank_of_value
                try:
                    pos = np.fromiter((lut[v] for v in uniq.tolist()), np.int64, len(uniq))
                except KeyError:
                    raise KeyError("value missing from dictionary") from None
            return pos[inv].astype(np.int64)
        try:
            return self.encode_rows_device(values).cpu().numpy()
        except KeyError:
            raise KeyError("value missing from dictionary") from None

    def row_codes_device(self, ranks):
        r = to_dev_i64(ranks)
        codes = torch.empty_like(r)
        lens = torch.empty(r.numel(), dtype=torch.uint8, device=r.device)
        dc, dl = self.dev_codes
        _lib.check(_lib.load().bsb_gather_codes(r.data_ptr(), r.numel(), dc.data_ptr(),
                                                dl.data_ptr(), codes.data_ptr(),
                                                lens.data_ptr(), stream()), "row_codes")
        return codes, lens

    def row_codes(self, ranks):
        """dictionary.py:399-401."""
        r = np.asarray(ranks, dtype=np.int64)
        return self.assignment.codes[r], self.assignment.lengths[r]

    def decode_padded(self, padded_codes) -> np.ndarray:
        """dictionary.py:403-411 (host); the device decode is fused into lookups."""
        q = np.asarray(padded_codes, dtype=np.uint64)
        srt, order = self._padded_order
        pos = np.searchsorted(srt, q)
        hit = (pos < self.n) & (srt[np.minimum(pos, self.n - 1)] == q)
        if not hit.all():
            raise LookupError("padded code not in dictionary")
        return self.table.values[order[pos]]

    def decode_ranks(self, ranks) -> np.ndarray:
        return self.table.values[np.asarray(ranks, dtype=np.int64)]

    # literal resolution (dictionary.py:418-485) -------------------------
    def _literal_value(self, value):
        if not self.numeric:
            if not isinstance(value, str):
                raise TypeError("string column needs a string literal")
            return value
        if isinstance(value, bool) or not isinstance(value, (int, np.integer)):
            raise TypeError("numeric column needs an integer literal")
        return int(value)

    def _code_at(self, rank: int):
        return int(self.assignment.codes[rank]), int(self.assignment.lengths[rank])

    def _resolve_one(self, op: Op, value) -> ResolvedPredicate:
        v = self._literal_value(value)
        vals = self.table.values
        n = self.n
        if op in (Op.EQ, Op.NE):
            if self.kind.ordered:
                i = int(np.searchsorted(vals, v))
                found = i < n and vals[i] == v
            else:
                i = self._rank_of_value.get(v, -1)
                found = i >= 0
            if found:
                return ResolvedPredicate.compare(op, *self._code_at(i))
            return ResolvedPredicate.constant(op is Op.NE)
        if not self.kind.ordered:
            raise ValueError("range predicate on a categorical column")
        if op in (Op.LT, Op.LE):
            cut = int(np.searchsorted(vals, v, side="left" if op is Op.LT else "right"))
            if cut == 0:
                return ResolvedPredicate.constant(False)
            if cut == n:
                return ResolvedPredicate.constant(True)
            return ResolvedPredicate.compare(Op.LE, *self._code_at(cut - 1))
        if op in (Op.GT, Op.GE):
            cut = int(np.searchsorted(vals, v, side="right" if op is Op.GT else "left"))
            if cut == n:
                return ResolvedPredicate.constant(False)
            if cut == 0:
                return ResolvedPredicate.constant(True)
            return ResolvedPredicate.compare(Op.GE, *self._code_at(cut))
        raise ValueError(f"cannot resolve operator {op}")

    def encode_literal(self, pred: Predicate) -> ResolvedPredicate:
        if pred.op is not Op.BETWEEN:
            return self._resolve_one(pred.op, pred.value)
        lo = self._resolve_one(Op.GE, pred.value)
        hi = self._resolve_one(Op.LE, pred.value_high)
        if (lo.is_trivial and not lo.trivial) or (hi.is_trivial and not hi.trivial):
            return ResolvedPredicate.constant(False)
        if lo.is_trivial and hi.is_trivial:
            return ResolvedPredicate.constant(True)
        if lo.is_trivial:
            return hi
        if hi.is_trivial:
            return lo
        return ResolvedPredicate.between(lo.code, lo.length, hi.code, hi.length)
