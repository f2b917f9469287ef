"""CPU restatement of ByteStore's scan/lookup hot path -- TEST INFRASTRUCTURE ONLY.

This module is the *checker* for the B200 product (``paper_2209_00220_b200``):
it restates, in plain numpy / Python, the algorithms of the reference package
``bytestore`` (arXiv 2209.00220, mounted read-only at /root/reference) for the
paths named by BASELINE.json's north_star.  Every function cites the reference
file:line whose behaviour it follows (paths relative to
``/root/reference/pkg/src/bytestore/``).  It is written independently (block /
level formulations of our own), not copied.

Who may use it: ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs.  The product never imports it.

Parity pinning: golden vectors produced by running the reference itself in
the build container (``tests/golden/make_golden.py``) plus the reference test
suite's known-answer values (``tests/test_oracle_golden.py``).

Conventions (reference ``bitvector.py:1-6``): 32 lanes per block, bit i of a
result lives at bit (i % 32) of uint32 word i // 32, LSB first; bits >= n_rows
are zero.  Predicates are ``Pred`` tuples in code space (reference
``predicate.py:62-95``): ``op`` in {EQ,NE,LT,LE,GT,GE,BETWEEN}, ``code`` /
``length`` (bytes) and ``code2`` / ``length2`` for BETWEEN, or ``trivial`` in
{True, False} for constant predicates.
"""

from __future__ import annotations

from collections import namedtuple
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "LANES", "Pred", "pred_compare", "pred_between", "pred_const",
    "pdep", "pext", "erase_rightmost", "propagate_rightmost", "lowest_set_index",
    "n_words", "bools_to_words", "words_to_bools", "words_count", "valid_words",
    "words_to_rows", "finalize", "OStats", "LStats",
    "bs_build", "bs_scan", "bs_lookup",
    "VbsCol", "vbs_build", "vbs_scan", "vbs_scan_serial", "vbs_lookup",
    "vbs_lookup_serial", "vbs_size_report",
    "freq_table", "fixed_assignment", "ppe_numerical", "padded_codes",
    "OracleDict", "zipf_pmf", "gen_zipf", "select_literals", "auc",
    "advise_column", "naive_filter",
]

LANES = 32
OPS = ("EQ", "NE", "LT", "LE", "GT", "GE", "BETWEEN")

Pred = namedtuple("Pred", "op code length code2 length2 trivial")


def pred_compare(op: str, code: int, length: int) -> Pred:
    """reference predicate.py:83-87 (ResolvedPredicate.compare)."""
    assert op in OPS and op != "BETWEEN"
    return Pred(op, int(code), int(length), 0, 0, None)


def pred_between(lo: int, lo_len: int, hi: int, hi_len: int) -> Pred:
    """reference predicate.py:89-91."""
    return Pred("BETWEEN", int(lo), int(lo_len), int(hi), int(hi_len), None)


def pred_const(value: bool) -> Pred:
    """reference predicate.py:79-81 (trivial predicate)."""
    return Pred(None, 0, 0, 0, 0, bool(value))


# ---------------------------------------------------------------------------
# scalar bit kernels -- reference bits.py:28-89 (semantic contract)

_W = 0xFFFFFFFF


def pdep(src: int, mask: int) -> int:
    """k-th low bit of src -> k-th set bit of mask (bits.py:28-44)."""
    src &= _W
    mask &= _W
    out, k = 0, 0
    while mask:
        low = mask & (-mask)
        if (src >> k) & 1:
            out |= low
        mask ^= low
        k += 1
    return out


def pext(src: int, mask: int) -> int:
    """bit of src at k-th set bit of mask -> bit k (bits.py:47-63)."""
    src &= _W
    mask &= _W
    out, k = 0, 0
    while mask:
        low = mask & (-mask)
        if src & low:
            out |= 1 << k
        mask ^= low
        k += 1
    return out


def erase_rightmost(x: int) -> int:
    """E(x) = x & (x-1) (bits.py:66-70)."""
    return x & (x - 1) if x else 0


def propagate_rightmost(x: int, width: int = 32) -> int:
    """P(x) = x ^ -x truncated (bits.py:73-82)."""
    return (x ^ (-x)) & ((1 << width) - 1) if x else 0


def lowest_set_index(x: int, width: int = 32) -> int:
    """index of the lowest set bit via P (bits.py:85-89)."""
    if x == 0:
        raise ValueError("word has no set bit")
    return width - 1 - bin(propagate_rightmost(x, width)).count("1")


# ---------------------------------------------------------------------------
# packed bitvector helpers -- reference bitvector.py:19-125, vbs.py:129-166


def n_words(n_rows: int) -> int:
    return (n_rows + 31) // 32


def bools_to_words(flags) -> np.ndarray:
    """LSB-first packing (bitvector.py:47-54)."""
    flags = np.asarray(flags, dtype=bool)
    n = len(flags)
    buf = np.zeros(n_words(n) * 4, dtype=np.uint8)
    packed = np.packbits(flags, bitorder="little")
    buf[: len(packed)] = packed
    return buf.view(np.uint32).copy()


def words_to_bools(words, n_rows: int) -> np.ndarray:
    """bitvector.py:64-69."""
    w = np.ascontiguousarray(words, dtype=np.uint32)
    return np.unpackbits(w.view(np.uint8), bitorder="little")[:n_rows].astype(bool)


def words_to_rows(words, n_rows: int) -> np.ndarray:
    """Ascending int64 row ids of set bits (bitvector.py:71-72)."""
    return np.flatnonzero(words_to_bools(words, n_rows)).astype(np.int64)


def words_count(words) -> int:
    """bitvector.py:74-75."""
    return int(np.bitwise_count(np.asarray(words, dtype=np.uint32)).sum())


def valid_words(n_rows: int) -> np.ndarray:
    """All-ones block words, tail block truncated (vbs.py:129-136)."""
    nb = n_words(n_rows)
    w = np.full(nb, 0xFFFFFFFF, dtype=np.uint32)
    if n_rows % 32:
        w[-1] = np.uint32((1 << (n_rows % 32)) - 1)
    return w


def _init_words(mask, n_rows: int) -> np.ndarray:
    """Input mask AND tail validity (vbs.py:139-154)."""
    v = valid_words(n_rows)
    if mask is None:
        return v
    m = np.asarray(mask, dtype=np.uint32)
    if m.shape != v.shape:
        raise ValueError("input mask length mismatch")
    return m & v


def finalize(op: str, gt, eq, valid):
    """Derive an operator from (gt, eq) lane masks (vbs.py:179-197)."""
    table = {
        "GT": lambda: gt,
        "GE": lambda: gt | eq,
        "EQ": lambda: eq,
        "NE": lambda: valid & ~eq,
        "LT": lambda: valid & ~(gt | eq),
        "LE": lambda: valid & ~gt,
    }
    if op not in table:
        raise ValueError(f"unsupported scan operator {op}")
    return table[op]()


# ---------------------------------------------------------------------------
# access statistics -- reference stats.py:18-97


@dataclass
class OStats:
    levels: int
    blocks_total: int = 0
    blocks_skipped: int = 0
    words_loaded: np.ndarray = None
    bytes_loaded: np.ndarray = None
    mask_bytes: int = 0
    block_depth: np.ndarray = None

    def __post_init__(self):
        if self.words_loaded is None:
            self.words_loaded = np.zeros(self.levels, dtype=np.int64)
        if self.bytes_loaded is None:
            self.bytes_loaded = np.zeros(self.levels, dtype=np.int64)

    @property
    def total_bytes(self) -> int:
        """stats.py:36-39 -- the advisor's "bytes" cost."""
        return int(self.bytes_loaded.sum()) + int(self.mask_bytes)

    def merge(self, o: "OStats") -> "OStats":
        """Pipelined BETWEEN legs (stats.py:47-67)."""
        L = max(self.levels, o.levels)
        w = np.zeros(L, np.int64)
        b = np.zeros(L, np.int64)
        w[: self.levels] += self.words_loaded
        w[: o.levels] += o.words_loaded
        b[: self.levels] += self.bytes_loaded
        b[: o.levels] += o.bytes_loaded
        d = None
        if self.block_depth is not None and o.block_depth is not None:
            d = np.maximum(self.block_depth, o.block_depth)
        return OStats(L, self.blocks_total, min(self.blocks_skipped, o.blocks_skipped),
                      w, b, self.mask_bytes + o.mask_bytes, d)

    def concat(self, o: "OStats") -> "OStats":
        """Disjoint block ranges (stats.py:69-84)."""
        if self.levels != o.levels:
            raise ValueError("level counts differ")
        return OStats(self.levels, self.blocks_total + o.blocks_total,
                      self.blocks_skipped + o.blocks_skipped,
                      self.words_loaded + o.words_loaded,
                      self.bytes_loaded + o.bytes_loaded,
                      self.mask_bytes + o.mask_bytes,
                      np.concatenate([self.block_depth, o.block_depth]))


@dataclass
class LStats:
    """stats.py:87-97."""
    levels_touched: int = 0
    bytes_loaded: int = 0
    mask_bytes: int = 0

    @property
    def total_bytes(self) -> int:
        return self.bytes_loaded + self.mask_bytes


def _trivial(value: bool, n_rows: int, mask, levels: int):
    """vbs.py:200-208: constants never touch slices."""
    nb = n_words(n_rows)
    st = OStats(levels, nb, nb, block_depth=np.zeros(nb, np.int8))
    if not value:
        return np.zeros(nb, np.uint32), st
    return _init_words(mask, n_rows).copy(), st


def _partition(nb: int, threads: int):
    """Contiguous block ranges, one per worker (vbs.py:211-215)."""
    threads = max(1, min(threads, nb))
    step = -(-nb // threads)
    return [(lo, min(lo + step, nb)) for lo in range(0, nb, step)]


def _lane_pack(flags2d: np.ndarray) -> np.ndarray:
    """(rows, 32) bools -> one LSB-first uint32 per row (movemask)."""
    return np.packbits(flags2d, axis=1, bitorder="little").view(np.uint32).ravel()


def _be_bytes(code: int, length: int):
    """Big-endian byte list of a `length`-byte literal (vbs.py:175-176)."""
    return [(int(code) >> (8 * (length - 1 - i))) & 0xFF for i in range(length)]


def _run_ranges(fn, nb: int, threads: int):
    spans = _partition(nb, threads)
    if len(spans) == 1:
        return [fn(*spans[0])]
    with ThreadPoolExecutor(len(spans)) as pool:
        return list(pool.map(lambda s: fn(*s), spans))


# ---------------------------------------------------------------------------
# ByteSlice -- reference byteslice.py:52-158


def bs_build(codes, width_bits: int) -> np.ndarray:
    """Left-aligned byte planes, shape (K, nb*32) (byteslice.py:56-73)."""
    c = np.ascontiguousarray(codes, dtype=np.uint64)
    n = len(c)
    if n == 0:
        raise ValueError("empty column")
    if not 1 <= width_bits <= 64:
        raise ValueError("width must be 1..64 bits")
    if width_bits < 64 and (c >> np.uint64(width_bits)).any():
        raise ValueError("code wider than declared width")
    K = -(-width_bits // 8)
    a = c << np.uint64(8 * K - width_bits)
    planes = np.zeros((K, n_words(n) * 32), np.uint8)
    for j in range(K):
        planes[j, :n] = (a >> np.uint64(8 * (K - 1 - j))).astype(np.uint8)
    return planes


def _bs_scan_one(planes, width_bits, n_rows, op, code, init, threads):
    K = planes.shape[0]
    lit = _be_bytes(int(code) << (8 * K - width_bits), K)  # byteslice.py:81
    nb = n_words(n_rows)

    def span(b0, b1):
        valid = init[b0:b1]
        eq = valid.copy()
        gt = np.zeros_like(valid)
        depth = np.zeros(b1 - b0, np.int8)
        st = OStats(K, b1 - b0, int((valid == 0).sum()))
        for j in range(K):
            act = np.flatnonzero(eq)
            if act.size == 0:
                break
            depth[act] = j + 1
            st.words_loaded[j] += act.size
            st.bytes_loaded[j] += act.size * 32
            blk = planes[j].reshape(-1, 32)[b0 + act]
            mg = _lane_pack(blk > lit[j])
            me = _lane_pack(blk == lit[j])
            z = eq[act]
            gt[act] |= z & mg
            eq[act] = z & me
        st.block_depth = depth
        return gt, eq, valid, st

    parts = _run_ranges(span, nb, threads)
    gt = np.concatenate([p[0] for p in parts])
    eq = np.concatenate([p[1] for p in parts])
    valid = np.concatenate([p[2] for p in parts])
    st = parts[0][3]
    for p in parts[1:]:
        st = st.concat(p[3])
    return finalize(op, gt, eq, valid).astype(np.uint32), st


def bs_scan(planes, width_bits: int, n_rows: int, pred: Pred, mask=None,
            threads: int = 1):
    """Early-stopping ByteSlice scan (byteslice.py:76-140).

    Returns (uint32 result words, OStats).  pred.length is ignored: the
    literal is left-aligned exactly like the codes (byteslice.py:81).
    """
    K = planes.shape[0]
    if pred.trivial is not None:
        return _trivial(pred.trivial, n_rows, mask, K)
    if pred.op == "BETWEEN":
        w1, s1 = bs_scan(planes, width_bits, n_rows,
                         pred_compare("GE", pred.code, pred.length), mask, threads)
        w2, s2 = bs_scan(planes, width_bits, n_rows,
                         pred_compare("LE", pred.code2, pred.length2), w1, threads)
        return w2, s1.merge(s2)
    init = _init_words(mask, n_rows)
    return _bs_scan_one(planes, width_bits, n_rows, pred.op, pred.code, init, threads)


def bs_lookup(planes, width_bits: int, rows):
    """Right-aligned codes of the given rows (byteslice.py:143-158)."""
    rows = np.asarray(rows, dtype=np.int64)
    K = planes.shape[0]
    out = np.zeros(len(rows), np.uint64)
    for j in range(K):
        out = (out << np.uint64(8)) | planes[j][rows].astype(np.uint64)
    st = LStats(K if len(rows) else 0, len(rows) * K if len(rows) else 0, 0)
    return out >> np.uint64(8 * K - width_bits), st


# ---------------------------------------------------------------------------
# Variable byte slices (PP-VBS) -- reference vbs.py:42-498


@dataclass
class VbsCol:
    n_rows: int
    K: int
    slices: list          # slices[0] padded to nb*32; slices[j>=1] packed rows with len > j
    exist: list           # exist[j-2]: uint32 per block, rows having byte j (j = 2..K)
    block_dir: np.ndarray  # (K-1, nb+1) int64: bytes of slice j before block b
    rows_of: list = field(default_factory=list)  # oracle-only: row of each packed byte

    @property
    def n_blocks(self) -> int:
        return n_words(self.n_rows)


def vbs_build(codes, lens) -> VbsCol:
    """vbs.py:68-114: BS_1 dense, BS_j>=2 packed, existence words, directory."""
    c = np.ascontiguousarray(codes, dtype=np.uint64)
    ln = np.ascontiguousarray(lens, dtype=np.uint8)
    n = len(c)
    if n == 0:
        raise ValueError("empty column")
    if len(ln) != n:
        raise ValueError("codes and lengths differ in length")
    if ln.min() < 1 or ln.max() > 8:
        raise ValueError("code lengths must be 1..8 bytes")
    short = ln < 8
    if (c[short] >> (np.uint64(8) * ln[short].astype(np.uint64))).any():
        raise ValueError("code wider than its declared length")
    K = int(ln.max())
    nb = n_words(n)
    first = np.zeros(nb * 32, np.uint8)
    first[:n] = (c >> (np.uint64(8) * (ln.astype(np.uint64) - np.uint64(1)))).astype(np.uint8)
    slices, exist, rows_of = [first], [], []
    bdir = np.zeros((max(K - 1, 0), nb + 1), np.int64)
    for j in range(2, K + 1):
        has = ln >= j
        rows = np.flatnonzero(has)
        sh = (ln[rows].astype(np.uint64) - np.uint64(j)) * np.uint64(8)
        slices.append((c[rows] >> sh).astype(np.uint8))
        flags = np.zeros(nb * 32, bool)
        flags[:n] = has
        exist.append(bools_to_words(flags))
        bdir[j - 2, 1:] = np.cumsum(np.bincount(rows >> 5, minlength=nb))
        rows_of.append(rows)
    return VbsCol(n, K, slices, exist, bdir, rows_of)


def _vbs_scan_one(col: VbsCol, op, code, length, init, threads):
    K = col.K
    if length > K:
        # the reference indexes past exist_bits here (vbs.py:274); device path
        # reports ValueError instead
        raise ValueError("literal longer than the column's longest code")
    lit = _be_bytes(code, length)
    nb = col.n_blocks
    first2d = col.slices[0].reshape(-1, 32)

    def span(b0, b1):
        nbl = b1 - b0
        valid = init[b0:b1]
        zeq = valid.copy()
        zgt = np.zeros(nbl, np.uint32)
        eqf = np.zeros(nbl, np.uint32)
        depth = np.zeros(nbl, np.int8)
        st = OStats(K, nbl, int((valid == 0).sum()))
        for j in range(1, length + 1):
            act = np.flatnonzero(zeq)
            if act.size == 0:
                break
            depth[act] = j
            st.words_loaded[j - 1] += act.size
            if j == 1:
                blk = first2d[b0 + act]
                mg = _lane_pack(blk > lit[0])
                me = _lane_pack(blk == lit[0])
                st.bytes_loaded[0] += act.size * 32
            else:
                # bytes of level j whose block is active, deposited at their lane
                rows = col.rows_of[j - 2]
                lo = col.block_dir[j - 2][b0 + act[0]]
                hi = col.block_dir[j - 2][b0 + act[-1] + 1]
                rows = rows[lo:hi]
                data = col.slices[j - 1][lo:hi]
                local = (rows >> 5) - b0
                slot = np.full(nbl, -1, np.int64)
                slot[act] = np.arange(act.size)
                keep = slot[local] >= 0
                st.bytes_loaded[j - 1] += int(keep.sum())
                rows, data, local = rows[keep], data[keep], local[keep]
                g = np.zeros((act.size, 32), bool)
                e = np.zeros((act.size, 32), bool)
                g[slot[local], rows & 31] = data > lit[j - 1]
                e[slot[local], rows & 31] = data == lit[j - 1]
                mg, me = _lane_pack(g), _lane_pack(e)
            z = zeq[act]
            if j < length:
                nxt = col.exist[j - 1][b0 + act]
                zgt[act] |= z & mg
                zeq[act] = z & me & nxt
            elif length < K:
                nxt = col.exist[j - 1][b0 + act]
                still = z & me
                zgt[act] |= (z & mg) | (still & nxt)   # existence shortcut
                eqf[act] = still & ~nxt
                zeq[act] = 0
            else:
                zgt[act] |= z & mg
                eqf[act] = z & me
                zeq[act] = 0
        live = nbl - st.blocks_skipped
        st.mask_bytes = live * 4 * (min(length + 1, K) - 1)   # vbs.py:286-287
        st.block_depth = depth
        return zgt, eqf, valid, st

    parts = _run_ranges(span, nb, threads)
    gt = np.concatenate([p[0] for p in parts])
    eq = np.concatenate([p[1] for p in parts])
    valid = np.concatenate([p[2] for p in parts])
    st = parts[0][3]
    for p in parts[1:]:
        st = st.concat(p[3])
    return finalize(op, gt, eq, valid).astype(np.uint32), st


def vbs_scan(col: VbsCol, pred: Pred, mask=None, threads: int = 1):
    """Alg. 3 over all blocks (vbs.py:222-324). Returns (words, OStats)."""
    if pred.trivial is not None:
        return _trivial(pred.trivial, col.n_rows, mask, col.K)
    if pred.op == "BETWEEN":
        w1, s1 = vbs_scan(col, pred_compare("GE", pred.code, pred.length), mask, threads)
        w2, s2 = vbs_scan(col, pred_compare("LE", pred.code2, pred.length2), w1, threads)
        return w2, s1.merge(s2)
    init = _init_words(mask, col.n_rows)
    return _vbs_scan_one(col, pred.op, pred.code, pred.length, init, threads)


def vbs_scan_serial(col: VbsCol, pred: Pred, mask=None):
    """Block-at-a-time Alg. 3 with scalar pdep (vbs.py:378-462)."""
    if pred.trivial is not None:
        return _trivial(pred.trivial, col.n_rows, mask, col.K)
    if pred.op == "BETWEEN":
        w1, s1 = vbs_scan_serial(col, pred_compare("GE", pred.code, pred.length), mask)
        w2, s2 = vbs_scan_serial(col, pred_compare("LE", pred.code2, pred.length2), w1)
        return w2, s1.merge(s2)
    K, l = col.K, pred.length
    if l > K:
        raise ValueError("literal longer than the column's longest code")
    lit = _be_bytes(pred.code, l)
    init = _init_words(mask, col.n_rows)
    nb = col.n_blocks
    st = OStats(K, nb)
    depth = np.zeros(nb, np.int8)
    out = np.zeros(nb, np.uint32)
    for b in range(nb):
        valid = int(init[b])
        if not valid:
            st.blocks_skipped += 1
            continue
        M = {j: int(col.exist[j - 2][b]) for j in range(2, min(l + 1, K) + 1)}
        st.mask_bytes += 4 * len(M)
        zeq, zgt, eqf = valid, 0, 0
        for j in range(1, l + 1):
            if not zeq:
                break
            depth[b] = j
            st.words_loaded[j - 1] += 1
            if j == 1:
                blk = col.slices[0][32 * b: 32 * b + 32]
                mg = sum(1 << r for r in range(32) if blk[r] > lit[0])
                me = sum(1 << r for r in range(32) if blk[r] == lit[0])
                st.bytes_loaded[0] += 32
            else:
                ex = M[j]
                s0 = int(col.block_dir[j - 2][b])
                seg = col.slices[j - 1][s0: s0 + bin(ex).count("1")]
                st.bytes_loaded[j - 1] += len(seg)
                pg = sum(1 << k for k, v in enumerate(seg) if v > lit[j - 1])
                pe = sum(1 << k for k, v in enumerate(seg) if v == lit[j - 1])
                mg, me = pdep(pg, ex), pdep(pe, ex)
            if j < l:
                zgt |= zeq & mg
                zeq = zeq & me & M[j + 1]
            elif l < K:
                still = zeq & me
                zgt |= (zeq & mg) | (still & M[l + 1])
                eqf = still & ~M[l + 1] & _W
                zeq = 0
            else:
                zgt |= zeq & mg
                eqf = zeq & me
                zeq = 0
        out[b] = finalize(pred.op, zgt, eqf, valid) & _W
    st.block_depth = depth
    return out, st


def vbs_lookup(col: VbsCol, rows):
    """Padded codes of the given rows (vbs.py:331-371).  Returns (codes, LStats).

    ``rows`` may be in any order (the bitvector form passes ascending rows).
    """
    rows = np.asarray(rows, dtype=np.int64)
    K = col.K
    out = col.slices[0][rows].astype(np.uint64) << np.uint64(8 * (K - 1))
    st = LStats()
    if len(rows) == 0:
        return out, st
    st.levels_touched = 1
    st.bytes_loaded = len(rows)
    alive = np.arange(len(rows))
    for j in range(2, K + 1):
        r = rows[alive]
        w = col.exist[j - 2][r >> 5]
        bit = (r & 31).astype(np.uint32)
        has = ((w >> bit) & np.uint32(1)).astype(bool)
        if not has.any():
            break
        st.levels_touched = j
        alive, r, w, bit = alive[has], r[has], w[has], bit[has]
        st.bytes_loaded += len(alive)
        below = (np.uint32(1) << bit) - np.uint32(1)
        pos = col.block_dir[j - 2][r >> 5] + np.bitwise_count(w & below).astype(np.int64)
        out[alive] |= col.slices[j - 1][pos].astype(np.uint64) << np.uint64(8 * (K - j))
    return out, st


def vbs_lookup_serial(col: VbsCol, sel_words) -> np.ndarray:
    """Alg. 4 with pext / P / E per selection word (vbs.py:465-498)."""
    K = col.K
    out = []
    for b, x in enumerate(np.asarray(sel_words, dtype=np.uint32).tolist()):
        if not x:
            continue
        ex = [int(col.exist[j - 2][b]) for j in range(2, K + 1)]
        beta = 1
        for j in range(2, K + 1):
            if x & ex[j - 2] == 0:
                break
            beta = j
        deep = [pext(x, ex[j - 2]) for j in range(2, beta + 1)]
        while x:
            lane = lowest_set_index(x)
            code = int(col.slices[0][32 * b + lane])
            x = erase_rightmost(x)
            got = 1
            for j in range(2, beta + 1):
                if not (ex[j - 2] >> lane) & 1:
                    break
                xj = deep[j - 2]
                off = int(col.block_dir[j - 2][b]) + lowest_set_index(xj)
                code = (code << 8) | int(col.slices[j - 1][off])
                deep[j - 2] = erase_rightmost(xj)
                got = j
            out.append(code << (8 * (K - got)))
    return np.array(out, dtype=np.uint64)


def vbs_size_report(col: VbsCol) -> dict:
    """vbs.py:505-517."""
    sb = [col.n_rows] + [len(s) for s in col.slices[1:]]
    mb = ((col.n_rows + 7) // 8) * (col.K - 1)
    db = col.n_blocks * (col.K - 1) * 4
    data = sum(sb) + mb
    return {"slice_bytes": sb, "mask_bytes": mb, "directory_bytes": db,
            "total_bytes": data + db, "avg_bits_per_code": 8.0 * data / col.n_rows}


# ---------------------------------------------------------------------------
# dictionary encoders -- reference dictionary.py:101-485 (numeric / ordered)


def freq_table(values):
    """Sorted distinct values + counts (dictionary.py:101-106)."""
    v = np.asarray(values).astype(np.int64)
    if v.ndim != 1 or v.size == 0:
        raise ValueError("column must be a nonempty 1-d sequence")
    u, c = np.unique(v, return_counts=True)
    return u, c.astype(np.int64)


def fixed_assignment(D: int):
    """Rank codes at w = max(1, ceil(log2 D)) bits (dictionary.py:233-242)."""
    if D <= 0:
        raise ValueError("need at least one value")
    w = max(1, (D - 1).bit_length())
    if w > 32:
        raise ValueError("dictionary width overflow (more than 2**32 values)")
    return np.arange(D, dtype=np.uint64), np.full(D, (w + 7) // 8, np.uint8), w


def _suffix_bytes(m: int) -> int:
    """least beta with 256**beta >= m, 0 for m <= 1 (dictionary.py:143-145)."""
    beta = 0
    while (1 << (8 * beta)) < m:
        beta += 1
    return beta


def ppe_numerical(weights):
    """Alg. 1: order-preserving variable byte codes (dictionary.py:148-196).

    A node covering [s, e) at depth b becomes a leaf when it has fewer than
    256 values or b >= 2; a leaf enumerates its values with 1 + (i - s) in the
    fewest bytes that hold size+1.  Otherwise its 255 heaviest values (ties to
    the lower index) take sub-codes 1..255 in value order and each gap range
    descends through pointer t = number of slots to its left.
    """
    w = np.asarray(weights, dtype=np.int64)
    D = len(w)
    if D == 0:
        raise ValueError("empty weight table")
    if (w < 0).any():
        raise ValueError("negative weight")
    codes = np.zeros(D, np.uint64)
    lens = np.zeros(D, np.uint8)
    todo = [(0, D, 0, 0)]  # (start, end, depth, prefix)
    while todo:
        s, e, b, prefix = todo.pop()
        size = e - s
        if size == 0:
            continue
        if size < 256 or b >= 2:
            beta = _suffix_bytes(size + 1)
            codes[s:e] = (np.uint64(prefix) << np.uint64(8 * beta)) + \
                np.arange(1, size + 1, dtype=np.uint64)
            lens[s:e] = b + beta
            continue
        # stable descending weight: heaviest first, equal weights by index
        order = np.lexsort((np.arange(size), -w[s:e]))[:255]
        slots = np.sort(order) + s
        codes[slots] = (np.uint64(prefix) << np.uint64(8)) + np.arange(1, 256, dtype=np.uint64)
        lens[slots] = b + 1
        bounds = [s - 1] + slots.tolist() + [e]
        for t in range(256):
            cs, ce = bounds[t] + 1, bounds[t + 1]
            if ce > cs:
                todo.append((cs, ce, b + 1, (prefix << 8) | t))
    return codes, lens


def padded_codes(codes, lens, K: int) -> np.ndarray:
    """code << 8*(K - len) (dictionary.py:360-368)."""
    return np.asarray(codes, np.uint64) << (np.uint64(8) * (np.uint64(K) - np.asarray(lens).astype(np.uint64)))


class OracleDict:
    """Numeric dictionary with fixed or prefix-preserving codes.

    Mirrors Dictionary.build / encode_rows / row_codes / decode_* /
    encode_literal (dictionary.py:316-485) for ordered numeric columns.
    """

    def __init__(self, values_sorted, weights, scheme: str):
        self.values = np.asarray(values_sorted, np.int64)
        self.weights = np.asarray(weights, np.int64)
        self.scheme = scheme
        if scheme == "fixed":
            self.codes, self.lens, self.width_bits = fixed_assignment(len(self.values))
        elif scheme == "prefix_preserving":
            self.codes, self.lens = ppe_numerical(self.weights)
            self.width_bits = 0
            if int(self.lens.max()) > 8:
                raise ValueError("code length overflow")
        else:
            raise ValueError(scheme)
        self.K = int(self.lens.max())
        self.padded = padded_codes(self.codes, self.lens, self.K)
        self._order = np.argsort(self.padded, kind="stable")
        self._sorted = self.padded[self._order]

    @classmethod
    def from_values(cls, values, scheme):
        u, c = freq_table(values)
        return cls(u, c, scheme)

    @property
    def n(self):
        return len(self.values)

    def encode_rows(self, values) -> np.ndarray:
        """dictionary.py:381-397."""
        v = np.asarray(values, np.int64)
        pos = np.searchsorted(self.values, v)
        if (pos >= self.n).any() or (self.values[np.minimum(pos, self.n - 1)] != v).any():
            raise KeyError("value missing from dictionary")
        return pos.astype(np.int64)

    def row_codes(self, ranks):
        return self.codes[ranks], self.lens[ranks]

    def decode_padded(self, q) -> np.ndarray:
        """dictionary.py:403-411."""
        q = np.asarray(q, np.uint64)
        pos = np.searchsorted(self._sorted, q)
        bad = (pos >= self.n) | (self._sorted[np.minimum(pos, self.n - 1)] != q)
        if bad.any():
            raise LookupError("padded code not in dictionary")
        return self.values[self._order[pos]]

    def decode_ranks(self, ranks) -> np.ndarray:
        return self.values[np.asarray(ranks, np.int64)]

    def _code(self, rank: int):
        return int(self.codes[rank]), int(self.lens[rank])

    def _resolve_one(self, op: str, value: int) -> Pred:
        """dictionary.py:427-463 (ordered kinds)."""
        vals = self.values
        if op in ("EQ", "NE"):
            pos = int(np.searchsorted(vals, value))
            if pos < self.n and vals[pos] == value:
                return pred_compare(op, *self._code(pos))
            return pred_const(op == "NE")
        if op in ("LT", "LE"):
            cut = int(np.searchsorted(vals, value, side="left" if op == "LT" else "right"))
            if cut == 0:
                return pred_const(False)
            if cut == self.n:
                return pred_const(True)
            return pred_compare("LE", *self._code(cut - 1))
        if op in ("GT", "GE"):
            cut = int(np.searchsorted(vals, value, side="right" if op == "GT" else "left"))
            if cut == self.n:
                return pred_const(False)
            if cut == 0:
                return pred_const(True)
            return pred_compare("GE", *self._code(cut))
        raise ValueError(op)

    def encode_literal(self, op: str, value, value_high=None) -> Pred:
        """dictionary.py:465-485."""
        if op != "BETWEEN":
            return self._resolve_one(op, int(value))
        lo = self._resolve_one("GE", int(value))
        hi = self._resolve_one("LE", int(value_high))
        for side in (lo, hi):
            if side.trivial is False:
                return pred_const(False)
        if lo.trivial is not None and hi.trivial is not None:
            return pred_const(True)
        if lo.trivial is not None:
            return hi
        if hi.trivial is not None:
            return lo
        return pred_between(lo.code, lo.length, hi.code, hi.length)


# ---------------------------------------------------------------------------
# synthetic data -- reference datagen.py:43-56


def zipf_pmf(s: float, domain: int) -> np.ndarray:
    r = np.arange(1, domain + 1, dtype=np.float64) ** -float(s)
    return r / r.sum()


def gen_zipf(s: float, domain_bits: int, n_rows: int, seed: int) -> np.ndarray:
    """Inverse-CDF Zipf draws on PCG64 uniforms; rank k -> value k-1."""
    cdf = np.cumsum(zipf_pmf(s, 1 << domain_bits))
    cdf[-1] = 1.0
    u = np.random.default_rng(seed).random(n_rows)
    return np.searchsorted(cdf, u, side="right").astype(np.int64)


# ---------------------------------------------------------------------------
# advisor -- reference advisor.py:47-150 (ordered columns)


def select_literals(values, count: int = 100):
    """Nearest-rank quantile literals probed with LT (advisor.py:47-59)."""
    srt = np.sort(np.asarray(values))
    n = len(srt)
    idx = np.minimum(n - 1, (np.arange(1, count + 1) * n) // count)
    return "LT", [int(x) for x in srt[idx]]


def auc(points) -> float:
    """Trapezoid of cost over selectivity, stable-sorted (advisor.py:69-76)."""
    if len(points) < 2:
        raise ValueError("need at least 2 profile points")
    s = np.array([p[0] for p in points], np.float64)
    y = np.array([p[1] for p in points], np.float64)
    o = np.argsort(s, kind="stable")
    return float(np.trapezoid(y[o], s[o]))


def advise_column(values, count: int = 100, cost="bytes", subsample=None):
    """Alg. 5 with cost 'bytes' or a callable(run) (advisor.py:119-150).

    Returns dict(chosen, auc_byteslice, auc_ppvbs, points_byteslice,
    points_ppvbs, degenerate).
    """
    v = np.asarray(values).astype(np.int64)
    if subsample is not None and len(v) > subsample:
        v = v[:: -(-len(v) // subsample)]
    u, c = freq_table(v)
    if len(u) < 2:
        return {"chosen": "byteslice", "degenerate": True}
    op, lits = select_literals(v, count)
    dfix = OracleDict(u, c, "fixed")
    dppe = OracleDict(u, c, "prefix_preserving")
    ranks = dfix.encode_rows(v)
    planes = bs_build(ranks, dfix.width_bits)
    col = vbs_build(*dppe.row_codes(ranks))
    n = len(v)

    def profile(scan_fn, d):
        pts = []
        for lit in lits:
            p = d.encode_literal(op, lit)
            run = lambda p=p: scan_fn(p)
            if cost == "bytes":
                y = float(run()[1].total_bytes)
            else:
                y = float(cost(run))
            words, _ = run()
            pts.append((words_count(words) / n, y))
        return pts

    pb = profile(lambda p: bs_scan(planes, dfix.width_bits, n, p), dfix)
    pv = profile(lambda p: vbs_scan(col, p), dppe)
    y, z = auc(pb), auc(pv)
    return {"chosen": "byteslice" if y <= z else "ppvbs", "auc_byteslice": y,
            "auc_ppvbs": z, "points_byteslice": pb, "points_ppvbs": pv,
            "degenerate": False}


def naive_filter(values, op: str, lo, hi=None) -> np.ndarray:
    """Raw-value oracle that knows nothing about codes (tests/helpers.py:35-52)."""
    v = np.asarray(values)
    return {
        "EQ": lambda: v == lo, "NE": lambda: v != lo, "LT": lambda: v < lo,
        "LE": lambda: v <= lo, "GT": lambda: v > lo, "GE": lambda: v >= lo,
        "BETWEEN": lambda: (v >= lo) & (v <= hi),
    }[op]()
