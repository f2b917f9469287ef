"""Parity of the CUDA path against the reference's golden vectors and the
CPU oracle.  Everything here calls through the C ABI on a B200; the bar is
bit-exactness (bitvectors, counts, stats, looked-up codes and values)."""

import numpy as np
import pytest
import torch

import oracle as O
from golden_io import load, stats_of

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected only on GPU boxes
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2209_00220_b200 as B  # noqa: E402
from paper_2209_00220_b200 import engine as E  # noqa: E402
from paper_2209_00220_b200.predicate import Op, Predicate, ResolvedPredicate  # noqa: E402


def rp(t):
    op, code, length, code2, length2, trivial = t
    if trivial is not None:
        return ResolvedPredicate.constant(trivial)
    if op == "BETWEEN":
        return ResolvedPredicate.between(code, length, code2, length2)
    return ResolvedPredicate.compare(Op[op], code, length)


def op_pred(t):
    op, code, length, code2, length2, trivial = t
    if trivial is not None:
        return O.pred_const(trivial)
    if op == "BETWEEN":
        return O.pred_between(code, length, code2, length2)
    return O.pred_compare(op, code, length)


def check_stats(st, want):
    assert st.levels == want["levels"]
    assert st.blocks_total == want["blocks_total"]
    assert st.blocks_skipped == want["blocks_skipped"]
    assert list(st.words_loaded) == want["words_loaded"].tolist()
    assert list(st.bytes_loaded) == want["bytes_loaded"].tolist()
    assert st.mask_bytes == want["mask_bytes"]
    assert st.total_bytes == want["total_bytes"]
    assert st.block_depth.tolist() == want["block_depth"].tolist()


# --------------------------------------------------------------- datagen


def test_gen_zipf_matches_reference():
    data, meta = load("zipf")
    for i, m in enumerate(meta):
        got = B.gen_zipf(B.ZipfSpec(m["s"], m["d"], m["n"], m["seed"]))
        assert np.array_equal(got, data[f"{i}/values"])


# ------------------------------------------------------------- ByteSlice


def test_byteslice_golden():
    data, meta = load("bs")
    for ci, m in enumerate(meta):
        codes = data[f"{ci}/codes"]
        col = B.build_byteslice(codes, m["w"])
        assert np.array_equal(col.slices, data[f"{ci}/slices"]), ci
        mask = B.ResultBitVector(m["n"], data[f"{ci}/mask"])
        for pi, t in enumerate(m["preds"]):
            for mi, msk in enumerate((None, mask)):
                key = f"{ci}/p{pi}m{mi}/"
                bv, st = B.scan_byteslice(col, rp(t), msk)
                want = data[key + "words"]
                assert np.array_equal(bv.words, want), key
                assert bv.count() == O.words_count(want)
                if pi % 3 == 0 or t[0] == "BETWEEN" or t[5] is not None:
                    check_stats(st, stats_of(data, key))
        sel = B.ResultBitVector(m["n"], data[f"{ci}/sel"])
        got, lst = B.lookup_byteslice(col, sel)
        assert np.array_equal(got, data[f"{ci}/lookup"])
        assert [lst.levels_touched, lst.bytes_loaded, lst.mask_bytes] == \
            data[f"{ci}/lookup_stats"].tolist()


def test_byteslice_random_large_between_and_masks():
    rng = np.random.default_rng(123)
    for w, n in ((16, (1 << 20) + 7), (20, 300_001), (32, 70_000), (9, 4097), (64, 5000)):
        hi_bound = (1 << w) if w < 64 else (1 << 63)
        codes = rng.integers(0, hi_bound, size=n, dtype=np.uint64)
        col = B.build_byteslice(codes, w)
        planes = O.bs_build(codes, w)
        K = planes.shape[0]
        mask = rng.random(n) < 0.7
        mw = O.bools_to_words(mask)
        for _ in range(6):
            a, b = sorted(int(x) for x in rng.choice(codes, 2))
            for p in (O.pred_between(a, K, b, K), O.pred_compare("LT", b, K),
                      O.pred_compare("EQ", a, K), O.pred_compare("NE", a, K)):
                rpred = rp(list(p))
                for m_o, m_d in ((None, None), (mw, B.ResultBitVector(n, mw))):
                    want, _ = O.bs_scan(planes, w, n, p, m_o)
                    bv, _ = B.scan_byteslice(col, rpred, m_d)
                    assert np.array_equal(bv.words, want)
                    assert bv.count() == O.words_count(want)


@pytest.mark.parametrize("small", [0, 1])
def test_byteslice_small_column_kernel_and_no_count(small):
    """Columns that fit one wave take bs_scan_small_kernel (every tile's
    sectors of a level in flight together, PDL launch); bsb_tune bs_small=0
    forces the persistent kernel.  Both equal the oracle for w = 8..64,
    ragged ends, every operator and BETWEEN; count = NULL returns the same
    words without a count."""
    import ctypes
    lib = B._lib.load()
    rng = np.random.default_rng(900 + small)
    assert lib.bsb_tune(b"bs_small", small) == 0
    try:
        for w, n in ((16, 1 << 24), (8, 1000), (24, (1 << 20) + 33), (64, 70_001), (40, 32)):
            hi_bound = (1 << w) if w < 64 else (1 << 63)
            codes = rng.integers(0, hi_bound, size=n, dtype=np.uint64)
            col = B.build_byteslice(codes, w)
            planes = O.bs_build(codes, w)
            K = planes.shape[0]
            a, b = sorted(int(x) for x in rng.choice(codes, 2))
            preds = [O.pred_between(a, K, b, K)] + [O.pred_compare(op, b, K) for op in
                                                    ("EQ", "NE", "LT", "LE", "GT", "GE")]
            out = torch.empty(-(-n // 32), dtype=torch.int32, device="cuda")
            for p in preds:
                want, _ = O.bs_scan(planes, w, n, p)
                bv, _ = B.scan_byteslice(col, rp(list(p)))
                assert np.array_equal(bv.words, want), (w, n, p[0])
                assert bv.count() == O.words_count(want)
                cp = rp(list(p)).to_c()
                out.fill_(-1)
                B._lib.check(lib.bsb_byteslice_scan(col.desc_ref, ctypes.byref(cp), None,
                                                    out.data_ptr(), None, None, None,
                                                    B._lib.stream_ptr()), "no-count scan")
                assert np.array_equal(out.cpu().numpy().view(np.uint32), want), (w, n)
    finally:
        lib.bsb_tune(b"bs_small", -1)


def test_byteslice_narrow_between_windows():
    """Narrow BETWEEN windows (level-1 inside rows found row by row), windows
    whose bounds share or neighbour their first byte, lo byte 0x00, lo > hi,
    skewed columns with many ties, with and without a mask."""
    rng = np.random.default_rng(321)
    for w, n in ((20, (1 << 19) + 5), (16, 100_003), (24, 65_536), (12, 777)):
        codes = np.minimum(rng.zipf(1.3, size=n) - 1, (1 << w) - 1).astype(np.uint64)
        codes[rng.random(n) < 0.3] = rng.integers(0, 1 << w, size=int((rng.random(n) < 0.3).sum()) or 1,
                                                  dtype=np.uint64)[:1]
        codes ^= rng.integers(0, 1 << w, size=n, dtype=np.uint64) * (rng.random(n) < 0.5)
        col = B.build_byteslice(codes, w)
        planes = O.bs_build(codes, w)
        K = planes.shape[0]
        mw = O.bools_to_words(rng.random(n) < 0.6)
        top = 1 << w
        srt = np.sort(codes)
        wins = [(int(srt[int(q * (n - 1))]), int(srt[int(min(1.0, q + d) * (n - 1))]))
                for q in (0.1, 0.5, 0.9, 0.999) for d in (0.0, 0.0005, 0.01, 0.2)]
        wins += [(0, 5), (0, top - 1), (top - 1, top - 1), (9, 3), (top // 2, top // 2 + 1),
                 (top // 2 - 1, top // 2), ((1 << (w - 8)) * 7, (1 << (w - 8)) * 8)]
        for a, b in wins:
            p = O.pred_between(a, K, b, K)
            for m_o, m_d in ((None, None), (mw, B.ResultBitVector(n, mw))):
                want, _ = O.bs_scan(planes, w, n, p, m_o)
                bv, _ = B.scan_byteslice(col, rp(list(p)), m_d)
                assert np.array_equal(bv.words, want), (w, n, a, b)
                assert bv.count() == O.words_count(want)


def test_byteslice_row_lookup_unsorted_duplicates():
    rng = np.random.default_rng(5)
    n, w = 100_003, 24
    codes = rng.integers(0, 1 << w, size=n, dtype=np.uint64)
    col = B.build_byteslice(codes, w)
    rows = rng.integers(0, n, size=50_000)
    got = B.lookup_byteslice_rows(col, torch.from_numpy(rows)).cpu().numpy()
    assert np.array_equal(got.view(np.uint64), codes[rows])
    # decode through a rank -> value table
    table = torch.from_numpy(rng.integers(-2**40, 2**40, size=1 << w)).cuda()
    vals = B.lookup_byteslice_rows(col, torch.from_numpy(rows), table).cpu().numpy()
    assert np.array_equal(vals, table.cpu().numpy()[codes[rows].astype(np.int64)])


@pytest.mark.parametrize("order", ["keep", "sort"])
def test_row_lookup_out_of_range_ids_raise_index_error(order):
    """An id outside [0, n_rows) is never read: the reference raises
    IndexError at its numpy fancy index (byteslice.py:154, vbs.py:357); the
    device lookups raise it too, or flag it in the async error word."""
    from paper_2209_00220_b200 import _lib
    from paper_2209_00220_b200.device import SORT_GATHER_MIN
    rng = np.random.default_rng(12)
    n = 70_001
    vals, od, codes, lens = _ppe_column(1.1, 16, n, 5)
    col_v = B.build_vbs(codes, lens)
    col_b = B.build_byteslice(codes.astype(np.uint64) & np.uint64(0xFFFF), 16)
    d = B.Dictionary.build(B.build_frequency_table(vals, B.ColumnKind.NUMERIC),
                           "prefix_preserving")
    m = SORT_GATHER_MIN * 2 if order == "sort" else 1000
    for bad in (n, -1, 1 << 40):
        ids = rng.integers(0, n, size=m)
        ids[m // 2] = bad
        t = torch.from_numpy(ids).cuda()
        with pytest.raises(IndexError):
            B.lookup_byteslice_rows(col_b, t, order=order)
        with pytest.raises(IndexError):
            B.lookup_vbs_rows(col_v, t, order=order)
        with pytest.raises(IndexError):
            B.lookup_vbs_rows_dec(col_v, t, d.dev_decoder, order=order)
        err = torch.zeros(1, dtype=torch.int32, device="cuda")
        B.lookup_byteslice_rows(col_b, t, order=order, err=err)
        assert int(err.item()) & _lib.ERR_INDEX
        err.zero_()
        B.lookup_vbs_rows_dec(col_v, t, d.dev_decoder, order=order, err=err)
        assert int(err.item()) & _lib.ERR_INDEX
    # in-range ids leave the word clear
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    ok = torch.from_numpy(rng.integers(0, n, size=m)).cuda()
    B.lookup_vbs_rows(col_v, ok, order=order, err=err)
    assert int(err.item()) == 0


def test_row_lookups_sorted_gather():
    """Long unsorted id lists (>= device.SORT_GATHER_MIN) are gathered in row
    order and scattered back: output in input order, duplicates, both
    layouts, codes and decoded values, and the order="keep" path."""
    from paper_2209_00220_b200.device import SORT_GATHER_MIN
    rng = np.random.default_rng(8)
    n = 300_007
    ids = rng.integers(0, n, size=max(2 * SORT_GATHER_MIN, 150_000))
    ids[:1000] = ids[1000:2000]  # duplicates
    codes = rng.integers(0, 1 << 20, size=n, dtype=np.uint64)
    col = B.build_byteslice(codes, 20)
    for order in ("auto", "keep", "sort"):
        got = B.lookup_byteslice_rows(col, torch.from_numpy(ids), order=order).cpu().numpy()
        assert np.array_equal(got.view(np.uint64), codes[ids]), order
    got = B.lookup_byteslice_rows(col, torch.from_numpy(np.sort(ids))).cpu().numpy()
    assert np.array_equal(got.view(np.uint64), codes[np.sort(ids)])
    for order in ("auto", "keep"):  # int32 codes (sorted gather under "auto")
        got = B.lookup_byteslice_rows(col, torch.from_numpy(ids), out_dtype=torch.int32,
                                      order=order).cpu().numpy()
        assert np.array_equal(got, codes[ids].astype(np.int32)), order
    vals, od, vcodes, lens = _ppe_column(1.1, 16, n, 9)
    vcol = B.build_vbs(vcodes, lens)
    K = vcol.max_len
    padded = vcodes << (np.uint64(8) * (np.uint64(K) - lens.astype(np.uint64)))
    assert K >= 3  # "auto" sorts
    for order in ("auto", "keep"):
        got = B.lookup_vbs_rows(vcol, torch.from_numpy(ids), order=order).cpu().numpy()
        assert np.array_equal(got.view(np.uint64), padded[ids]), order
    d = B.Dictionary.build(B.build_frequency_table(vals, B.ColumnKind.NUMERIC),
                           "prefix_preserving")
    assert np.array_equal(d.row_codes(d.encode_rows(vals))[0], vcodes)
    got = B.lookup_vbs_rows_dec(vcol, torch.from_numpy(ids), d.dev_decoder,
                                out_dtype=torch.int32).cpu().numpy()
    assert np.array_equal(got, vals[ids].astype(np.int32))


@pytest.mark.parametrize("n", [1_500, 70_001, 3_000_017, (1 << 25) + 12_345])
def test_row_lookups_bucket_pairs(n):
    """Row-id lookups through bucket-ordered (row, position) pairs
    (bsb_rows_bucket + *_lookup_pairs): output in input order with duplicates,
    skewed id lists (one hot bucket), one- and two-pass bucket plans, both
    layouts, codes / decoded values, bad ids reported; and the pairs
    themselves are a permutation of (row, position) ordered by bucket."""
    import ctypes

    from paper_2209_00220_b200 import _lib
    from paper_2209_00220_b200.device import (BUCKET_GATHER_MIN, BUCKET_ROWS_MIN, auto_gather,
                                              gather_pairs, stream)
    rng = np.random.default_rng(n)
    m = 200_003 if n < (1 << 25) else (1 << 22) + 3  # the last: the *_auto entry points
    ids = rng.integers(0, n, size=m)
    ids[:1000] = ids[1000:2000]  # duplicates
    ids[5000:60_000] = rng.integers(n // 3, n // 3 + min(n // 4, 900), size=55_000)  # hot bucket
    t = torch.from_numpy(ids).cuda()
    # the pairs: every (row, position) once, buckets ascending
    pairs = torch.empty(m, dtype=torch.int64, device="cuda")
    _lib.check(_lib.load().bsb_rows_bucket(t.data_ptr(), m, n, pairs.data_ptr(), None, stream()),
               "bsb_rows_bucket")
    ph = pairs.cpu().numpy().view(np.uint64)
    prow, ppos = (ph & np.uint64(0xFFFFFFFF)).astype(np.int64), (ph >> np.uint64(32)).astype(np.int64)
    assert np.array_equal(np.sort(ppos), np.arange(m))
    assert np.array_equal(prow, ids[ppos])
    bits = max(1, int(n - 1).bit_length())
    bb = min(13, max(1, bits - 10))
    bucket = np.minimum(prow >> (bits - bb), (1 << bb) - 1)
    assert np.all(np.diff(bucket) >= 0)
    codes = rng.integers(0, 1 << 20, size=n, dtype=np.uint64)
    col = B.build_byteslice(codes, 20)
    got = B.lookup_byteslice_rows(col, t, order="bucket").cpu().numpy()
    assert np.array_equal(got.view(np.uint64), codes[ids])
    got = B.lookup_byteslice_rows(col, t, out_dtype=torch.int32, order="auto").cpu().numpy()
    assert np.array_equal(got, codes[ids].astype(np.int32))
    vals, od, vcodes, lens = _ppe_column(1.1, 16, n, 9)
    vcol = B.build_vbs(vcodes, lens)
    K = vcol.max_len
    padded = vcodes << (np.uint64(8) * (np.uint64(K) - lens.astype(np.uint64)))
    got = B.lookup_vbs_rows(vcol, t, order="bucket").cpu().numpy()
    assert np.array_equal(got.view(np.uint64), padded[ids])
    if n < 100_000:  # the reference-packed deep layout through the pairs as well
        pcol = B.build_vbs(vcodes, lens, deep_mode="packed")
        got = B.lookup_vbs_rows(pcol, t, order="bucket").cpu().numpy()
        assert np.array_equal(got.view(np.uint64), padded[ids])
    d = B.Dictionary.build(B.build_frequency_table(vals, B.ColumnKind.NUMERIC),
                           "prefix_preserving")
    for order in ("bucket", "auto"):
        got = B.lookup_vbs_rows_dec(vcol, t, d.dev_decoder, out_dtype=torch.int32,
                                    order=order).cpu().numpy()
        assert np.array_equal(got, vals[ids].astype(np.int32)), order
    # ascending lists are gathered as given under "auto"; same values
    srt = np.sort(ids)
    got = B.lookup_byteslice_rows(col, torch.from_numpy(srt), order="auto").cpu().numpy()
    assert np.array_equal(got.view(np.uint64), codes[srt])
    got = B.lookup_vbs_rows_dec(vcol, torch.from_numpy(srt), d.dev_decoder, out_dtype=torch.int32,
                                order="auto").cpu().numpy()
    assert np.array_equal(got, vals[srt].astype(np.int32))
    for lst, want in ((ids, 1), (srt, 0)):  # the device-side verdict gates the pair lookups
        tl = torch.from_numpy(lst).cuda()
        pp, uns = gather_pairs(tl, n, check=True)
        assert int(uns.item()) == want
        o32 = torch.empty(m, dtype=torch.int32, device="cuda")
        err = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.check(_lib.load().bsb_byteslice_lookup_pairs(
            col.desc_ref, pp.data_ptr(), tl.data_ptr(), uns.data_ptr(), m, None, None, None,
            o32.data_ptr(), err.data_ptr(), stream()), "lookup_pairs")
        assert np.array_equal(o32.cpu().numpy(), codes[lst].astype(np.int32))
        assert int(err.item()) == 0
    assert auto_gather(m, n) == (m >= BUCKET_GATHER_MIN and n >= BUCKET_ROWS_MIN)
    # bad ids: IndexError / the async error word, through the pairs as well
    for bad in (n, -1, 1 << 40):
        ids2 = ids.copy()
        ids2[m // 2] = bad
        t2 = torch.from_numpy(ids2).cuda()
        with pytest.raises(IndexError):
            B.lookup_byteslice_rows(col, t2, order="bucket")
        err = torch.zeros(1, dtype=torch.int32, device="cuda")
        B.lookup_vbs_rows_dec(vcol, t2, d.dev_decoder, order="bucket", err=err)
        assert int(err.item()) & _lib.ERR_INDEX


def test_bits_to_rows_any_alignment_and_size():
    """Bitvector -> ascending row ids over 16-byte aligned words (super-tiles
    of 4 tiles, 16-byte loads) and over words at a 4-byte offset (the
    one-word-per-lane form), ragged sizes around the 4096-row super-tile, with
    a row offset; and the fused lookup over the same selections."""
    from paper_2209_00220_b200 import _lib
    from paper_2209_00220_b200.device import stream
    lib = _lib.load()
    rng = np.random.default_rng(5)
    for n in (1, 31, 1024, 4095, 4096, 4097, 8192 + 33, 1_000_003):
        for p in (0.0, 0.02, 0.5, 1.0):
            flags = rng.random(n) < p
            want = np.flatnonzero(flags) + 1000
            words = np.zeros((n + 31) // 32 + 1, np.uint32)
            words[1:] = O.bools_to_words(flags)
            buf = torch.from_numpy(words.view(np.int32)).cuda()
            for off in (0, 1):  # off = 1: the data as given, at a 4-byte offset
                if off == 0:
                    w = buf[1:].clone()
                    assert w.data_ptr() % 16 == 0
                else:
                    w = buf[1:]
                    assert w.data_ptr() % 16 == 4
                out = torch.empty(max(len(want), 1), dtype=torch.int64, device="cuda")
                cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
                _lib.check(lib.bsb_bits_to_rows_async(w.data_ptr(), n, 1000, out.data_ptr(),
                                                      cnt.data_ptr(), stream()), "bits_to_rows")
                assert int(cnt.item()) == len(want), (n, p, off)
                assert np.array_equal(out[:len(want)].cpu().numpy(), want), (n, p, off)


def test_rows_bucket_edge_sizes():
    """bsb_rows_bucket at the edges: one id, chunk-size boundaries, a one-row
    column, bucket counts of 2 .. 2^13, an id list that is only 8-byte aligned
    (the first pass then loads its chunks without the bulk copy), all ids in
    one bucket, and ascending lists forced through the pairs."""
    rng = np.random.default_rng(77)
    cases = [(1, 1), (1, 5), (33, 1), (33, 4095), (1024, 4096), (1025, 4097), (5000, 8193),
             (1 << 17, 12_289), (1 << 21, 40_001), ((1 << 23) + 3, 70_001)]
    for n, m in cases:
        codes = rng.integers(0, 1 << 16, size=n, dtype=np.uint64)
        col = B.build_byteslice(codes, 16)
        for kind in ("random", "one_bucket", "ascending", "unaligned"):
            if kind == "one_bucket":
                ids = rng.integers(0, min(n, 700), size=m)
            elif kind == "ascending":
                ids = np.sort(rng.integers(0, n, size=m))
            else:
                ids = rng.integers(0, n, size=m)
            if kind == "unaligned":
                buf = torch.empty(m + 1, dtype=torch.int64, device="cuda")
                t = buf[1:]
                t.copy_(torch.from_numpy(ids))
                assert t.data_ptr() % 16 == 8
            else:
                t = torch.from_numpy(ids).cuda()
            got = B.lookup_byteslice_rows(col, t, order="bucket").cpu().numpy()
            assert np.array_equal(got.view(np.uint64), codes[ids]), (n, m, kind)


def test_row_lookup_auto_is_graph_capturable():
    """The _auto row-id lookup (order verdict on the device, both gathers
    gated on it, no host synchronisation with an error word) captured once as
    a CUDA graph: replays over new random lists and over an ascending one
    return codes[ids] each time."""
    n, m = (1 << 25) + 777, (1 << 22) + 5
    rng = np.random.default_rng(1)
    codes = rng.integers(0, 1 << 20, size=n, dtype=np.uint64)
    col = B.build_byteslice(codes, 20)
    t = torch.from_numpy(rng.integers(0, n, size=m)).cuda()
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        B.lookup_byteslice_rows(col, t, out_dtype=torch.int32, err=err)  # attributes, pools
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            out = B.lookup_byteslice_rows(col, t, out_dtype=torch.int32, err=err)
        for rep in range(3):
            t.copy_(torch.from_numpy(rng.integers(0, n, size=m)) if rep < 2
                    else torch.sort(t).values)
            g.replay()
            torch.cuda.synchronize()
            assert np.array_equal(out.cpu().numpy(),
                                  codes[t.cpu().numpy()].astype(np.int32)), rep
    assert int(err.item()) == 0


def test_byteslice_errors():
    with pytest.raises(ValueError):
        B.build_byteslice([], 8)
    with pytest.raises(ValueError):
        B.build_byteslice([1], 0)
    with pytest.raises(ValueError):
        B.build_byteslice([256], 8)
    with pytest.raises(ValueError):
        B.build_byteslice([1, 2], 8, B.LaneConfig(16))
    col = B.build_byteslice([5, 6], 4)
    with pytest.raises(ValueError):
        B.scan_byteslice(col, ResolvedPredicate.compare(Op.EQ, 5, 1),
                         B.ResultBitVector.zeros(3))
    out, st = B.lookup_byteslice(col, B.ResultBitVector.zeros(2))
    assert out.tolist() == [] and st.total_bytes == 0


# ----------------------------------------------------------------- PP-VBS


@pytest.mark.parametrize("mode", ["packed", "sliced"])
def test_vbs_golden(mode):
    data, meta = load("vbs")
    for ci, m in enumerate(meta):
        col = B.build_vbs(data[f"{ci}/codes"], data[f"{ci}/lens"], deep_mode=mode)
        K = col.max_len
        assert K == m["K"]
        sl = col.slices
        assert np.array_equal(sl[0], data[f"{ci}/bs1"])
        for j in range(2, K + 1):
            assert np.array_equal(sl[j - 1], data[f"{ci}/bs{j}"])
            assert np.array_equal(col.mask_words(j), data[f"{ci}/m{j}"])
        assert np.array_equal(col.block_dir_host, data[f"{ci}/dir"])
        mask = B.ResultBitVector(m["n"], data[f"{ci}/mask"])
        for pi, t in enumerate(m["preds"]):
            for mi, msk in enumerate((None, mask)):
                key = f"{ci}/p{pi}m{mi}/"
                bv, st = B.scan_vbs(col, rp(t), msk)
                want = data[key + "words"]
                assert np.array_equal(bv.words, want), key
                assert bv.count() == O.words_count(want)
                check_stats(st, stats_of(data, key))
        for si in range(3):
            sel = B.ResultBitVector(m["n"], data[f"{ci}/sel{si}"])
            got, lst = B.lookup_vbs(col, sel)
            assert np.array_equal(got, data[f"{ci}/lookup{si}"])
            assert [lst.levels_touched, lst.bytes_loaded, lst.mask_bytes] == \
                data[f"{ci}/lookup_stats{si}"].tolist()


def _ppe_column(s, d, n, seed):
    vals = O.gen_zipf(s, d, n, seed)
    od = O.OracleDict.from_values(vals, "prefix_preserving")
    codes, lens = od.row_codes(od.encode_rows(vals))
    return vals, od, codes, lens


@pytest.mark.parametrize("mode", ["packed", "sliced"])
def test_vbs_zipf_between_windows_vs_oracle(mode):
    """cfg2-shaped (Zipf 1.2 over 2^20, scaled to 2^20 rows), the four
    BETWEEN windows of SURVEY.md §8(d), fused single pass vs oracle legs."""
    n = 1 << 20
    vals, od, codes, lens = _ppe_column(1.2, 20, n, 42)
    col = B.build_vbs(codes, lens, deep_mode=mode)
    ocol = O.vbs_build(codes, lens)
    srt = np.sort(vals)
    q = lambda x: int(srt[min(n - 1, int(x * n))])  # noqa: E731
    for p in (0.001, 0.01, 0.1, 0.5):
        mm = min(p, 0.25)
        opred = od.encode_literal("BETWEEN", q(1 - p - mm), q(1 - mm))
        want, _ = O.vbs_scan(ocol, opred)
        bv, _ = B.scan_vbs(col, rp(list(opred)))
        assert np.array_equal(bv.words, want), p
        assert np.array_equal(O.words_to_bools(want, n),
                              O.naive_filter(vals, "BETWEEN", q(1 - p - mm), q(1 - mm)))


def test_vbs_shallow_rows_settled_by_the_literal():
    """SLICED deep-space scans read no first-slice byte when the literals
    alone settle every 1-byte-code row: a first byte of 255 (a value right of
    every first-level slot: all long codes of a Zipf column) under LE / LT /
    NE matches them all, under GE / GT / EQ / BETWEEN none, and a 1-byte 0 /
    255 literal does the same from the other side.  Every operator, masked
    (sparse and dense) and unmasked, against the oracle and the raw values."""
    n = (1 << 18) + 777
    vals, od, codes, lens = _ppe_column(1.1, 16, n, 3)
    col = B.build_vbs(codes, lens, deep_mode="sliced")
    ocol = O.vbs_build(codes, lens)
    K = ocol.K
    rng = np.random.default_rng(9)
    first = (codes >> (np.uint64(8) * (lens.astype(np.uint64) - np.uint64(1)))) & np.uint64(0xFF)
    right = np.unique(vals[(lens > 1) & (first == 255)])  # long codes right of every slot
    other = np.unique(vals[(lens > 1) & (first != 255)])  # long codes in a gap between slots
    assert len(right) > 100
    lits = [int(right[0]), int(right[len(right) // 2]), int(right[-1]),
            int(vals.min()), int(np.unique(vals[lens == 1]).max())]
    lits += [int(other[len(other) // 2])] if len(other) else []
    masks = [None, O.bools_to_words(rng.random(n) < 0.5), O.bools_to_words(rng.random(n) < 0.01)]
    for v in lits:
        for op in ("EQ", "NE", "LT", "LE", "GT", "GE"):
            opred = od.encode_literal(op, v)
            for m_o in masks:
                want, _ = O.vbs_scan(ocol, opred, m_o)
                bv, _ = B.scan_vbs(col, rp(list(opred)),
                                   None if m_o is None else B.ResultBitVector(n, m_o))
                assert np.array_equal(bv.words, want), (v, op)
            assert np.array_equal(O.words_to_bools(O.vbs_scan(ocol, opred)[0], n),
                                  O.naive_filter(vals, op, v)), (v, op)
    for lo, hi in ((lits[0], lits[1]), (lits[3], lits[2]), (lits[4], lits[1]), (lits[3], lits[4])):
        opred = od.encode_literal("BETWEEN", lo, hi)
        for m_o in masks:
            want, _ = O.vbs_scan(ocol, opred, m_o)
            bv, _ = B.scan_vbs(col, rp(list(opred)),
                               None if m_o is None else B.ResultBitVector(n, m_o))
            assert np.array_equal(bv.words, want), (lo, hi)
    # raw code-space literals: 1-byte 0x00 / 0xFF and a 2-byte 0xFF.. literal
    for lit, ll in ((0, 1), (255, 1), (0xFF00, 2), (0xFFFF, 2)):
        if ll > K:
            continue
        for op in ("EQ", "NE", "LT", "LE", "GT", "GE"):
            p = O.pred_compare(op, lit, ll)
            for m_o in masks[:2]:
                want, _ = O.vbs_scan(ocol, p, m_o)
                bv, _ = B.scan_vbs(col, rp(list(p)),
                                   None if m_o is None else B.ResultBitVector(n, m_o))
                assert np.array_equal(bv.words, want), (lit, ll, op)


@pytest.mark.parametrize("mode", ["packed", "sliced"])
def test_vbs_random_codes_all_ops_masks_vs_oracle(mode):
    rng = np.random.default_rng(77)
    for n, K in ((50_001, 3), (20_000, 8), (3000, 5), (33, 2), (1, 1)):
        lens = rng.integers(1, K + 1, size=n).astype(np.uint8)
        byts = rng.integers(0, 256, size=(n, 8), dtype=np.uint64)
        byts[:, 0] |= np.uint64(1)
        codes = np.zeros(n, np.uint64)
        for k in range(8):
            use = lens > k
            codes[use] |= byts[use, k] << np.uint64(8 * k)
        col = B.build_vbs(codes, lens, deep_mode=mode)
        ocol = O.vbs_build(codes, lens)
        mw = O.bools_to_words(rng.random(n) < 0.5)
        for _ in range(4):
            r = int(rng.integers(0, n))
            lit, ll = int(codes[r]), int(lens[r])
            for op in ("EQ", "NE", "LT", "LE", "GT", "GE"):
                p = O.pred_compare(op, lit, ll)
                for m_o in (None, mw):
                    want, st_w = O.vbs_scan(ocol, p, m_o)
                    bv, st = B.scan_vbs(col, rp(list(p)),
                                        None if m_o is None else B.ResultBitVector(n, m_o))
                    assert np.array_equal(bv.words, want), (n, K, op)
            a, b = sorted(rng.integers(0, n, 2).tolist())
            pa = int(codes[a]) << (8 * (ocol.K - int(lens[a])))
            pb = int(codes[b]) << (8 * (ocol.K - int(lens[b])))
            if pa > pb:
                a, b = b, a
            p = O.pred_between(int(codes[a]), int(lens[a]), int(codes[b]), int(lens[b]))
            want, st_w = O.vbs_scan(ocol, p, mw)
            bv, st = B.scan_vbs(col, rp(list(p)), B.ResultBitVector(n, mw))
            assert np.array_equal(bv.words, want)
            assert st.total_bytes == st_w.total_bytes
            assert st.block_depth.tolist() == st_w.block_depth.tolist()


def test_vbs_sliced_deep_space_scan_vs_oracle():
    """Scans of SLICED columns run in deep-row space (deep[0]), with and
    without input masks.
    Code bytes from a small alphabet with 0x00 / 0xFF (the compare shortcuts)
    and many ties; literals of every length 1..K, present or not; every op and
    BETWEEN with lo/hi bytes in either order below the first level (both the
    shallow-rows-cannot-match variant and the level-1 variant)."""
    rng = np.random.default_rng(2209)
    alpha = np.array([0x00, 0x01, 0x7F, 0x80, 0xFE, 0xFF], dtype=np.uint64)
    for n, K in ((70_001, 2), (50_000, 3), (33_333, 5), (4097, 8), (31, 4)):
        lens = rng.integers(1, K + 1, size=n).astype(np.uint8)
        lens[rng.random(n) < 0.5] = 1  # ~half the rows shallow
        byts = alpha[rng.integers(0, len(alpha), size=(n, 8))]
        byts[:, 0] |= np.uint64(1)
        codes = np.zeros(n, np.uint64)
        for k in range(8):
            use = lens > k
            codes[use] |= byts[use, k] << np.uint64(8 * k)
        col = B.build_vbs(codes, lens, deep_mode="sliced")
        assert col.deep[0] is not None and col._desc.deep1_shared == 0
        ocol = O.vbs_build(codes, lens)

        def lit():
            ll = int(rng.integers(1, K + 1))
            bs = alpha[rng.integers(0, len(alpha), size=ll)]
            bs[-1] |= np.uint64(1)
            return sum(int(b) << (8 * (ll - 1 - i)) for i, b in enumerate(bs)), ll

        # masks: dense, sparse, and whole 32-row blocks / 1024-row tiles masked out
        dense = O.bools_to_words(rng.random(n) < 0.7)
        sparse = O.bools_to_words(rng.random(n) < 0.02)
        holes = O.bools_to_words((np.arange(n) // 1024) % 3 != 1)
        masks = [None, dense, sparse, holes]
        for _ in range(6):
            c, ll = lit()
            for op in ("EQ", "NE", "LT", "LE", "GT", "GE"):
                p = O.pred_compare(op, c, ll)
                for m_o in masks:
                    want, _ = O.vbs_scan(ocol, p, m_o)
                    bv, _ = B.scan_vbs(col, rp(list(p)),
                                       None if m_o is None else B.ResultBitVector(n, m_o))
                    assert np.array_equal(bv.words, want), (n, K, op, hex(c), ll)
                    assert bv.count() == O.words_count(want)
            c2, l2 = lit()
            if K >= 2 and rng.random() < 0.5:  # share the first byte (no level-1 pass)
                c2 = (c >> (8 * (ll - 1)) << (8 * (l2 - 1))) | (c2 & ((1 << (8 * (l2 - 1))) - 1))
            for lo, hi in (((c, ll), (c2, l2)), ((c2, l2), (c, ll))):
                p = O.pred_between(lo[0], lo[1], hi[0], hi[1])
                for m_o in masks:
                    want, _ = O.vbs_scan(ocol, p, m_o)
                    bv, _ = B.scan_vbs(col, rp(list(p)),
                                       None if m_o is None else B.ResultBitVector(n, m_o))
                    assert np.array_equal(bv.words, want), (n, K, hex(lo[0]), hex(hi[0]))
                    assert bv.count() == O.words_count(want)


@pytest.mark.parametrize("x", [0x00, 0x80, 0xFF])
def test_vbs_sliced_zone_map_uniform_first_byte(x):
    """All deep rows share their first byte (PPE's right-most pointer in the
    skewed columns): level 1 of the deep rows is settled from the column's
    zone map.  Literals whose first byte is below, equal to and above it."""
    rng = np.random.default_rng(77 + x)
    n, K = 90_001, 5
    lens = rng.integers(1, K + 1, size=n).astype(np.uint8)
    byts = rng.integers(0, 256, size=(n, 8), dtype=np.uint64)
    byts[:, 0] |= np.uint64(1)
    codes = np.zeros(n, np.uint64)
    for k in range(8):
        use = lens > k
        codes[use] |= byts[use, k] << np.uint64(8 * k)
    deep = lens >= 2
    top = (lens.astype(np.uint64) - np.uint64(1)) * np.uint64(8)
    codes[deep] = (codes[deep] & ~(np.uint64(0xFF) << top[deep])) | (np.uint64(x) << top[deep])
    col = B.build_vbs(codes, lens, deep_mode="sliced")
    assert col.deep1_range == (x, x) and col._desc.deep1_shared == x + 1
    assert col.deep[0] is None  # the zone map makes the level-1 plane unnecessary
    ocol = O.vbs_build(codes, lens)
    mw = O.bools_to_words(rng.random(n) < 0.5)
    for r in rng.integers(0, n, size=8):
        c, ll = int(codes[r]), int(lens[r])
        for fb in {max(x - 1, 0), x, min(x + 1, 255)}:
            c2 = (fb << (8 * (ll - 1))) | (c & ((1 << (8 * (ll - 1))) - 1))
            for op in ("EQ", "NE", "LT", "LE", "GT", "GE"):
                p = O.pred_compare(op, c2, ll)
                for m_o in (None, mw):
                    want, _ = O.vbs_scan(ocol, p, m_o)
                    bv, _ = B.scan_vbs(col, rp(list(p)),
                                       None if m_o is None else B.ResultBitVector(n, m_o))
                    assert np.array_equal(bv.words, want), (x, op, hex(c2), ll)
            if fb == x:  # without the zone map the row-space kernel serves the column
                B.scan_vbs(col, rp(list(O.pred_compare("EQ", c2, ll))))
                lib = B._lib.load()
                assert lib.bsb_tune(b"ds_zonemap", 0) == 0
                try:
                    p = O.pred_compare("GE", c2, ll)
                    want, _ = O.vbs_scan(ocol, p)
                    bv, _ = B.scan_vbs(col, rp(list(p)))
                    assert np.array_equal(bv.words, want), (x, "no zone map")
                finally:
                    lib.bsb_tune(b"ds_zonemap", 1)
            r2 = int(rng.integers(0, n))
            lo, hi = sorted([(c2 << (8 * (K - ll)), c2, ll),
                             (int(codes[r2]) << (8 * (K - int(lens[r2]))), int(codes[r2]),
                              int(lens[r2]))])
            p = O.pred_between(lo[1], lo[2], hi[1], hi[2])
            want, _ = O.vbs_scan(ocol, p)
            bv, _ = B.scan_vbs(col, rp(list(p)))
            assert np.array_equal(bv.words, want), (x, "BETWEEN")


@pytest.mark.parametrize("mode", ["packed", "sliced"])
def test_vbs_row_lookup_decode_vs_oracle(mode):
    n = 200_000
    vals, od, codes, lens = _ppe_column(1.0, 20, n, 4)
    col = B.build_vbs(codes, lens, deep_mode=mode)
    ocol = O.vbs_build(codes, lens)
    rng = np.random.default_rng(6)
    rows = rng.integers(0, n, size=100_000)
    got = B.lookup_vbs_rows(col, torch.from_numpy(rows)).cpu().numpy().view(np.uint64)
    want, _ = O.vbs_lookup(ocol, rows)
    assert np.array_equal(got, want)
    table = B.FrequencyTable(od.values, od.weights, B.ColumnKind.NUMERIC)
    d = B.Dictionary.build(table, "prefix_preserving")
    sp, dv = d.dev_decode
    v = B.lookup_vbs_rows(col, torch.from_numpy(rows), sp, dv).cpu().numpy()
    assert np.array_equal(v, vals[rows])
    v32 = B.lookup_vbs_rows(col, torch.from_numpy(np.sort(rows)), sp, dv,
                            out_dtype=torch.int32).cpu().numpy()
    assert np.array_equal(v32, vals[np.sort(rows)].astype(np.int32))


def _sel_cases(n, rng):
    yield np.zeros(n, bool)
    yield np.ones(n, bool)
    for p in (0.001, 0.05, 0.5):
        yield rng.random(n) < p
    f = np.zeros(n, bool)
    f[-1] = True  # last (ragged) row only
    yield f


@pytest.fixture(params=["one_kernel", "popcount_scan"])
def fused_lookup_form(request):
    """Small columns take the one-kernel cooperative fused lookup; coop_tiles =
    0 forces the tile popcount + scan + lookup sequence of big columns."""
    from paper_2209_00220_b200 import _lib
    lib = _lib.load()
    lib.bsb_tune(b"coop_tiles", 0 if request.param == "popcount_scan" else -1)
    yield request.param
    lib.bsb_tune(b"coop_tiles", -1)


@pytest.mark.parametrize("mode", ["packed", "sliced"])
def test_vbs_fused_bits_lookup_and_tree_decode(mode, fused_lookup_form):
    """bsb_vbs_lookup_bits (bitvector -> codes / values in one kernel) and
    the PPE tree decoder equal the oracle's lookup + the row values."""
    n = 150_001
    vals, od, codes, lens = _ppe_column(1.0, 20, n, 9)
    col = B.build_vbs(codes, lens, deep_mode=mode)
    ocol = O.vbs_build(codes, lens)
    d = B.Dictionary.build(B.FrequencyTable(od.values, od.weights, B.ColumnKind.NUMERIC),
                           "prefix_preserving")
    dec = d.dev_decoder
    assert dec.kind == 3  # ppe_numerical dictionaries decode through the tree
    rng = np.random.default_rng(10)
    for flags in _sel_cases(n, rng):
        rows = np.flatnonzero(flags)
        bv = B.ResultBitVector(n, O.bools_to_words(flags))
        got = B.lookup_vbs_bits(col, bv).cpu().numpy().view(np.uint64)
        want, _ = O.vbs_lookup(ocol, rows)
        assert np.array_equal(got, want)
        v = B.lookup_vbs_bits(col, bv, dec).cpu().numpy()
        assert np.array_equal(v, vals[rows])
        v32 = B.lookup_vbs_bits(col, bv, dec, out_dtype=torch.int32).cpu().numpy()
        assert np.array_equal(v32, vals[rows].astype(np.int32))
    rows = rng.integers(0, n, size=77_777)
    v = B.lookup_vbs_rows_dec(col, torch.from_numpy(rows), dec).cpu().numpy()
    assert np.array_equal(v, vals[rows])
    # random codes up to 8 bytes (deepest stage), ragged row counts
    for n2, K in ((40_003, 8), (1100, 2), (5, 3)):
        lens = rng.integers(1, K + 1, size=n2).astype(np.uint8)
        byts = rng.integers(0, 256, size=(n2, 8), dtype=np.uint64)
        byts[:, 0] |= np.uint64(1)
        codes = np.zeros(n2, np.uint64)
        for k in range(8):
            use = lens > k
            codes[use] |= byts[use, k] << np.uint64(8 * k)
        col = B.build_vbs(codes, lens, deep_mode=mode)
        ocol = O.vbs_build(codes, lens)
        for flags in _sel_cases(n2, rng):
            rows = np.flatnonzero(flags)
            got = B.lookup_vbs_bits(col, B.ResultBitVector(n2, O.bools_to_words(flags)))
            want, _ = O.vbs_lookup(ocol, rows)
            assert np.array_equal(got.cpu().numpy().view(np.uint64), want), (n2, K)


def test_tree_decoder_equals_binary_search_decoder():
    """Decoder kinds 2 (sorted padded codes) and 3 (PPE tree) agree on every
    code of several dictionaries, incl. single-byte-only and deep ones."""
    from paper_2209_00220_b200 import _lib
    for s, dd, n, seed in ((1.0, 8, 5000, 1), (1.2, 20, 300_000, 2), (0.5, 22, 400_000, 3)):
        vals, od, codes, lens = _ppe_column(s, dd, n, seed)
        col = B.build_vbs(codes, lens)
        d = B.Dictionary.build(B.FrequencyTable(od.values, od.weights, B.ColumnKind.NUMERIC),
                               "prefix_preserving")
        rows = torch.arange(n, dtype=torch.int64)
        v3 = B.lookup_vbs_rows_dec(col, rows, d.dev_decoder).cpu().numpy()
        sp, dv = d.dev_decode
        dec2 = _lib.BsbDecode()
        dec2.kind, dec2.values, dec2.sorted_padded, dec2.n_dict = 2, dv.data_ptr(), \
            sp.data_ptr(), sp.numel()
        v2 = B.lookup_vbs_rows_dec(col, rows, dec2).cpu().numpy()
        assert np.array_equal(v3, vals) and np.array_equal(v2, vals)


def test_byteslice_fused_bits_lookup(fused_lookup_form):
    rng = np.random.default_rng(12)
    for n, w in ((70_001, 13), (4096, 24), (33, 40)):
        codes = rng.integers(0, 1 << min(w, 62), n, dtype=np.int64).astype(np.uint64)
        col = B.build_byteslice(codes, w)
        for flags in _sel_cases(n, rng):
            rows = np.flatnonzero(flags)
            bv = B.ResultBitVector(n, O.bools_to_words(flags))
            got = B.lookup_byteslice_bits(col, bv).cpu().numpy().view(np.uint64)
            assert np.array_equal(got, codes[rows]), (n, w)
    # rank-table decode of a fixed dictionary
    vals = rng.integers(-10**9, 10**9, 100_000)
    d = B.Dictionary.build(B.FrequencyTable(*np.unique(vals, return_counts=True),
                                            B.ColumnKind.NUMERIC), "fixed")
    ranks = d.encode_rows(vals)
    col = B.build_byteslice(ranks, d.assignment.width_bits)
    flags = rng.random(len(vals)) < 0.3
    v = B.lookup_byteslice_bits(col, B.ResultBitVector(len(vals), O.bools_to_words(flags)),
                                d.dev_decoder).cpu().numpy()
    assert np.array_equal(v, vals[flags])


def test_vbs_errors(fused_lookup_form):
    col = B.build_vbs([1, 2], [1, 1])
    with pytest.raises(ValueError):
        B.scan_vbs(col, ResolvedPredicate.compare(Op.EQ, 0x0101, 2))
    with pytest.raises(ValueError):
        B.build_vbs([0x1FF], [1])
    with pytest.raises(ValueError):
        B.build_vbs([1], [9])
    with pytest.raises(ValueError):
        B.build_vbs([1, 2], [1])
    # decode of a code the dictionary does not hold -> LookupError
    d = B.Dictionary.build(B.FrequencyTable(np.arange(3), np.array([3, 2, 1]),
                                            B.ColumnKind.NUMERIC), "prefix_preserving")
    bad = B.build_vbs([9], [1])
    sp, dv = d.dev_decode
    with pytest.raises(LookupError):
        B.lookup_vbs_rows(bad, torch.zeros(1, dtype=torch.int64), sp, dv)
    with pytest.raises(LookupError):
        B.lookup_vbs_rows_dec(bad, torch.zeros(1, dtype=torch.int64), d.dev_decoder)
    with pytest.raises(LookupError):
        B.lookup_vbs_bits(bad, B.ResultBitVector(1, np.ones(1, np.uint32)), d.dev_decoder)
    fx = B.Dictionary.build(B.FrequencyTable(np.arange(3), np.array([3, 2, 1]),
                                             B.ColumnKind.NUMERIC), "fixed")
    bcol = B.build_byteslice(np.array([1, 5], np.int64), 8)
    with pytest.raises(LookupError):
        B.lookup_byteslice_bits(bcol, B.ResultBitVector(2, np.array([3], np.uint32)),
                                fx.dev_decoder)


# --------------------------------------------- encoders, advisor, engine


def test_freq_table_and_encode_rows_vs_oracle():
    rng = np.random.default_rng(8)
    for vals in (O.gen_zipf(1.2, 20, 1 << 20, 42), rng.integers(-10**12, 10**12, 50_000),
                 rng.integers(-3, 3, 1000), np.array([7]), np.arange(70_000)[::-1].copy()):
        t = B.build_frequency_table(vals, B.ColumnKind.NUMERIC)
        u, c = O.freq_table(vals)
        assert np.array_equal(t.values, u) and np.array_equal(t.weights, c)
        d = B.Dictionary.build(t, "fixed")
        assert np.array_equal(d.encode_rows(vals), np.searchsorted(u, vals))
    with pytest.raises(KeyError):
        d.encode_rows(np.array([123456789]))


def test_advisor_bytes_mode_matches_reference():
    data, meta = load("advisor")
    for i, m in enumerate(meta):
        a = B.advise_column("c", data[f"{i}/values"], B.ColumnKind.NUMERIC,
                            count=m["count"], cost="bytes", subsample=m["subsample"])
        assert a.chosen == m["chosen"]
        assert a.auc_byteslice == m["auc_bs"] and a.auc_ppvbs == m["auc_vbs"]
        assert [(p.selectivity, p.time) for p in a.points_byteslice] == \
            [tuple(x) for x in data[f"{i}/pts_bs"].tolist()]
        assert [(p.selectivity, p.time) for p in a.points_ppvbs] == \
            [tuple(x) for x in data[f"{i}/pts_vbs"].tolist()]


def test_advisor_wall_mode_picks_and_tie():
    rng = np.random.default_rng(9)
    uni = rng.integers(0, 1 << 12, size=1 << 20, dtype=np.int64)
    sk = B.gen_zipf(B.ZipfSpec(1.5, 12, 1 << 20, seed=9))
    assert B.advise_column("u", uni, B.ColumnKind.NUMERIC, count=20, cost="bytes").chosen \
        == "byteslice"
    assert B.advise_column("z", sk, B.ColumnKind.NUMERIC, count=20, cost="bytes").chosen \
        == "ppvbs"
    tie = B.advise_column("t", uni[:4096], B.ColumnKind.NUMERIC, count=5,
                          cost=lambda run: 1.0)
    assert tie.chosen == "byteslice"
    w = B.advise_column("u", uni, B.ColumnKind.NUMERIC, count=10, cost="wall")
    assert w.auc_byteslice > 0 and w.auc_ppvbs > 0
    deg = B.advise_column("c", np.zeros(100, np.int64), B.ColumnKind.NUMERIC)
    assert deg.degenerate and deg.chosen == "byteslice"


def test_fixture_query_192_through_engine():
    f, _ = load("fixture")
    schema = E.Schema([E.ColumnSpec("qty", B.ColumnKind.NUMERIC, "byteslice"),
                       E.ColumnSpec("amount", B.ColumnKind.NUMERIC, "ppvbs")])
    store, _ = E.ingest_arrays({"qty": f["qty"], "amount": f["amount"]}, schema,
                               policy="forced")
    q = E.execute(store, E.Query.conjunction(
        [Predicate("amount", Op.LE, 4), Predicate("qty", Op.GT, 50)], ["amount", "qty"]))
    assert q.n_selected == 192
    assert np.array_equal(q.selection.words, f["selection"])
    assert np.array_equal(q.columns["amount"], f["proj_amount"])
    assert np.array_equal(q.columns["qty"], f["proj_qty"])


def test_conjunction_call_equals_pipelined_oracle():
    rng = np.random.default_rng(10)
    n = 300_007
    cols = {"u16": rng.integers(0, 1 << 16, n), "z12": O.gen_zipf(1.0, 12, n, 11),
            "u24": rng.integers(0, 1 << 24, n), "z16": O.gen_zipf(1.5, 16, n, 12)}
    layouts = {"u16": "byteslice", "z12": "ppvbs", "u24": "byteslice", "z16": "ppvbs"}
    schema = E.Schema([E.ColumnSpec(k, B.ColumnKind.NUMERIC, v) for k, v in layouts.items()])
    store, _ = E.ingest_arrays(cols, schema, policy="forced")
    srt = {k: np.sort(v) for k, v in cols.items()}
    qq = lambda k, x: int(srt[k][min(n - 1, int(x * n))])  # noqa: E731
    preds = [Predicate("u16", Op.LT, 32768),
             Predicate("z12", Op.BETWEEN, qq("z12", 0.2), qq("z12", 0.9)),
             Predicate("u24", Op.GE, qq("u24", 0.6)), Predicate("z16", Op.LE, qq("z16", 0.7))]
    res = E.execute(store, E.Query([preds, [Predicate("u16", Op.EQ, 5)]], ["u24", "z12"]))
    want = np.ones(n, bool)
    for p in preds:
        want &= O.naive_filter(cols[p.column], p.op.name, p.value, p.value_high)
    want |= cols["u16"] == 5
    assert np.array_equal(res.selection.to_bools(), want)
    assert res.n_selected == int(want.sum())
    assert np.array_equal(res.columns["u24"], cols["u24"][want])
    assert np.array_equal(res.columns["z12"], cols["z12"][want])


@pytest.mark.parametrize("mode", ["packed", "sliced"])
def test_conj_scan_mask_trivial_and_long_chains(mode):
    """bsb_conj_scan == the pipelined oracle for chains longer than
    BSB_MAX_CONJ, constant predicates inside the chain and an input mask."""
    rng = np.random.default_rng(21)
    n = 70_001
    vals, od, codes, lens = _ppe_column(1.1, 16, n, 22)
    col_v = B.build_vbs(codes, lens, deep_mode=mode)
    ocol = O.vbs_build(codes, lens)
    u = rng.integers(0, 1 << 12, n)
    col_b = B.build_byteslice(u, 12)
    planes = O.bs_build(u, 12)
    srt = np.sort(vals)
    mw = O.bools_to_words(rng.random(n) < 0.7)
    chain, opreds = [], []
    for i in range(11):
        if i % 5 == 4:
            t = bool(i % 2)
            chain.append((("ppvbs", col_v), ResolvedPredicate.constant(t)))
            opreds.append(("v", O.pred_const(t)))
        elif i % 2:
            lo, hi = sorted(int(x) for x in rng.choice(srt, 2))
            p = od.encode_literal("BETWEEN", lo, hi)
            chain.append((("ppvbs", col_v), rp(list(p))))
            opreds.append(("v", p))
        else:
            c = int(rng.integers(0, 1 << 12))
            chain.append((("byteslice", col_b), ResolvedPredicate.compare(Op.GE, c, 2)))
            opreds.append(("b", O.pred_compare("GE", c, 2)))
    got = E.conj_scan([c for c, _ in chain], [p for _, p in chain], B.ResultBitVector(n, mw))
    want = mw
    for kind, p in opreds:
        want = (O.vbs_scan(ocol, p, want)[0] if kind == "v"
                else O.bs_scan(planes, 12, n, p, want)[0])
    assert np.array_equal(got.words, want)
    assert got.count() == O.words_count(want)


@pytest.mark.parametrize("ppm,cfg", [(0, 0), (50_000, 0), (1_000_000, 0), (1_000_000, 1),
                                     (1_000_000, 2), (1_000_000, 3)])
def test_conj_chain_masked_and_epilogue_kernels_vs_oracle(ppm, cfg):
    """Masked PP-VBS scans inside bsb_conj_scan: with sparse_ppm = 10^6 every
    gated scan runs the compacted kernel (work over the masked-in blocks
    only; every shape dsm_cfg selects), with 0 it scans the column whole and
    ANDs the mask into the words (EPI kernel); both equal the pipelined
    oracle for random 1..8-byte codes (SLICED columns with and without the
    first-byte zone map), every operator, literals of every length and
    sparse / dense running masks."""
    lib = B._lib.load()
    rng = np.random.default_rng(91)
    assert lib.bsb_tune(b"sparse_ppm", ppm) == 0
    assert lib.bsb_tune(b"dsm_cfg", cfg) == 0
    try:
        for n, K, shared in ((70_001, 5, False), (40_000, 8, True), (3000, 3, False)):
            lens = rng.integers(1, K + 1, size=n).astype(np.uint8)
            byts = rng.integers(0, 256, size=(n, 8), dtype=np.uint64)
            byts[:, 0] |= np.uint64(1)
            codes = np.zeros(n, np.uint64)
            for k in range(8):
                use = lens > k
                codes[use] |= byts[use, k] << np.uint64(8 * k)
            if shared:  # every deep row starts with 0xFF (zone map)
                top = (lens >= 2)
                codes[top] = (codes[top] & ~(np.uint64(0xFF) << (np.uint64(8) * (
                    lens[top].astype(np.uint64) - np.uint64(1))))) | (
                    np.uint64(0xFF) << (np.uint64(8) * (lens[top].astype(np.uint64) -
                                                        np.uint64(1))))
            col = B.build_vbs(codes, lens, deep_mode="sliced")
            ocol = O.vbs_build(codes, lens)
            u = rng.integers(0, 1 << 16, n)
            col_b = B.build_byteslice(u, 16)
            planes = O.bs_build(u, 16)
            for sel in (0.005, 0.3):
                c = int((1 << 16) * sel)
                pb = O.pred_compare("LT", c, 2)
                first, _ = O.bs_scan(planes, 16, n, pb)
                for _ in range(3):
                    r = int(rng.integers(0, n))
                    lit, ll = int(codes[r]), int(lens[r])
                    for op in ("EQ", "NE", "LT", "LE", "GT", "GE"):
                        p = O.pred_compare(op, lit, ll)
                        want, _ = O.vbs_scan(ocol, p, first)
                        got = E.conj_scan([("byteslice", col_b), ("ppvbs", col)],
                                          [rp(list(pb)), rp(list(p))])
                        assert np.array_equal(got.words, want), (n, K, op, sel)
                        assert got.count() == O.words_count(want)
                    a, b = sorted(rng.integers(0, n, 2).tolist())
                    pa = int(codes[a]) << (8 * (ocol.K - int(lens[a])))
                    pz = int(codes[b]) << (8 * (ocol.K - int(lens[b])))
                    if pa > pz:
                        a, b = b, a
                    p = O.pred_between(int(codes[a]), int(lens[a]), int(codes[b]), int(lens[b]))
                    want, _ = O.vbs_scan(ocol, p, first)
                    got = E.conj_scan([("byteslice", col_b), ("ppvbs", col)],
                                      [rp(list(pb)), rp(list(p))])
                    assert np.array_equal(got.words, want), (n, K, "BETWEEN", sel)
    finally:
        lib.bsb_tune(b"sparse_ppm", -1)
        lib.bsb_tune(b"dsm_cfg", -1)


@pytest.mark.parametrize("cfg", [0, 1, 2, 3])
def test_masked_sliced_scans_compacted_and_epi_vs_oracle(cfg):
    """Public masked scan_vbs on SLICED columns: the sampled mask density
    gates the compacted kernel (sparse masks) against EPI (dense masks);
    ds_masked=1 forces EPI.  Masks of 0.1 % .. 50 % density, masks with
    empty and full stretches, ragged column ends, every operator and
    BETWEEN: words, counts equal the oracle."""
    lib = B._lib.load()
    rng = np.random.default_rng(400 + cfg)
    assert lib.bsb_tune(b"dsm_cfg", cfg) == 0
    try:
        for n, K in ((300_007, 4), (1 << 17, 6), (40_001, 2)):
            lens = rng.integers(1, K + 1, size=n).astype(np.uint8)
            byts = rng.integers(0, 256, size=(n, 8), dtype=np.uint64)
            byts[:, 0] |= np.uint64(1)
            codes = np.zeros(n, np.uint64)
            for k in range(8):
                use = lens > k
                codes[use] |= byts[use, k] << np.uint64(8 * k)
            col = B.build_vbs(codes, lens, deep_mode="sliced")
            ocol = O.vbs_build(codes, lens)
            masks = []
            for dens in (0.001, 0.03, 0.5):
                masks.append(rng.random(n) < dens)
            stretch = np.zeros(n, bool)
            stretch[n // 3: n // 3 + 5000] = True
            stretch[-37:] = True
            masks.append(stretch)
            for mb in masks:
                mw = O.bools_to_words(mb)
                r = int(rng.integers(0, n))
                lit, ll = int(codes[r]), int(lens[r])
                preds = [O.pred_compare(op, lit, ll) for op in ("EQ", "NE", "LT", "GE")]
                a, b = sorted(rng.integers(0, n, 2).tolist())
                pa = int(codes[a]) << (8 * (ocol.K - int(lens[a])))
                pz = int(codes[b]) << (8 * (ocol.K - int(lens[b])))
                if pa > pz:
                    a, b = b, a
                preds.append(O.pred_between(int(codes[a]), int(lens[a]), int(codes[b]),
                                            int(lens[b])))
                for p in preds:
                    want, _ = O.vbs_scan(ocol, p, mw)
                    for forced_epi in (0, 1):
                        lib.bsb_tune(b"ds_masked", forced_epi)
                        bv, _ = B.scan_vbs(col, rp(list(p)), B.ResultBitVector(n, mw))
                        assert np.array_equal(bv.words, want), (n, K, p[0], forced_epi)
                        assert bv.count() == O.words_count(want)
    finally:
        lib.bsb_tune(b"ds_masked", -1)
        lib.bsb_tune(b"dsm_cfg", -1)


@pytest.mark.parametrize("n", [1, 1000, 70_001, 1 << 20])
def test_fused_byteslice_pairs_vs_oracle(n):
    """bsb_conj_scan runs consecutive ByteSlice predicates as one fused
    kernel (TMA-staged level-1 sectors, AND in registers): the words equal
    the pipelined oracle for every operator, BETWEEN, columns of different
    widths (1..4 slices), ragged row counts, with and without an input
    mask, and equal the unfused chain (bsb_tune conj_fuse=0)."""
    lib = B._lib.load()
    rng = np.random.default_rng(n)
    ws = (8, 12, 20, 32)
    cols, planes, vals = [], [], []
    for w in ws:
        v = rng.integers(0, 1 << w, n, dtype=np.uint64)
        vals.append(v)
        cols.append(B.build_byteslice(v, w))
        planes.append(O.bs_build(v, w))
    mw = O.bools_to_words(rng.random(n) < 0.6)
    for trial in range(6):
        i, j = rng.choice(4, 2, replace=False)
        chain, opreds = [], []
        for c in (i, j):
            v = vals[c]
            a, b = sorted(int(x) for x in rng.choice(v, 2))
            if trial % 3 == 0:
                p = O.pred_between(a, 1, b, 1)
            else:
                p = O.pred_compare(("LT", "GE", "EQ", "NE", "LE", "GT")[trial], a, 1)
            chain.append((("byteslice", cols[c]), rp(list(p))))
            opreds.append((c, p))
        for m in (None, mw):
            want = m
            for c, p in opreds:
                want, _ = O.bs_scan(planes[c], ws[c], n, p, want)
            got = E.conj_scan([x for x, _ in chain], [p for _, p in chain],
                              None if m is None else B.ResultBitVector(n, m))
            assert np.array_equal(got.words, want), (n, trial, m is None)
            assert got.count() == O.words_count(want)
            assert lib.bsb_tune(b"conj_fuse", 0) == 0
            try:
                unf = E.conj_scan([x for x, _ in chain], [p for _, p in chain],
                                  None if m is None else B.ResultBitVector(n, m))
            finally:
                lib.bsb_tune(b"conj_fuse", 1)
            assert np.array_equal(unf.words, want)


def _same_stats(st, o):
    assert st.levels == o.levels
    assert st.blocks_total == o.blocks_total
    assert st.blocks_skipped == o.blocks_skipped
    assert list(st.words_loaded) == list(o.words_loaded)
    assert list(st.bytes_loaded) == list(o.bytes_loaded)
    assert st.mask_bytes == o.mask_bytes
    assert st.block_depth.tolist() == o.block_depth.tolist()


@pytest.mark.parametrize("rows_kernel", [0, 1])
def test_sliced_scan_stats_deep_space_vs_oracle(rows_kernel):
    """ScanStats of SLICED PP-VBS scans (the deep-space stats kernel, and the
    row-parallel one with bsb_tune stats_rows=1) == the oracle's for every
    operator, BETWEEN (two pipelined legs: leg 2 counts rows passing GE(lo)),
    input masks, zone-mapped and deep[0] columns, literals of every length;
    the result words equal the plain scan's."""
    lib = B._lib.load()
    rng = np.random.default_rng(33)
    assert lib.bsb_tune(b"stats_rows", rows_kernel) == 0
    try:
        cases = []
        vals, od, codes, lens = _ppe_column(1.2, 16, 50_003, 7)     # zone map
        cases.append((codes, lens))
        for n, K in ((40_001, 5), (3000, 8), (70, 3)):              # deep[0]
            lens = rng.integers(1, K + 1, size=n).astype(np.uint8)
            byts = rng.integers(0, 256, size=(n, 8), dtype=np.uint64)
            byts[:, 0] |= np.uint64(1)
            codes = np.zeros(n, np.uint64)
            for k in range(8):
                use = lens > k
                codes[use] |= byts[use, k] << np.uint64(8 * k)
            cases.append((codes, lens))
        for codes, lens in cases:
            n = len(codes)
            col = B.build_vbs(codes, lens, deep_mode="sliced")
            ocol = O.vbs_build(codes, lens)
            mw = O.bools_to_words(rng.random(n) < 0.4)
            for _ in range(3):
                r = int(rng.integers(0, n))
                lit, ll = int(codes[r]), int(lens[r])
                for op in ("EQ", "NE", "LT", "LE", "GT", "GE"):
                    p = O.pred_compare(op, lit, ll)
                    for m_o in (None, mw):
                        want, ost = O.vbs_scan(ocol, p, m_o)
                        bv, st = B.scan_vbs(col, rp(list(p)),
                                            None if m_o is None else B.ResultBitVector(n, m_o))
                        _same_stats(st.materialize(), ost)
                        assert np.array_equal(bv.words, want), op
                a, b = sorted(rng.integers(0, n, 2).tolist())
                pa = int(codes[a]) << (8 * (ocol.K - int(lens[a])))
                pz = int(codes[b]) << (8 * (ocol.K - int(lens[b])))
                if pa > pz:
                    a, b = b, a
                p = O.pred_between(int(codes[a]), int(lens[a]), int(codes[b]), int(lens[b]))
                for m_o in (None, mw):
                    want, ost = O.vbs_scan(ocol, p, m_o)
                    bv, st = B.scan_vbs(col, rp(list(p)),
                                        None if m_o is None else B.ResultBitVector(n, m_o))
                    _same_stats(st.materialize(), ost)
                    assert np.array_equal(bv.words, want)
    finally:
        lib.bsb_tune(b"stats_rows", 0)


def test_device_bitvector_ops():
    rng = np.random.default_rng(12)
    for n in (1, 31, 32, 33, 1000, 100_001):
        a = B.ResultBitVector.from_bools(rng.random(n) < 0.3)
        b = B.ResultBitVector.from_bools(rng.random(n) < 0.6)
        da, db = a.to_device(), b.to_device()
        assert (da & db) == (a & b) and (da | db) == (a | b) and (~da) == (~a)
        assert da.count() == a.count()
        assert np.array_equal(da.to_indices(), a.to_indices())
        assert np.array_equal(da.row_ids(5).cpu().numpy(), a.to_indices() + 5)


def test_row_range_shards_concatenate_to_the_full_scan():
    """SURVEY.md §8(e) on one GPU: each tile-aligned row-range shard built and
    scanned on its own (global dictionary, as every rank does) -- ByteSlice
    and PP-VBS through the deep-row-space kernel, with and without masks --
    concatenates to the full column's words, and the shard counts' exclusive
    prefix gives each shard's first global match."""
    from paper_2209_00220_b200.sharded import shard_range
    n = (1 << 20) + 777
    vals, od, codes, lens = _ppe_column(1.2, 18, n, 5)
    of = O.OracleDict.from_values(vals, "fixed")
    ranks = of.encode_rows(vals)
    w = max(1, int(ranks.max()).bit_length())
    full_v = B.build_vbs(codes, lens)
    full_b = B.build_byteslice(ranks, w)
    srt = np.sort(vals)
    mw = O.bools_to_words(np.random.default_rng(1).random(n) < 0.4)
    for p in (0.001, 0.1, 0.5):
        lo, hi = int(srt[int((1 - p - min(p, .25)) * n)]), int(srt[int((1 - min(p, .25)) * n)])
        pv = od.encode_literal("BETWEEN", lo, hi)
        rb = of.encode_literal("BETWEEN", lo, hi)
        for masked in (False, True):
            m_full = B.ResultBitVector(n, mw) if masked else None
            want_v, _ = B.scan_vbs(full_v, rp(list(pv)), m_full)
            want_b, _ = B.scan_byteslice(full_b, rp(list(rb)), m_full)
            assert np.array_equal(want_v.words, want_b.words)
            for world in (2, 3, 8):
                parts, counts = [], []
                for rank in range(world):
                    r0, r1 = shard_range(n, world, rank)
                    if r1 <= r0:
                        continue
                    col = B.build_vbs(codes[r0:r1], lens[r0:r1])
                    m = (B.ResultBitVector(r1 - r0, O.bools_to_words(
                        O.words_to_bools(mw, n)[r0:r1])) if masked else None)
                    bv, _ = B.scan_vbs(col, rp(list(pv)), m)
                    parts.append(O.words_to_bools(bv.words, r1 - r0))
                    counts.append(bv.count())
                got = np.concatenate(parts)
                assert np.array_equal(got, O.words_to_bools(want_v.words, n)), (p, world)
                assert sum(counts) == want_v.count()
                offs = np.concatenate([[0], np.cumsum(counts)[:-1]])
                first = np.flatnonzero(got)
                r0s = [shard_range(n, world, r)[0] for r in range(len(counts))]
                for k, c in enumerate(counts):
                    if c:
                        assert first[offs[k]] >= r0s[k]


@pytest.mark.parametrize("tiles", [0, 1, 4])
def test_vbs_sliced_all_rows_deep(tiles):
    """Every code has >= 2 bytes: a 1-tile super-tile spans up to 33 deep
    blocks (the deep-block pass runs twice), and forced 4-tile super-tiles up
    to 129; unaligned deep-row bases; every op, BETWEEN, masks."""
    rng = np.random.default_rng(31 + tiles)
    lib = B._lib.load()
    n, K = 70_003, 4
    lens = rng.integers(2, K + 1, size=n).astype(np.uint8)
    byts = rng.integers(0, 256, size=(n, 8), dtype=np.uint64)
    byts[:, 0] |= np.uint64(1)
    byts[:, 1] &= np.uint64(3)  # few distinct second bytes: many ties
    codes = np.zeros(n, np.uint64)
    for k in range(8):
        use = lens > k
        codes[use] |= byts[use, k] << np.uint64(8 * k)
    col = B.build_vbs(codes, lens, deep_mode="sliced")
    ocol = O.vbs_build(codes, lens)
    mw = O.bools_to_words(rng.random(n) < 0.3)
    assert lib.bsb_tune(b"ds_tiles", tiles) == 0
    try:
        for r in rng.integers(0, n, size=5):
            c, ll = int(codes[r]), int(lens[r])
            for op in ("EQ", "NE", "LT", "LE", "GT", "GE"):
                p = O.pred_compare(op, c, ll)
                for m_o in (None, mw):
                    want, _ = O.vbs_scan(ocol, p, m_o)
                    bv, _ = B.scan_vbs(col, rp(list(p)),
                                       None if m_o is None else B.ResultBitVector(n, m_o))
                    assert np.array_equal(bv.words, want), (tiles, op)
            r2 = int(rng.integers(0, n))
            a, b = sorted([(int(codes[r]) << (8 * (K - ll)), c, ll),
                           (int(codes[r2]) << (8 * (K - int(lens[r2]))), int(codes[r2]),
                            int(lens[r2]))])
            p = O.pred_between(a[1], a[2], b[1], b[2])
            for m_o in (None, mw):
                want, _ = O.vbs_scan(ocol, p, m_o)
                bv, _ = B.scan_vbs(col, rp(list(p)),
                                   None if m_o is None else B.ResultBitVector(n, m_o))
                assert np.array_equal(bv.words, want), (tiles, "BETWEEN")
    finally:
        lib.bsb_tune(b"ds_tiles", 0)
