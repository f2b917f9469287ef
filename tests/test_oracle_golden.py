"""Pin the CPU oracle against the reference: golden vectors + known answers.

The golden fixtures were produced by running the reference package itself
(tests/golden/make_golden.py).  The worked examples below restate the
reference test-suite's known-answer values (file:line cited per test).
"""

import json

import numpy as np
import pytest

import oracle as O
from golden_io import load, stats_of


def _pred(t):
    op, code, length, code2, length2, trivial = t
    if trivial is not None:
        return O.pred_const(trivial)
    if op == "BETWEEN":
        return O.pred_between(code, length, code2, length2)
    return O.pred_compare(op, code, length)


def _check_stats(st, want):
    assert st.words_loaded.tolist() == want["words_loaded"].tolist()
    assert st.bytes_loaded.tolist() == want["bytes_loaded"].tolist()
    assert st.block_depth.tolist() == want["block_depth"].tolist()
    assert st.levels == want["levels"]
    assert st.blocks_total == want["blocks_total"]
    assert st.blocks_skipped == want["blocks_skipped"]
    assert st.mask_bytes == want["mask_bytes"]
    assert st.total_bytes == want["total_bytes"]


# --- bit kernels: tests/test_bits.py:12-27 + golden pdep/pext -----------------


def test_bit_kernel_worked_examples():
    assert O.pdep(0b1011, 0b11010010) == 0b10010010
    assert O.pext(0b10010010, 0b11010010) == 0b1011
    x = 0b01010010
    assert O.erase_rightmost(x) == 0b01010000
    assert O.propagate_rightmost(x, 8) == 0b11111100
    assert O.lowest_set_index(x, 8) == 1
    with pytest.raises(ValueError):
        O.lowest_set_index(0)


def test_bit_kernels_golden():
    d = np.load(__import__("golden_io").GOLDEN + "/bits.npz")["pdep_pext"]
    for src, mask, dep, ext in d.tolist():
        assert O.pdep(src, mask) == dep
        assert O.pext(src, mask) == ext


# --- bitvector layout: tests/test_bitvector.py:15-30 -------------------------


def test_bitvector_lsb_first():
    w = O.bools_to_words(np.isin(np.arange(40), [0, 33]))
    assert w.tolist() == [1, 2]
    assert O.words_to_rows(w, 40).tolist() == [0, 33]
    assert O.valid_words(33).tolist() == [0xFFFFFFFF, 1]


# --- datagen ------------------------------------------------------------------


def test_zipf_golden():
    data, meta = load("zipf")
    for i, m in enumerate(meta):
        got = O.gen_zipf(m["s"], m["d"], m["n"], m["seed"])
        assert np.array_equal(got, data[f"{i}/values"])


# --- dictionary: tests/test_dictionary.py:63-110, 320-382 + golden ------------


def test_ppe_known_answers():
    c, l = O.ppe_numerical([5, 4, 3])
    assert c.tolist() == [1, 2, 3] and l.tolist() == [1, 1, 1]
    c, l = O.ppe_numerical(np.arange(300, 0, -1))
    assert c[:255].tolist() == list(range(1, 256))
    assert c[255:].tolist() == [(255 << 8) + 1 + i for i in range(45)]
    assert l[255:].tolist() == [2] * 45
    c, l = O.ppe_numerical(np.ones(70000, np.int64))
    assert (l == 1).sum() == 255 and (l == 2).sum() == 255 and (l == 5).sum() == 69490


def test_ppe_golden():
    data, _ = load("dict")
    for i in range(int(data["n_ppe"])):
        c, l = O.ppe_numerical(data[f"ppe{i}/weights"])
        assert np.array_equal(c, data[f"ppe{i}/codes"]), i
        assert np.array_equal(l, data[f"ppe{i}/lengths"]), i


def test_fixed_widths_golden():
    data, _ = load("dict")
    for n, w in data["fixed_widths"].tolist():
        assert O.fixed_assignment(n)[2] == w


def test_literal_resolution_and_decode_golden():
    data, _ = load("dict")
    res = json.loads(str(data["resolution"]))
    for k, block in enumerate(res):
        d = O.OracleDict.from_values(data[f"res{k}/values"], block["scheme"])
        for op, lo, hi, *want in block["cases"]:
            got = d.encode_literal(op, lo, hi)
            assert list(got) == want, (k, op, lo, hi)
        if f"res{k}/padded" in data:
            assert np.array_equal(d.padded, data[f"res{k}/padded"])
            assert np.array_equal(d.decode_padded(d.padded), data[f"res{k}/decoded"])


def test_decode_errors():
    d = O.OracleDict(np.arange(300), np.arange(300, 0, -1), "prefix_preserving")
    assert d.decode_padded([0xFF01])[0] == 255
    assert d.decode_padded([0x0100])[0] == 0
    with pytest.raises(LookupError):
        d.decode_padded([0x0000])
    with pytest.raises(LookupError):
        d.decode_padded([0xFFFF])


# --- ByteSlice: tests/test_byteslice.py:28-45 + golden -----------------------


def test_byteslice_alignment_known_answer():
    p = O.bs_build([0b10000001101], 11)
    assert p[0][0] == 0b10000001 and p[1][0] == 0b10100000
    codes = [0b10000001101, 0, 2047, 1024]
    got, st = O.bs_lookup(O.bs_build(codes, 11), 11, np.arange(4))
    assert got.tolist() == codes and st.bytes_loaded == 8


def test_byteslice_golden():
    data, meta = load("bs")
    for ci, m in enumerate(meta):
        codes = data[f"{ci}/codes"]
        planes = O.bs_build(codes, m["w"])
        assert np.array_equal(planes, data[f"{ci}/slices"])
        mask = data[f"{ci}/mask"]
        for pi, t in enumerate(m["preds"]):
            for mi, msk in enumerate((None, mask)):
                key = f"{ci}/p{pi}m{mi}/"
                words, st = O.bs_scan(planes, m["w"], m["n"], _pred(t), msk)
                assert np.array_equal(words, data[key + "words"]), key
                _check_stats(st, stats_of(data, key))
        rows = O.words_to_rows(data[f"{ci}/sel"], m["n"])
        got, lst = O.bs_lookup(planes, m["w"], rows)
        assert np.array_equal(got, data[f"{ci}/lookup"])
        assert [lst.levels_touched, lst.bytes_loaded, lst.mask_bytes] == \
            data[f"{ci}/lookup_stats"].tolist()


def test_byteslice_threads_identical():
    data, meta = load("bs")
    ci = len(meta) - 1
    planes = O.bs_build(data[f"{ci}/codes"], 11)
    p = O.pred_compare("GE", 1024, 2)
    a, sa = O.bs_scan(planes, 11, meta[ci]["n"], p, threads=1)
    b, sb = O.bs_scan(planes, 11, meta[ci]["n"], p, threads=4)
    assert np.array_equal(a, b)
    assert sa.bytes_loaded.tolist() == sb.bytes_loaded.tolist()
    assert sa.block_depth.tolist() == sb.block_depth.tolist()


# --- PP-VBS: tests/test_vbs.py:37-153, test_acceptance.py:276-303 + golden ----


def test_vbs_worked_examples():
    col = O.vbs_build([0x81, 0xC0, 0x77A9, 0x8189], [1, 1, 2, 2])
    w, st = O.vbs_scan(col, O.pred_compare("GT", 0x81, 1))
    assert O.words_to_rows(w, 4).tolist() == [1, 3]
    assert st.bytes_loaded.tolist() == [32, 0] and st.block_depth.tolist() == [1]
    assert st.mask_bytes == 4
    w, st = O.vbs_scan(col, O.pred_compare("GT", 0x8050, 2))
    assert O.words_to_rows(w, 4).tolist() == [0, 1, 3]
    assert st.block_depth.tolist() == [1]
    w, _ = O.vbs_scan(col, O.pred_compare("EQ", 0xC0, 1))
    assert O.words_to_rows(w, 4).tolist() == [1]
    w, st = O.vbs_scan(col, O.pred_compare("GT", 0x8150, 2))
    assert O.words_to_rows(w, 4).tolist() == [1, 3] and st.block_depth.tolist() == [2]
    got, lst = O.vbs_lookup(col, [2, 3])
    assert got.tolist() == [0x77A9, 0x8189] and lst.bytes_loaded == 4
    got, lst = O.vbs_lookup(col, [0])
    assert got.tolist() == [0x8100] and lst.bytes_loaded == 1
    # existence word (tests/test_vbs.py:52-55)
    lens = [1, 2, 1, 1, 1, 2, 1, 1]
    c = O.vbs_build([0x0101 if x == 2 else 0x01 for x in lens], lens)
    assert int(c.exist[0][0]) == 0x22
    # 56-byte block (tests/test_vbs.py:71-80)
    lens = [3] * 6 + [2] * 4 + [1] * 22
    rep = O.vbs_size_report(O.vbs_build([0x010101] * 6 + [0x0101] * 4 + [1] * 22, lens))
    assert rep["slice_bytes"] == [32, 10, 6] and rep["mask_bytes"] == 8
    assert rep["avg_bits_per_code"] == 14.0


def test_vbs_golden():
    data, meta = load("vbs")
    for ci, m in enumerate(meta):
        col = O.vbs_build(data[f"{ci}/codes"], data[f"{ci}/lens"])
        assert col.K == m["K"]
        assert np.array_equal(col.slices[0], data[f"{ci}/bs1"])
        for j in range(2, col.K + 1):
            assert np.array_equal(col.slices[j - 1], data[f"{ci}/bs{j}"])
            assert np.array_equal(col.exist[j - 2], data[f"{ci}/m{j}"])
        assert np.array_equal(col.block_dir, data[f"{ci}/dir"])
        mask = data[f"{ci}/mask"]
        for pi, t in enumerate(m["preds"]):
            for mi, msk in enumerate((None, mask)):
                key = f"{ci}/p{pi}m{mi}/"
                words, st = O.vbs_scan(col, _pred(t), msk)
                assert np.array_equal(words, data[key + "words"]), key
                _check_stats(st, stats_of(data, key))
                if m["n"] <= 1000:
                    w2, st2 = O.vbs_scan_serial(col, _pred(t), msk)
                    assert np.array_equal(w2, words)
                    _check_stats(st2, stats_of(data, key))
        for si in range(3):
            sel = data[f"{ci}/sel{si}"]
            got, lst = O.vbs_lookup(col, O.words_to_rows(sel, m["n"]))
            assert np.array_equal(got, data[f"{ci}/lookup{si}"])
            assert [lst.levels_touched, lst.bytes_loaded] == \
                data[f"{ci}/lookup_stats{si}"][:2].tolist()
            if m["n"] <= 1000:
                assert np.array_equal(O.vbs_lookup_serial(col, sel), got)


def test_vbs_threads_identical():
    data, meta = load("vbs")
    ci = 5
    col = O.vbs_build(data[f"{ci}/codes"], data[f"{ci}/lens"])
    for t in meta[ci]["preds"][:12]:
        a, sa = O.vbs_scan(col, _pred(t), threads=1)
        b, sb = O.vbs_scan(col, _pred(t), threads=4)
        assert np.array_equal(a, b)
        assert sa.block_depth.tolist() == sb.block_depth.tolist()


def test_literal_longer_than_column_rejected():
    col = O.vbs_build([1, 2], [1, 1])
    with pytest.raises(ValueError):
        O.vbs_scan(col, O.pred_compare("EQ", 0x0101, 2))


# --- advisor: tests/test_advisor.py:43-92 + golden ---------------------------


def test_auc_rules():
    assert O.auc([(0, 3.0), (1, 3.0)]) == pytest.approx(3.0)
    assert O.auc([(0, 0.0), (1, 2.0)]) == pytest.approx(1.0)
    with pytest.raises(ValueError):
        O.auc([(0, 1.0)])


def test_advisor_golden():
    data, meta = load("advisor")
    for i, m in enumerate(meta):
        a = O.advise_column(data[f"{i}/values"], count=m["count"], cost="bytes",
                            subsample=m["subsample"])
        assert a["chosen"] == m["chosen"]
        assert a["auc_byteslice"] == m["auc_bs"]
        assert a["auc_ppvbs"] == m["auc_vbs"]
        assert np.array_equal(np.array(a["points_byteslice"]), data[f"{i}/pts_bs"])
        assert np.array_equal(np.array(a["points_ppvbs"]), data[f"{i}/pts_vbs"])


def test_advisor_tie_goes_to_byteslice():
    a = O.advise_column(np.arange(1000) % 7, count=5, cost=lambda run: 1.0)
    assert a["chosen"] == "byteslice" and a["auc_byteslice"] == a["auc_ppvbs"]


# --- end-to-end pinned query (tests/test_acceptance.py:459-466) ---------------


def test_fixture_conjunction_192():
    f, _ = load("fixture")
    qty, amount = f["qty"], f["amount"]
    n = len(qty)
    d_amt = O.OracleDict.from_values(amount, "prefix_preserving")
    d_qty = O.OracleDict.from_values(qty, "fixed")
    col = O.vbs_build(*d_amt.row_codes(d_amt.encode_rows(amount)))
    planes = O.bs_build(d_qty.encode_rows(qty), d_qty.width_bits)
    w1, _ = O.vbs_scan(col, d_amt.encode_literal("LE", 4))
    w2, _ = O.bs_scan(planes, d_qty.width_bits, n, d_qty.encode_literal("GT", 50), w1)
    assert O.words_count(w2) == 192 == int(f["n_selected"])
    assert np.array_equal(w2, f["selection"])
    rows = O.words_to_rows(w2, n)
    assert np.array_equal(d_amt.decode_padded(O.vbs_lookup(col, rows)[0]), f["proj_amount"])
