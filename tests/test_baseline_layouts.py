"""Baseline layouts (Bit-Packed, VBP, PE-VBP) against
vectors produced by the reference itself (tests/golden/make_golden_baseline.py):
prefix-free codes on the host (CPU), packed streams / planes, scans with
ScanStats, lookups and a five-layout store file on the GPU."""

import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


def _g():
    z = np.load(os.path.join(GOLD, "baseline.npz"))
    return z, json.loads(str(z["meta"]))


def _rp(t):
    from paper_2209_00220_b200.predicate import Op, ResolvedPredicate
    op, code, length, code2, length2, trivial = t
    if trivial is not None:
        return ResolvedPredicate.constant(trivial)
    if op == "BETWEEN":
        return ResolvedPredicate.between(code, length, code2, length2)
    return ResolvedPredicate.compare(Op[op], code, length)


def test_prefix_free_assignment_matches_reference():
    from paper_2209_00220_b200.dictionary import prefix_free_assignment
    z, meta = _g()
    for i in range(len(meta["prefix_free"])):
        a = prefix_free_assignment(z[f"pf{i}/weights"])
        assert np.array_equal(a.codes, z[f"pf{i}/codes"]), i
        assert np.array_equal(a.lengths, z[f"pf{i}/lengths"]), i
        assert a.width_bits == int(z[f"pf{i}/width"])


def _check_stats(st, z, key):
    assert st.levels == int(z[key + "/levels"])
    assert st.blocks_total == int(z[key + "/blocks_total"])
    assert st.blocks_skipped == int(z[key + "/blocks_skipped"])
    assert list(st.words_loaded) == z[key + "/words_loaded"].tolist()
    assert list(st.bytes_loaded) == z[key + "/bytes_loaded"].tolist()
    assert st.total_bytes == int(z[key + "/total_bytes"])
    assert st.block_depth.tolist() == z[key + "/block_depth"].tolist()


@pytest.mark.gpu
def test_bitpacked_and_vbp_scans_lookups_vs_reference():
    import paper_2209_00220_b200 as B
    from paper_2209_00220_b200.bitpacked import build_bitpacked, lookup_bitpacked, scan_bitpacked
    from paper_2209_00220_b200.vbp import build_vbp, lookup_vbp, scan_vbp
    z, meta = _g()
    for ci, case in enumerate(meta["cases"]):
        n, w = case["n"], case["w"]
        codes = z[f"c{ci}/codes"]
        bp = build_bitpacked(codes, w)
        vb = build_vbp(codes, w, "plain")
        assert np.array_equal(bp.bits, z[f"c{ci}/bits"]), ci
        assert np.array_equal(vb.planes, z[f"c{ci}/planes"]), ci
        mask = B.ResultBitVector(n, z[f"c{ci}/mask"])
        for pi, t in enumerate(case["preds"]):
            p = _rp(t)
            for mi, m in enumerate((None, mask)):
                key = f"c{ci}/p{pi}/m{mi}"
                r1 = scan_bitpacked(bp, p, m)
                assert np.array_equal(r1.words, z[key + "/bp"]), (ci, t, mi)
                assert r1.count() == int(np.bitwise_count(z[key + "/bp"]).sum())
                r2, st = scan_vbp(vb, p, m)
                assert np.array_equal(r2.words, z[key + "/vbp"]), (ci, t, mi)
                _check_stats(st, z, key + "/st")
        sel = B.ResultBitVector(n, z[f"c{ci}/sel"])
        assert np.array_equal(lookup_bitpacked(bp, sel), z[f"c{ci}/lookup_bp"])
        assert np.array_equal(lookup_vbp(vb, sel)[0], z[f"c{ci}/lookup_vbp"])


@pytest.mark.gpu
def test_pevbp_scans_and_decode_vs_reference():
    import paper_2209_00220_b200 as B
    from paper_2209_00220_b200 import engine as E
    z, meta = _g()
    for i, pf in enumerate(meta["prefix_free"]):
        v = z[f"pf{i}/values"]
        schema = E.Schema([E.ColumnSpec("c", B.ColumnKind.NUMERIC, "pevbp")])
        store, _ = E.ingest_arrays({"c": v}, schema, policy="forced")
        st = store.columns["c"]
        assert np.array_equal(st.column.planes, z[f"pf{i}/planes"]), i
        for k, t in enumerate(pf["preds"]):
            bv, stats = E.scan_layout("pevbp", st.column, _rp(t))
            assert np.array_equal(bv.words, z[f"pf{i}/q{k}/words"]), (i, k)
            _check_stats(stats, z, f"pf{i}/q{k}/st")
            assert np.array_equal(E.lookup_decode(st, bv), z[f"pf{i}/q{k}/decoded"])


@pytest.mark.gpu
def test_five_layout_store_and_query_vs_reference(tmp_path):
    import paper_2209_00220_b200 as B
    from paper_2209_00220_b200 import engine as E
    from paper_2209_00220_b200.predicate import Op, Predicate
    from paper_2209_00220_b200.store import read_store, store_bytes
    z, meta = _g()
    lay = meta["store_layouts"]
    cols = {k: z[f"store/col/{k}"] for k in lay}
    schema = E.Schema([E.ColumnSpec(k, B.ColumnKind.NUMERIC, lay[k]) for k in lay])
    store, _ = E.ingest_arrays(cols, schema, policy="forced")
    want = open(os.path.join(GOLD, "baseline_store.byst"), "rb").read()
    assert store_bytes(store) == want
    loaded = read_store(os.path.join(GOLD, "baseline_store.byst"))
    sb = np.sort(cols["b"])
    q = [[Predicate("a", Op.LT, 2500), Predicate("b", Op.BETWEEN, int(sb[300]), int(sb[2000])),
          Predicate("c", Op.NE, 0)], [Predicate("d", Op.EQ, int(cols["d"][0]))]]
    for st in (store, loaded):
        res = E.execute(st, E.Query(q, list(cols)))
        assert np.array_equal(res.selection.to_bools(), z["store/sel"])
        for k in cols:
            assert np.array_equal(res.columns[k], z[f"store/proj/{k}"]), k
