"""BYST store parity against files written by the reference itself
(tests/golden/make_golden_store.py): dictionary sections from the host
encoders (CPU), and on the GPU the whole file from ingest_arrays + device
layouts, plus reading the reference's files into device layouts."""

import json
import os
import struct

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


def _golden():
    z = np.load(os.path.join(GOLD, "store.npz"))
    cols = {k[4:]: z[k] for k in z.files if k.startswith("col/")}
    return cols, json.loads(str(z["meta"]))


def _sections(buf: bytes) -> dict:
    assert buf[:4] == b"BYST" and struct.unpack_from("<I", buf, 4)[0] == 1
    off, out = 8, {}
    while off < len(buf):
        (nl,) = struct.unpack_from("<I", buf, off)
        name = buf[off + 4: off + 4 + nl].decode()
        (pl,) = struct.unpack_from("<Q", buf, off + 4 + nl)
        out[name] = buf[off + 12 + nl: off + 12 + nl + pl]
        off += 12 + nl + pl
    return out


def test_store_dictionary_sections_match_reference_bytes():
    """Host encoders (np.unique table + fixed / native ppe_numerical) produce
    the reference's dictionary sections byte for byte."""
    from paper_2209_00220_b200.dictionary import ColumnKind, Dictionary, FrequencyTable
    from paper_2209_00220_b200.store import _dict_payload, _parse_dict
    cols, meta = _golden()
    for case in meta:
        secs = _sections(open(os.path.join(GOLD, f"store_{case}.byst"), "rb").read())
        manifest = json.loads(secs["manifest"])
        for e in manifest["columns"]:
            v = cols[e["name"]]
            u, c = np.unique(v, return_counts=True)
            d = Dictionary.build(FrequencyTable(u, c, ColumnKind.NUMERIC), e["scheme"])
            want = secs[f"col:{e['name']}:dict"]
            assert _dict_payload(d) == want, (case, e["name"])
            back = _parse_dict(want)
            assert np.array_equal(back.table.values, u)
            assert np.array_equal(back.assignment.codes, d.assignment.codes)
            assert np.array_equal(back.assignment.lengths, d.assignment.lengths)


def test_store_rejects_bad_files(tmp_path):
    from paper_2209_00220_b200.store import read_store
    p = tmp_path / "x.byst"
    p.write_bytes(b"NOPE" + b"\0" * 8)
    with pytest.raises(ValueError):
        read_store(p)
    p.write_bytes(b"BYST" + struct.pack("<I", 2))
    with pytest.raises(ValueError):
        read_store(p)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["forced", "advised"])
def test_store_write_equals_reference_bytes(case):
    import paper_2209_00220_b200 as B
    from paper_2209_00220_b200 import engine as E
    from paper_2209_00220_b200.store import store_bytes
    cols, meta = _golden()
    m = meta[case]
    names = list(m["layouts"])
    schema = E.Schema([E.ColumnSpec(k, B.ColumnKind.NUMERIC, m["layouts"][k]) for k in names])
    store, _ = E.ingest_arrays({k: cols[k] for k in names}, schema, policy=m["policy"],
                               advise_cost="bytes", advise_count=m["advise_count"])
    want = open(os.path.join(GOLD, f"store_{case}.byst"), "rb").read()
    got = store_bytes(store)
    gs, ws = _sections(got), _sections(want)
    assert list(gs) == list(ws)
    for k in ws:
        assert gs[k] == ws[k], k
    assert got == want


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["forced", "advised"])
def test_store_read_reference_file_scans_and_lookups(case, tmp_path):
    import paper_2209_00220_b200 as B
    from paper_2209_00220_b200 import engine as E
    from paper_2209_00220_b200.predicate import Op, Predicate
    from paper_2209_00220_b200.store import read_store, store_bytes, write_store
    import oracle as O
    cols, meta = _golden()
    path = os.path.join(GOLD, f"store_{case}.byst")
    store = read_store(path)
    assert store.n_rows == len(next(iter(cols.values())))
    # round trip: reading then writing gives the same bytes
    out = tmp_path / "rt.byst"
    write_store(out, store)
    assert out.read_bytes() == open(path, "rb").read()
    rng = np.random.default_rng(31)
    for name, v in cols.items():
        srt = np.sort(v)
        lo, hi = sorted(int(x) for x in rng.choice(srt, 2))
        for p in (Predicate(name, Op.BETWEEN, lo, hi), Predicate(name, Op.LT, hi),
                  Predicate(name, Op.GE, lo), Predicate(name, Op.EQ, int(v[5]))):
            res = E.execute(store, E.Query([[p]], [name]))
            want = O.naive_filter(v, p.op.name, p.value, p.value_high)
            assert res.n_selected == int(want.sum()), (case, name, p)
            assert np.array_equal(res.columns[name], v[want]), (case, name, p)


# ------------------------------------------------ categorical / ordered strings
def _strings():
    z = np.load(os.path.join(GOLD, "strings.npz"))
    return z, json.loads(str(z["meta"]))


_STR_KINDS = {"cat_a": "categorical", "cat_b": "categorical", "ostr": "ordered_string",
              "num": "numeric"}


def test_string_dictionaries_match_reference():
    """ppe_categorical (Alg. 2), frequency tables (categorical: count desc,
    first appearance) and literal resolution equal the reference's."""
    from paper_2209_00220_b200.dictionary import (ColumnKind, Dictionary,
                                                  build_frequency_table, ppe_categorical)
    from paper_2209_00220_b200.predicate import Op, Predicate
    z, meta = _strings()
    for i, n in enumerate(meta["ppecat_sizes"]):
        a = ppe_categorical(n)
        assert np.array_equal(a.codes, z[f"ppecat/{i}/codes"]), n
        assert np.array_equal(a.lengths, z[f"ppecat/{i}/lengths"]), n
    for k in ("cat_a", "cat_b", "ostr"):
        kind = ColumnKind(_STR_KINDS[k])
        t = build_frequency_table(z[f"col/{k}"], kind)
        assert np.array_equal(t.values.astype(str), z[f"table/{k}/values"])
        assert np.array_equal(t.weights, z[f"table/{k}/weights"])
        for scheme in ("fixed", "prefix_preserving"):
            d = Dictionary.build(t, scheme)
            for v, op, rop, code, length, triv in meta["literals"][f"{k}/{scheme}"]:
                r = d.encode_literal(Predicate(k, Op[op], v))
                assert [r.op.name if r.op else None, r.code, r.length, r.trivial] == \
                    [rop, code, length, triv], (k, scheme, v, op)
        # the host dictionary sections of the reference's store files
        for case in meta["cases"]:
            secs = _sections(open(os.path.join(GOLD, f"strings_{case}.byst"), "rb").read())
            e = {c["name"]: c for c in json.loads(secs["manifest"])["columns"]}[k]
            from paper_2209_00220_b200.store import _dict_payload
            assert _dict_payload(Dictionary.build(t, e["scheme"])) == secs[f"col:{k}:dict"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["forced", "advised"])
def test_string_store_and_queries_match_reference(case, tmp_path):
    """ingest_arrays of string + numeric columns writes the reference's store
    bytes (advisor included); reading the reference's file and running the
    reference's queries gives its selections and projected values."""
    import paper_2209_00220_b200 as B
    from paper_2209_00220_b200 import engine as E
    from paper_2209_00220_b200.predicate import Op, Predicate
    from paper_2209_00220_b200.store import read_store, store_bytes
    z, meta = _strings()
    m = meta["cases"][case]
    names = list(_STR_KINDS)
    cols = {k: z[f"col/{k}"] for k in names}
    schema = E.Schema([E.ColumnSpec(k, B.ColumnKind(_STR_KINDS[k]), m["layouts"][k])
                       for k in names])
    store, _ = E.ingest_arrays(cols, schema, policy=m["policy"], advise_cost="bytes",
                               advise_count=m["advise_count"])
    want = open(os.path.join(GOLD, f"strings_{case}.byst"), "rb").read()
    gs, ws = _sections(store_bytes(store)), _sections(want)
    for k in ws:
        assert gs[k] == ws[k], k
    loaded = read_store(os.path.join(GOLD, f"strings_{case}.byst"))
    ca, so = cols["cat_a"], np.sort(cols["ostr"])
    u, c = np.unique(ca, return_counts=True)
    top, rare = str(u[np.argmax(c)]), str(u[np.argmin(c)])
    queries = [
        [[Predicate("cat_a", Op.EQ, top)]],
        [[Predicate("cat_a", Op.NE, rare), Predicate("cat_b", Op.EQ, str(cols["cat_b"][7]))]],
        [[Predicate("cat_a", Op.EQ, "absent")], [Predicate("cat_b", Op.NE, "absent")]],
        [[Predicate("ostr", Op.BETWEEN, str(so[300]), str(so[1500]))]],
        [[Predicate("ostr", Op.LT, "s00005"), Predicate("num", Op.GE, 0)]],
        [[Predicate("ostr", Op.GE, "s00100"), Predicate("cat_b", Op.EQ, str(cols["cat_b"][3]))]],
    ]
    for st in (store, loaded):
        for qi, groups in enumerate(queries):
            res = E.execute(st, E.Query(groups, ["cat_a", "ostr", "num"]))
            assert res.n_selected == m["n_selected"][qi], (case, qi)
            assert np.array_equal(res.selection.to_bools(), z[f"q/{case}/{qi}/sel"])
            for c in ("cat_a", "ostr"):
                assert np.array_equal(np.asarray(res.columns[c]).astype(str),
                                      z[f"q/{case}/{qi}/{c}"]), (case, qi, c)
            assert np.array_equal(res.columns["num"], z[f"q/{case}/{qi}/num"])


def test_schema_parse_kind():
    import paper_2209_00220_b200 as B
    from paper_2209_00220_b200 import engine as E
    assert E.Schema.parse_kind("semi_categorical_string") is B.ColumnKind.ORDERED_STRING
    with pytest.raises(ValueError):
        E.Schema.parse_kind("float")

