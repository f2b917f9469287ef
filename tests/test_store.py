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
