"""Bit-exact parity at BASELINE.json's full sizes.

The reference's own check is ``naive_filter`` over the raw values
(tests/helpers.py:35-52; grid at tests/test_acceptance.py:74-140).  At 2^24
to 2^31+ rows the CPU oracle would take minutes, so the same filter runs on
the device (torch) and is packed into bitvector words; every scan's words
must equal it word for word, and every lookup must return exactly the raw
values of its rows.  cfg5 (4 x 2^32 rows) is checked segment by segment by
bench.py before it is timed (bench_cfg5.check_parity); here the same code
runs on a reduced table.
"""

import numpy as np
import pytest
import torch

from devcheck import pack_bools

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2209_00220_b200 as B  # noqa: E402
from paper_2209_00220_b200 import engine as E  # noqa: E402
from paper_2209_00220_b200.predicate import Op, Predicate, ResolvedPredicate  # noqa: E402

N = 1 << 28


def _q(values, weights, n, x):
    cum = np.cumsum(weights)
    return int(values[np.searchsorted(cum, min(n - 1, int(x * n)), side="right")])


@pytest.fixture(scope="module")
def cfg2():
    vals = B.gen_zipf_device(B.ZipfSpec(1.2, 20, N, 42))
    schema = E.Schema([E.ColumnSpec("v", B.ColumnKind.NUMERIC, "ppvbs"),
                       E.ColumnSpec("w", B.ColumnKind.NUMERIC, "byteslice")])
    store, _ = E.ingest_arrays({"v": vals, "w": vals}, schema, policy="forced")
    return vals, store


def test_cfg2_windows_bit_exact_vs_raw_filter(cfg2):
    """cfg2 (2^28 rows, Zipf 1.2 / 2^20): the four BETWEEN windows on both
    layouts == packed device filter of the raw values, word for word; GE and
    LE legs likewise; lookups of the 0.1% / 1% selections == raw values."""
    vals, store = cfg2
    t = store.columns["v"].dictionary.table
    for p in (0.001, 0.01, 0.1, 0.5):
        m = min(p, 0.25)
        lo, hi = _q(t.values, t.weights, N, 1 - p - m), _q(t.values, t.weights, N, 1 - m)
        want = pack_bools((vals >= lo) & (vals <= hi))
        want_ge = pack_bools(vals >= lo)
        want_le = pack_bools(vals <= hi)
        for name in ("v", "w"):
            st = store.columns[name]
            d = st.dictionary
            bv, _ = E.scan_layout(st.layout, st.column,
                                  d.encode_literal(Predicate(name, Op.BETWEEN, lo, hi)))
            assert torch.equal(bv.dwords, want), (name, p)
            ge, _ = E.scan_layout(st.layout, st.column, d.encode_literal(Predicate(name, Op.GE, lo)))
            le, _ = E.scan_layout(st.layout, st.column, d.encode_literal(Predicate(name, Op.LE, hi)))
            assert torch.equal(ge.dwords, want_ge), (name, p, "GE")
            assert torch.equal(le.dwords, want_le), (name, p, "LE")
            if p <= 0.01:
                got = E.lookup_decode_bits(st, bv)
                rows = torch.nonzero((vals >= lo) & (vals <= hi)).flatten()
                assert torch.equal(got, vals[rows]), (name, p)


def test_cfg1_lt_scan_and_lookup_bit_exact():
    """cfg1: 2^24 uniform 16-bit codes, ByteSlice w=16, LT 6554 (10%): words
    == filter, fused lookup == the matching codes in row order."""
    n = 1 << 24
    codes = torch.from_numpy(np.random.default_rng(1).integers(0, 65536, n)).cuda()
    col = B.build_byteslice(codes, 16)
    bv, _ = B.scan_byteslice(col, ResolvedPredicate.compare(Op.LT, 6554, 2))
    flags = codes < 6554
    assert torch.equal(bv.dwords, pack_bools(flags))
    got = B.lookup_byteslice_bits(col, bv)
    assert torch.equal(got.to(torch.int64), codes[flags])


@pytest.fixture(scope="module")
def cfg3():
    n = N
    codes = torch.from_numpy(np.random.default_rng(3).integers(0, 1 << 24, n)).cuda()
    col_b = B.build_byteslice(codes, 24)
    vals = B.gen_zipf_device(B.ZipfSpec(1.0, 20, n, seed=4))
    from paper_2209_00220_b200.dictionary import freq_table_and_ranks
    u, c, ranks = freq_table_and_ranks(vals)
    d = B.Dictionary.build(B.FrequencyTable(u.cpu().numpy(), c.cpu().numpy(),
                                            B.ColumnKind.NUMERIC), "prefix_preserving")
    cv, lv = d.row_codes_device(ranks)
    col_v = B.build_vbs(cv, lv)
    del cv, lv, ranks
    return codes, col_b, vals, col_v, d


def test_cfg3_lookups_return_raw_values(cfg3):
    """cfg3 (2^28 rows): 2^24 random row ids (unsorted with duplicates, and
    sorted) and 1% / 20% bitvectors -> int32 values == raw values, ByteSlice
    (identity codes) and PP-VBS (decoded through the PPE tree)."""
    codes, col_b, vals, col_v, d = cfg3
    ids = torch.from_numpy(np.random.default_rng(5).integers(0, N, N >> 4)).cuda()
    for rows in (ids, torch.sort(ids).values):
        got_b = B.lookup_byteslice_rows(col_b, rows, out_dtype=torch.int32)
        assert torch.equal(got_b.to(torch.int64), codes[rows])
        got_v = B.lookup_vbs_rows_dec(col_v, rows, d.dev_decoder, out_dtype=torch.int32)
        assert torch.equal(got_v.to(torch.int64), vals[rows])
    g = torch.Generator(device="cuda").manual_seed(6)
    for p in (0.01, 0.20):
        flags = torch.rand(N, device="cuda", generator=g) < p
        sel = B.DeviceBitVector(N, pack_bools(flags))
        got_b = B.lookup_byteslice_bits(col_b, sel)
        assert torch.equal(got_b.to(torch.int64), codes[flags]), p
        got_v = B.lookup_vbs_bits(col_v, sel, d.dev_decoder, out_dtype=torch.int32)
        assert torch.equal(got_v.to(torch.int64), vals[flags]), p


def test_cfg4_conjunction_projections_and_sum():
    """cfg4 (2^27 rows): u16 < 32768 AND z12 BETWEEN q(.2),q(.9) AND
    u24 >= q(.6) AND z16 <= q(.7) in one conj_scan over mixed layouts ==
    filter words; projections u32 / z24 / u20 == raw values of the selected
    rows; SUM(u32) == the int64 sum of the raw values."""
    n = 1 << 27
    rng = {nm: np.random.default_rng(100 + i) for i, nm in enumerate(
        ("u16", "u24", "u20", "u32"))}
    raw = {"u16": rng["u16"].integers(0, 1 << 16, n), "u24": rng["u24"].integers(0, 1 << 24, n),
           "u20": rng["u20"].integers(0, 1 << 20, n),
           "u32": rng["u32"].integers(-(1 << 31), 1 << 31, n)}
    raw = {k: torch.from_numpy(v).cuda() for k, v in raw.items()}
    raw["z12"] = B.gen_zipf_device(B.ZipfSpec(1.0, 12, n, 109))
    raw["z16"] = B.gen_zipf_device(B.ZipfSpec(1.5, 16, n, 110))
    raw["z24"] = B.gen_zipf_device(B.ZipfSpec(1.0, 24, n, 112))
    layouts = {"u16": "byteslice", "z12": "ppvbs", "u24": "byteslice", "z16": "ppvbs",
               "u32": "byteslice", "z24": "ppvbs", "u20": "byteslice"}
    schema = E.Schema([E.ColumnSpec(k, B.ColumnKind.NUMERIC, v) for k, v in layouts.items()])
    store, _ = E.ingest_arrays({k: raw[k] for k in layouts}, schema, policy="forced")

    def q(nm, x):
        t = store.columns[nm].dictionary.table
        return _q(t.values, t.weights, n, x)
    preds = [Predicate("u16", Op.LT, 32768),
             Predicate("z12", Op.BETWEEN, q("z12", 0.2), q("z12", 0.9)),
             Predicate("u24", Op.GE, q("u24", 0.6)),
             Predicate("z16", Op.LE, q("z16", 0.7))]
    flags = ((raw["u16"] < 32768) & (raw["z12"] >= preds[1].value)
             & (raw["z12"] <= preds[1].value_high) & (raw["u24"] >= preds[2].value)
             & (raw["z16"] <= preds[3].value))
    stored = [store.columns[p.column] for p in preds]
    sel = E.conj_scan([(s.layout, s.column) for s in stored],
                      [s.dictionary.encode_literal(p) for s, p in zip(stored, preds)])
    assert torch.equal(sel.dwords, pack_bools(flags))
    for nm in ("u32", "z24", "u20"):
        got = E.lookup_decode_bits(store.columns[nm], sel)
        assert torch.equal(got, raw[nm][flags]), nm
    got_sum = int(E.lookup_decode_bits(store.columns["u32"], sel).sum().item())
    assert got_sum == int(raw["u32"][flags].sum().item())
    res = E.execute(store, E.Query([preds], ["u20"]))
    assert res.n_selected == int(flags.sum().item())


def test_cfg5_sharded_table_reduced_segments():
    """bench_cfg5 on 8 segments of 2^22 rows (the cfg5 generators, global
    dictionaries, quantiles and predicates): every segment's bitvector of
    every query == the packed raw filter, the AND's compacted global row ids
    == filter rows + segment start (check_parity raises otherwise), and the
    shards of 2 and 4 ranks reproduce the 1-rank segments."""
    import bench_cfg5 as C
    tab = C.Cfg5Table(1, 0, 1 << 22)
    step = C.Cfg5Step(tab, 1)
    step.run_query("and4", torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    step.ids = torch.empty(max(1, int(step.counts[4].sum().item())), dtype=torch.int64,
                           device="cuda")
    sel = C.check_parity(tab, step)
    assert sel["and4"] > 0 and sel["u0"] > 0
    from paper_2209_00220_b200.sharded import owned_segments
    assert [list(owned_segments(8, 4, r)) for r in range(4)] == [[0, 1], [2, 3], [4, 5], [6, 7]]


def test_rows_beyond_int32_range():
    """A column of 2^31 + 12345 rows (one byte plane, and a PP-VBS column of
    1- and 2-byte codes): scan words == filter past row 2^31, compaction
    emits ids >= 2^31, row-id lookups of ids >= 2^31 return the codes."""
    free, _ = torch.cuda.mem_get_info()
    if free < 60e9:
        pytest.skip("needs ~60 GB of free device memory")
    n = (1 << 31) + 12345
    codes = torch.empty(n, dtype=torch.int64, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(9)
    for i in range(0, n, 1 << 28):
        codes[i:i + (1 << 28)] = torch.randint(0, 256, (min(1 << 28, n - i),), device="cuda",
                                               generator=g)
    col = B.build_byteslice(codes, 8)
    bv, _ = B.scan_byteslice(col, ResolvedPredicate.compare(Op.GE, 250, 1))
    flags = codes >= 250
    assert torch.equal(bv.dwords, pack_bools(flags))
    tail = torch.arange(n - 5000, n, device="cuda")
    assert torch.equal(B.lookup_byteslice_rows(col, tail).to(torch.int64), codes[tail])
    ids = bv.row_ids()
    assert ids.numel() == int(flags.sum().item())
    assert torch.equal(ids[-100:], torch.nonzero(flags).flatten()[-100:])
    del col, bv, ids
    lens = (codes >= 200).to(torch.uint8) + 1           # 1- or 2-byte codes
    vcodes = torch.where(lens == 2, (codes << 8) | 7, codes)
    vcol = B.build_vbs(vcodes, lens)
    vbv, _ = B.scan_vbs(vcol, ResolvedPredicate.compare(Op.GE, (250 << 8) | 7, 2))
    want = (lens == 2) & (codes >= 250)
    assert torch.equal(vbv.dwords, pack_bools(want))
    got = B.lookup_vbs_rows(vcol, tail)
    pad = torch.where(lens[tail] == 2, vcodes[tail], vcodes[tail] << 8)
    assert torch.equal(got, pad)


@pytest.mark.parametrize("s,d", [(0.6, 16), (1.1, 24), (1.2, 20), (2.0, 12)])
def test_ragged_columns_every_supertile_size(s, d):
    """Ragged row counts and columns whose deep-row fraction selects each
    super-tile size of the SLICED kernel: PP-VBS and ByteSlice == the packed
    raw filter, with and without an input mask."""
    n = (1 << 24) + 12345
    vals = B.gen_zipf_device(B.ZipfSpec(s, d, n, 77))
    schema = E.Schema([E.ColumnSpec("v", B.ColumnKind.NUMERIC, "ppvbs"),
                       E.ColumnSpec("w", B.ColumnKind.NUMERIC, "byteslice")])
    store, _ = E.ingest_arrays({"v": vals, "w": vals}, schema, policy="forced")
    srt = torch.sort(vals).values
    g = torch.Generator(device="cuda").manual_seed(5)
    maskb = torch.rand(n, device="cuda", generator=g) < 0.7
    mask = B.DeviceBitVector(n, pack_bools(maskb))
    for a, b in ((0.1, 0.3), (0.995, 0.999), (0.0, 0.6)):
        lo, hi = int(srt[int(a * (n - 1))]), int(srt[int(b * (n - 1))])
        want = (vals >= lo) & (vals <= hi)
        for m, wm in ((None, want), (mask, want & maskb)):
            w = pack_bools(wm)
            for name in ("v", "w"):
                st = store.columns[name]
                p = st.dictionary.encode_literal(Predicate(name, Op.BETWEEN, lo, hi))
                bv, _ = E.scan_layout(st.layout, st.column, p, m)
                assert torch.equal(bv.dwords, w), (s, d, a, b, name, m is None)
