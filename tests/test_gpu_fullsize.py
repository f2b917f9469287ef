"""Size-independent properties at BASELINE.json's full sizes (2^28 rows), where
the CPU oracle would take minutes: the cfg2 column's BETWEEN windows on
PP-VBS and ByteSlice agree bit for bit, BETWEEN == GE AND LE on both
layouts, counts equal a device histogram of the raw values, and the fused
lookups decode exactly the raw values of the selected rows."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2209_00220_b200 as B  # noqa: E402
from paper_2209_00220_b200 import engine as E  # noqa: E402
from paper_2209_00220_b200.predicate import Op, Predicate  # noqa: E402

N = 1 << 28


@pytest.fixture(scope="module")
def cfg2():
    vals = B.gen_zipf_device(B.ZipfSpec(1.2, 20, N, 42))
    schema = E.Schema([E.ColumnSpec("v", B.ColumnKind.NUMERIC, "ppvbs"),
                       E.ColumnSpec("w", B.ColumnKind.NUMERIC, "byteslice")])
    store, _ = E.ingest_arrays({"v": vals, "w": vals}, schema, policy="forced")
    return vals, store


def test_fullsize_windows_layouts_agree_and_between_is_ge_and_le(cfg2):
    vals, store = cfg2
    t = store.columns["v"].dictionary.table
    cum = np.cumsum(t.weights)
    q = lambda x: int(t.values[np.searchsorted(cum, min(N - 1, int(x * N)), side="right")])  # noqa
    for p in (0.001, 0.01, 0.1, 0.5):
        m = min(p, 0.25)
        lo, hi = q(1 - p - m), q(1 - m)
        want = int(((vals >= lo) & (vals <= hi)).sum().item())   # device histogram
        bits = {}
        for name in ("v", "w"):
            st = store.columns[name]
            d = st.dictionary
            bv, _ = E.scan_layout(st.layout, st.column,
                                  d.encode_literal(Predicate(name, Op.BETWEEN, lo, hi)))
            ge, _ = E.scan_layout(st.layout, st.column, d.encode_literal(Predicate(name, Op.GE, lo)))
            le, _ = E.scan_layout(st.layout, st.column, d.encode_literal(Predicate(name, Op.LE, hi)))
            assert bv.count() == want, (name, p)
            assert torch.equal(bv.dwords, (ge & le).dwords), (name, p)
            bits[name] = bv
        assert torch.equal(bits["v"].dwords, bits["w"].dwords), p
        if p <= 0.01:
            for name in ("v", "w"):
                got = E.lookup_decode_bits(store.columns[name], bits[name])
                rows = bits[name].row_ids()
                assert torch.equal(got, vals[rows]), (name, p)


@pytest.mark.parametrize("s,d", [(0.6, 16), (1.1, 24), (1.2, 20), (2.0, 12)])
def test_ragged_columns_every_supertile_size(s, d):
    """Ragged row counts and columns whose deep-row fraction selects each
    super-tile size of the SLICED kernel: PP-VBS == ByteSlice == a device
    filter of the raw values, with and without an input mask."""
    n = (1 << 24) + 12345
    vals = B.gen_zipf_device(B.ZipfSpec(s, d, n, 77))
    schema = E.Schema([E.ColumnSpec("v", B.ColumnKind.NUMERIC, "ppvbs"),
                       E.ColumnSpec("w", B.ColumnKind.NUMERIC, "byteslice")])
    store, _ = E.ingest_arrays({"v": vals, "w": vals}, schema, policy="forced")
    srt = torch.sort(vals).values
    g = torch.Generator(device="cuda").manual_seed(5)
    maskb = torch.rand(n, device="cuda", generator=g) < 0.7
    words = torch.zeros(-(-n // 32) * 32, dtype=torch.int64, device="cuda")
    words[:n] = maskb.to(torch.int64)
    shifts = torch.arange(32, device="cuda", dtype=torch.int64)
    mw = (words.view(-1, 32) << shifts).sum(1).to(torch.int64).to(torch.int32)
    mask = B.bitvector.DeviceBitVector(n, mw)
    for a, b in ((0.1, 0.3), (0.995, 0.999), (0.0, 0.6)):
        lo, hi = int(srt[int(a * (n - 1))]), int(srt[int(b * (n - 1))])
        want = (vals >= lo) & (vals <= hi)
        for m, wm in ((None, want), (mask, want & maskb)):
            res = []
            for name in ("v", "w"):
                st = store.columns[name]
                p = st.dictionary.encode_literal(Predicate(name, Op.BETWEEN, lo, hi))
                bv, _ = E.scan_layout(st.layout, st.column, p, m)
                res.append(bv)
            assert torch.equal(res[0].dwords, res[1].dwords), (s, d, a, b)
            assert res[0].count() == int(wm.sum().item()), (s, d, a, b, m is None)
