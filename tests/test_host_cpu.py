"""CPU-only checks: the C ABI library loads and exports every declared symbol,
host-side logic of the product (literal resolution, PPE assignment, bitvector
host type, advisor AUC/literal rules) matches the oracle / golden vectors.
No device compute happens here."""

import os
import re
import subprocess

import numpy as np
import pytest

import oracle as O
from golden_io import load

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bytestore_b200.h")


def _declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bsb_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2209_00220_b200 import _build, _lib
    if not os.path.exists(_lib.LIB_PATH):
        _build.build()
    return _lib.load()


def test_library_exports_every_header_symbol(lib):
    from paper_2209_00220_b200 import _lib
    declared = _declared_functions()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    # the ctypes binding declares exactly the header's functions
    assert sorted(_lib.EXPORTED_SYMBOLS) == declared
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    for name in declared:
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_tune_knobs(lib):
    # host-side knobs of the deep-row-space PP-VBS scan; unknown keys rejected
    keys = (b"ds_serial", b"ds_tiles", b"ds_unroll", b"ds_enable", b"ds_zonemap", b"ds_masked",
            b"dsm_cfg", b"sparse_ppm", b"conj_fuse", b"stats_rows", b"ctas_per_sm")
    for key in keys:
        assert lib.bsb_tune(key, 1) == 0
    for key in keys:  # < 0: back to the defaults (later tests in this process)
        assert lib.bsb_tune(key, -1) == 0
    assert lib.bsb_tune(b"no_such_knob", 1) != 0
    assert lib.bsb_tune(None, 1) != 0


def test_library_is_sm100a(lib):
    from paper_2209_00220_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert lib.bsb_stride_for(1) == 1024 and lib.bsb_stride_for(1025) == 2048


def test_ppe_numerical_native_matches_golden(lib):
    from paper_2209_00220_b200.dictionary import ppe_numerical
    data, _ = load("dict")
    for i in range(int(data["n_ppe"])):
        a = ppe_numerical(data[f"ppe{i}/weights"])
        assert np.array_equal(a.codes, data[f"ppe{i}/codes"]), i
        assert np.array_equal(a.lengths, data[f"ppe{i}/lengths"]), i


def test_ppe_decode_tree_on_golden_codes():
    """The lookup kernels' PPE tree decoder (host-built tables) maps every
    reference-generated ppe_numerical code back to its rank, and refuses
    code sets that are not ppe-shaped."""
    from paper_2209_00220_b200.dictionary import ppe_decode_tree
    data, _ = load("dict")
    for i in range(int(data["n_ppe"])):
        t = ppe_decode_tree(data[f"ppe{i}/codes"], data[f"ppe{i}/lengths"])
        assert t is not None, i
    # a deep leaf whose suffixes do not enumerate 1..size is not ppe-shaped
    assert ppe_decode_tree(np.array([0x01, 0x020105], np.uint64),
                           np.array([1, 3], np.uint8)) is None


def test_ppe_errors(lib):
    from paper_2209_00220_b200.dictionary import ppe_numerical
    with pytest.raises(ValueError):
        ppe_numerical([])
    with pytest.raises(ValueError):
        ppe_numerical([1, -1])


def test_literal_resolution_matches_golden(lib):
    import json

    from paper_2209_00220_b200.dictionary import ColumnKind, Dictionary, FrequencyTable
    from paper_2209_00220_b200.predicate import Op, Predicate
    data, _ = load("dict")
    res = json.loads(str(data["resolution"]))
    for k, block in enumerate(res):
        u, c = np.unique(data[f"res{k}/values"], return_counts=True)
        d = Dictionary.build(FrequencyTable(u, c, ColumnKind.NUMERIC), block["scheme"])
        for op, lo, hi, *want in block["cases"]:
            p = Predicate("c", Op[op], lo, hi) if op == "BETWEEN" else Predicate("c", Op[op], lo)
            r = d.encode_literal(p)
            got = [None if r.is_trivial else r.op.name, r.code, r.length, r.code2, r.length2,
                   r.trivial]
            assert got == want, (k, op, lo, hi)
        if f"res{k}/padded" in data:
            assert np.array_equal(d.padded, data[f"res{k}/padded"])
            assert np.array_equal(d.decode_padded(d.padded), data[f"res{k}/decoded"])


def test_decode_and_type_errors(lib):
    from paper_2209_00220_b200.dictionary import ColumnKind, Dictionary, FrequencyTable
    from paper_2209_00220_b200.predicate import Op, Predicate
    d = Dictionary.build(FrequencyTable(np.arange(300), np.arange(300, 0, -1),
                                        ColumnKind.NUMERIC), "prefix_preserving")
    assert d.decode_padded([0xFF01])[0] == 255 and d.decode_padded([0x0100])[0] == 0
    with pytest.raises(LookupError):
        d.decode_padded([0])
    with pytest.raises(TypeError):
        d.encode_literal(Predicate("c", Op.EQ, "x"))
    with pytest.raises(TypeError):
        d.encode_literal(Predicate("c", Op.EQ, True))
    cat = Dictionary.build(FrequencyTable(np.array(["b", "a"]), np.array([2, 1]),
                                          ColumnKind.CATEGORICAL), "prefix_preserving")
    with pytest.raises(ValueError):  # range predicate on a categorical column
        cat.encode_literal(Predicate("c", Op.LT, "b"))
    with pytest.raises(TypeError):
        cat.encode_literal(Predicate("c", Op.EQ, 3))
    with pytest.raises(ValueError):
        Dictionary.build(FrequencyTable(np.array(["a"]), np.array([1]), ColumnKind.CATEGORICAL),
                         "unknown_scheme")


def test_predicate_and_lane_validation():
    from paper_2209_00220_b200.predicate import LaneConfig, Op, Predicate, ResolvedPredicate
    with pytest.raises(ValueError):
        Predicate("c", Op.BETWEEN, 5)
    with pytest.raises(ValueError):
        Predicate("c", Op.BETWEEN, 5, 1)
    with pytest.raises(ValueError):
        Predicate("c", Op.EQ, 1, 2)
    with pytest.raises(ValueError):
        Op.parse("~")
    assert Op.parse("<>") is Op.NE
    with pytest.raises(ValueError):
        LaneConfig(12)
    with pytest.raises(ValueError):
        LaneConfig(16).require_device()
    p = ResolvedPredicate.between(1, 1, 0xFFFF, 2).to_c()
    assert (p.op, p.trivial, p.code, p.length, p.code2, p.length2) == (6, -1, 1, 1, 0xFFFF, 2)
    assert ResolvedPredicate.constant(False).to_c().trivial == 0


def test_host_bitvector_matches_reference_layout():
    from paper_2209_00220_b200.bitvector import ResultBitVector
    v = ResultBitVector.from_indices(40, [0, 33])
    assert v.words.tolist() == [1, 2]
    u = ResultBitVector(33, np.array([0xFFFFFFFF, 0xFFFFFFFF], np.uint32))
    assert u.count() == 33
    words = np.array([0xFFFFFFFF, 0xFFFFFFFF], np.uint32)
    ResultBitVector(33, words)
    assert words[1] == 0xFFFFFFFF  # caller memory is never mutated
    assert (~ResultBitVector.zeros(33)).count() == 33
    with pytest.raises(ValueError):
        ResultBitVector(10, np.zeros(2, np.uint32))


def test_advisor_host_rules():
    from paper_2209_00220_b200.advisor import ProfilePoint, _quantile_literals, auc
    assert auc([ProfilePoint(0, 3.0), ProfilePoint(1, 3.0)]) == pytest.approx(3.0)
    with pytest.raises(ValueError):
        auc([ProfilePoint(0, 1.0)])
    rng = np.random.default_rng(4)
    for vals in (rng.integers(0, 50, 1000), O.gen_zipf(1.2, 10, 5000, 3), np.arange(7)):
        u, c = np.unique(vals, return_counts=True)
        got = _quantile_literals(u, c, len(vals), 37)
        _, want = O.select_literals(vals, 37)
        assert got.tolist() == want
    # identical cost points -> identical float AUC as the oracle
    data, meta = load("advisor")
    for i, m in enumerate(meta):
        pb = [ProfilePoint(s, t) for s, t in data[f"{i}/pts_bs"]]
        pv = [ProfilePoint(s, t) for s, t in data[f"{i}/pts_vbs"]]
        assert auc(pb) == m["auc_bs"] and auc(pv) == m["auc_vbs"]
        assert ("byteslice" if auc(pb) <= auc(pv) else "ppvbs") == m["chosen"]


def test_pcg64_chunked_stream_is_identical():
    a = np.random.default_rng(7).random(10_000)
    r = np.random.default_rng(7)
    b = np.concatenate([r.random(3000), r.random(7000)])
    assert np.array_equal(a, b)


def test_device_path_fails_loudly_without_cuda():
    import torch

    from paper_2209_00220_b200 import build_byteslice
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(RuntimeError, match="CUDA"):
        build_byteslice(np.arange(10), 4)


def test_row_ids_must_be_integers():
    """device._to_dev rejects floating / bool data before touching a device
    (numpy fancy indexing in the reference rejects them too); integer dtypes
    of another width convert by value, not by bit reinterpretation."""
    import torch

    from paper_2209_00220_b200.device import to_dev_i64
    for bad in (torch.tensor([1.0, 2.0], dtype=torch.float64), torch.tensor([True, False]),
                np.array([0.5, 1.5]), np.array([True])):
        with pytest.raises(TypeError):
            to_dev_i64(bad)


def test_bits_module_matches_oracle():
    """Host bit helpers (reference bits.py API) agree with the oracle's
    restatement on random words, and keep the reference's edge cases."""
    import random
    from paper_2209_00220_b200 import bits as H
    rnd = random.Random(3)
    for _ in range(2000):
        x, m = rnd.getrandbits(32), rnd.getrandbits(32)
        assert H.pdep(x, m) == O.pdep(x, m)
        assert H.pext(x, m) == O.pext(x, m)
        assert H.pext(H.pdep(x, m), m) == x & ((1 << bin(m).count("1")) - 1)
        if x:
            assert H.lowest_set_index(x) == (x & -x).bit_length() - 1
            assert H.erase_rightmost(x) == x & (x - 1)
    assert H.erase_rightmost(0) == 0 and H.propagate_rightmost(0) == 0
    with pytest.raises(ValueError):
        H.lowest_set_index(0)
