"""Layout dispatch and query execution (mirror of reference engine.py).

The dispatch point (engine.py:172-221) is where device layouts plug in.
``execute`` (engine.py:311-353) runs every conjunction as one device call
(bsb_conj_scan: predicate i sees the running result as its input mask and
blocks already ruled out load nothing from later columns), ORs disjunction
arms on the device and gathers + decodes each projected column straight from
the selection bitvector with the fused lookup kernels.

All five reference layouts run on the device: "byteslice" and "ppvbs" (the
north-star path) plus the paper's comparison baselines "bitpacked", "vbp"
and "pevbp".  CSV ingest (engine.py:114-165, file
I/O) is out of scope: ``ingest_arrays`` takes in-memory columns.

Timings: the reference writes one "scan" row per predicate (engine.py:
322-332).  Here a conjunction runs as one device call, so every predicate
of a group gets a row with ``op`` = its operator name, ``fused`` = True and
an equal share of the group's measured seconds (the rows still sum to the
conjunction's time).
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .advisor import advise_column
from .bitpacked import (build_bitpacked, bitpacked_size_report, lookup_bitpacked_bits,
                        scan_bitpacked)
from .bitvector import DeviceBitVector, as_device_bits
from .byteslice import (build_byteslice, byteslice_size_report, lookup_byteslice_bits,
                        lookup_byteslice_rows, scan_byteslice)
from .datagen import PRNG_NAME
from .device import device, stream
from .dictionary import ColumnKind, Dictionary, table_and_ranks
from .predicate import DEFAULT_LANES, LaneConfig, Predicate, ResolvedPredicate
from .vbp import build_vbp, lookup_vbp_bits, pad_codes, scan_vbp, vbp_size_report
from .vbs import build_vbs, lookup_vbs_bits, lookup_vbs_rows_dec, scan_vbs, vbs_size_report

__all__ = ["LAYOUTS", "DEVICE_LAYOUTS", "DataError", "ColumnSpec", "Schema", "Query",
           "QueryResult", "Store", "StoredColumn", "build_layout", "scan_layout",
           "lookup_decode", "lookup_decode_rows", "lookup_decode_bits", "execute", "ingest_arrays",
           "IngestReport", "size_report", "conj_scan", "conj_order"]

LAYOUTS = ("bitpacked", "byteslice", "vbp", "pevbp", "ppvbs")
DEVICE_LAYOUTS = LAYOUTS
_CONJ_LAYOUTS = ("byteslice", "ppvbs")  # layouts bsb_conj_scan chains natively
FORMAT_VERSION = 1

_SCHEME_FOR = {"bitpacked": "fixed", "byteslice": "fixed", "vbp": "fixed",
               "pevbp": "prefix_free", "ppvbs": "prefix_preserving"}


class DataError(Exception):
    """Input data problem: NULLs, bad literals, unknown columns."""


@dataclass(frozen=True)
class ColumnSpec:
    name: str
    kind: ColumnKind
    layout: str | None = None

    def __post_init__(self):
        if self.layout is not None and self.layout not in LAYOUTS:
            raise ValueError(f"unknown layout {self.layout!r}")


@dataclass
class Schema:
    columns: list

    def __post_init__(self):
        names = [c.name for c in self.columns]
        if len(set(names)) != len(names):
            raise ValueError("duplicate column names in schema")

    @staticmethod
    def parse_kind(text: str) -> ColumnKind:
        """engine.py:44-50, 79-84 (incl. the semi_categorical_string alias)."""
        kinds = {"numeric": ColumnKind.NUMERIC, "categorical": ColumnKind.CATEGORICAL,
                 "ordered_string": ColumnKind.ORDERED_STRING,
                 "semi_categorical_string": ColumnKind.ORDERED_STRING}
        if text not in kinds:
            raise ValueError(f"unknown column kind {text!r}")
        return kinds[text]


@dataclass
class IngestReport:
    rows: list = field(default_factory=list)    # per-column timing dicts
    advice: dict = field(default_factory=dict)  # name -> ColumnAdvice


@dataclass
class Query:
    groups: list
    projection: list

    @classmethod
    def conjunction(cls, predicates, projection) -> "Query":
        return cls([list(predicates)], list(projection))


@dataclass
class QueryResult:
    n_selected: int
    columns: dict
    timings: list
    selection: object


@dataclass
class StoredColumn:
    name: str
    kind: ColumnKind
    scheme: str
    layout: str
    dictionary: Dictionary
    column: object


@dataclass
class Store:
    manifest: dict
    columns: dict

    @property
    def n_rows(self) -> int:
        return int(self.manifest["n_rows"])


def _require_device_layout(layout: str):
    if layout not in DEVICE_LAYOUTS:
        raise ValueError(f"unknown layout {layout!r}")


def build_layout(layout: str, dictionary: Dictionary, ranks, lanes: LaneConfig = DEFAULT_LANES):
    """engine.py:172-188."""
    _require_device_layout(layout)
    a = dictionary.assignment
    if layout == "ppvbs":
        codes, lens = dictionary.row_codes_device(ranks)
        return build_vbs(codes, lens, lanes)
    r = ranks if isinstance(ranks, torch.Tensor) else np.asarray(ranks, dtype=np.int64)
    if layout == "byteslice":
        return build_byteslice(r, a.width_bits, lanes)
    lanes.require_device()
    if layout == "bitpacked":
        return build_bitpacked(r, a.width_bits)
    if layout == "vbp":
        return build_vbp(r, a.width_bits, "plain")
    rh = r.cpu().numpy() if isinstance(r, torch.Tensor) else r   # pevbp
    codes, lens = dictionary.row_codes(rh)
    return build_vbp(pad_codes(codes, lens, a.width_bits), a.width_bits, "padded_encoding")


def scan_layout(layout: str, column, pred, mask=None, threads: int = 1):
    """engine.py:191-201: (bitvector, ScanStats or None for bitpacked)."""
    _require_device_layout(layout)
    if layout == "byteslice":
        return scan_byteslice(column, pred, mask, threads)
    if layout == "ppvbs":
        return scan_vbs(column, pred, mask, threads)
    if layout == "bitpacked":
        return scan_bitpacked(column, pred, mask, threads), None
    return scan_vbp(column, pred, mask, threads)


def lookup_decode_rows(stored: StoredColumn, rows: torch.Tensor, out_dtype=torch.int64):
    """Device gather + decode of a row-id tensor (any order)."""
    if stored.layout == "ppvbs":
        return lookup_vbs_rows_dec(stored.column, rows, stored.dictionary.dev_decoder,
                                   out_dtype)
    if stored.layout != "byteslice":
        raise ValueError(f"row-id lookups are not provided for layout {stored.layout!r}")
    return lookup_byteslice_rows(stored.column, rows, stored.dictionary.dev_values, out_dtype)


def lookup_decode_bits(stored: StoredColumn, selection, out_dtype=torch.int64):
    """Fused selection -> decoded values on the device (ascending rows)."""
    dec = stored.dictionary.dev_decoder
    if stored.layout == "ppvbs":
        return lookup_vbs_bits(stored.column, selection, dec, out_dtype)
    if stored.layout == "byteslice":
        return lookup_byteslice_bits(stored.column, selection, dec, out_dtype)
    if stored.layout == "bitpacked":
        return lookup_bitpacked_bits(stored.column, selection, dec, out_dtype)
    _require_device_layout(stored.layout)
    return lookup_vbp_bits(stored.column, selection, dec, out_dtype)


def _to_values(stored: StoredColumn, dev: torch.Tensor) -> np.ndarray:
    """Device lookup output -> host values: numeric values as they are; for
    string kinds the device returned ranks (Dictionary.dev_values)."""
    h = dev.cpu().numpy()
    if stored.dictionary.numeric:
        return h
    return stored.dictionary.table.values[h]


def lookup_decode(stored: StoredColumn, selection) -> np.ndarray:
    """engine.py:204-221: selected rows of one column, decoded to values."""
    sel = as_device_bits(selection)
    if sel.count() == 0:
        return stored.dictionary.table.values[:0]
    return _to_values(stored, lookup_decode_bits(stored, sel))


def size_report(stored: StoredColumn) -> dict:
    if stored.layout == "bitpacked":
        return bitpacked_size_report(stored.column)
    if stored.layout in ("vbp", "pevbp"):
        return vbp_size_report(stored.column)
    if stored.layout == "ppvbs":
        return vbs_size_report(stored.column)
    return byteslice_size_report(stored.column)


def conj_order(layouts) -> list:
    """Evaluation order of a conjunction: ByteSlice predicates first (stable),
    so consecutive ones run as fused pairs with the AND in registers, then
    the PP-VBS predicates, which AND the running mask into their result
    words.  AND is commutative and idempotent, so the bitvector equals the
    reference's left-to-right pipeline (engine.py:322-332) for any order."""
    idx = list(range(len(layouts)))
    return ([i for i in idx if layouts[i] == "byteslice"] +
            [i for i in idx if layouts[i] != "byteslice"])


def conj_scan(columns, preds, mask=None) -> DeviceBitVector:
    """Fused conjunction over (layout, column) pairs and resolved predicates,
    evaluated in conj_order.

    More than BSB_MAX_CONJ predicates are chained 8 at a time, each chunk
    taking the previous result as its input mask (same semantics).
    """
    if len(columns) != len(preds):
        raise ValueError("one predicate per column")
    order = conj_order([layout for layout, _ in columns])
    columns = [columns[i] for i in order]
    preds = [preds[i] for i in order]
    lib = _lib.load()
    n = None
    for layout, col in columns:
        _require_device_layout(layout)
        n = col.n_rows if n is None else n
        if col.n_rows != n:
            raise ValueError("columns differ in row count")
    running = None if mask is None else as_device_bits(mask)
    if not columns:
        return running
    if any(layout not in _CONJ_LAYOUTS for layout, _ in columns):
        # baseline layouts: the same pipelined semantics, one scan call each
        for (layout, col), p in zip(columns, preds):
            running = as_device_bits(scan_layout(layout, col, p, running)[0])
        return running
    for c0 in range(0, len(columns), _lib.MAX_CONJ):
        chunk = list(zip(columns, preds))[c0:c0 + _lib.MAX_CONJ]
        refs = (_lib.BsbColumnRef * len(chunk))()
        cps = (_lib.BsbPred * len(chunk))()
        keep = []
        for i, ((layout, col), p) in enumerate(chunk):
            refs[i].layout = _lib.LAYOUT_PPVBS if layout == "ppvbs" else _lib.LAYOUT_BYTESLICE
            if layout == "ppvbs":
                refs[i].vbs = ctypes.pointer(col._desc)
            else:
                refs[i].byteslice = ctypes.pointer(col._desc)
            keep.append(refs[i])
            cps[i] = p.to_c()
        dev = device()
        out = torch.empty(-(-n // 32), dtype=torch.int32, device=dev)
        cnt = torch.empty(1, dtype=torch.int64, device=dev)
        _lib.check(lib.bsb_conj_scan(len(chunk), refs, cps,
                                     None if running is None else running.dwords.data_ptr(),
                                     out.data_ptr(), cnt.data_ptr(), stream()), "conj_scan")
        running = DeviceBitVector(n, out, cnt)
    return running


def _resolve(stored: StoredColumn, pred: Predicate) -> ResolvedPredicate:
    try:
        return stored.dictionary.encode_literal(pred)
    except (TypeError, ValueError) as exc:
        raise DataError(f"predicate on {pred.column!r}: {exc}") from None


def execute(store: Store, query: Query, threads: int = 1, out_dtype=torch.int64) -> QueryResult:
    """engine.py:311-353 with device conjunctions and fused lookups."""
    for name in query.projection:
        if name not in store.columns:
            raise DataError(f"unknown projection column {name!r}")
    for group in query.groups:
        for pred in group:
            if pred.column not in store.columns:
                raise DataError(f"unknown predicate column {pred.column!r}")
    timings = []
    arms = []
    for group in query.groups:
        cols, preds = [], []
        for pred in group:
            st = store.columns[pred.column]
            cols.append((st.layout, st.column))
            preds.append(_resolve(st, pred))
        t0 = time.perf_counter()
        if cols:
            running = conj_scan(cols, preds)
        else:
            running = DeviceBitVector.ones(store.n_rows)  # engine.py:333-334
        torch.cuda.current_stream().synchronize()
        dt = time.perf_counter() - t0
        for pred in group:
            timings.append({"column": pred.column, "phase": "scan", "op": pred.op.name,
                            "seconds": dt / len(group), "fused": True})
        arms.append(running)
    selection = arms[0]
    for extra in arms[1:]:
        selection = selection | extra
    n_sel = selection.count()
    out = {}
    for name in query.projection:
        st = store.columns[name]
        if n_sel == 0:
            out[name] = st.dictionary.table.values[:0]
            timings.append({"column": name, "phase": "lookup", "op": "", "seconds": 0.0})
            continue
        t0 = time.perf_counter()
        out[name] = _to_values(st, lookup_decode_bits(st, selection, out_dtype))
        timings.append({"column": name, "phase": "lookup", "op": "",
                        "seconds": time.perf_counter() - t0})
    return QueryResult(n_sel, out, timings, selection)


def ingest_arrays(columns: dict, schema: Schema | None = None, policy: str = "advisor", *,
                  advise_cost="wall", advise_count: int = 100, subsample: int | None = None,
                  lanes: LaneConfig = DEFAULT_LANES):
    """In-memory columns {name: values} (numpy / torch / lists) -> (Store,
    per-column report rows), the ingest path without the CSV reader."""
    store, rows, _ = _ingest(columns, schema, policy, advise_cost, advise_count, subsample,
                             lanes)
    return store, rows


def _ingest(columns: dict, schema: Schema | None, policy: str, advise_cost, advise_count: int,
            subsample: int | None, lanes: LaneConfig):
    """engine.py:239-297 over in-memory columns {name: values} (no CSV I/O).

    Per column: advise (unless the schema forces a layout), build the
    frequency table + ranks in one device sort, assign codes, build the
    device layout.  Returns (Store, report rows, {name: ColumnAdvice}).
    """
    if policy not in ("advisor", "forced"):
        raise ValueError(f"unknown layout policy {policy!r}")
    specs = schema.columns if schema is not None else [
        ColumnSpec(k, ColumnKind.NUMERIC) for k in columns]
    n_rows = None
    stored, entries, report, advised = {}, [], [], {}
    for spec in specs:
        vals = columns[spec.name]
        n = vals.numel() if isinstance(vals, torch.Tensor) else len(vals)
        if n_rows is not None and n != n_rows:
            raise DataError("columns differ in row count")
        n_rows = n
        layout, advice, advise_s = spec.layout, None, 0.0
        if layout is None:
            if policy == "forced":
                raise DataError(f"column {spec.name!r}: forced policy needs a layout")
            t0 = time.perf_counter()
            advice = advise_column(spec.name, vals, spec.kind, count=advise_count,
                                   cost=advise_cost, subsample=subsample, lanes=lanes)
            advise_s = time.perf_counter() - t0
            layout = advice.chosen
            advised[spec.name] = advice
        _require_device_layout(layout)
        t0 = time.perf_counter()
        try:
            table, ranks = table_and_ranks(vals, spec.kind)
            d = Dictionary.build(table, _SCHEME_FOR[layout])
        except ValueError as exc:
            raise DataError(f"column {spec.name!r}: {exc}") from None
        col = build_layout(layout, d, ranks, lanes)
        torch.cuda.current_stream().synchronize()
        encode_s = time.perf_counter() - t0
        stored[spec.name] = StoredColumn(spec.name, spec.kind, _SCHEME_FOR[layout], layout, d,
                                         col)
        e = {"name": spec.name, "kind": spec.kind.value, "scheme": _SCHEME_FOR[layout],
             "layout": layout, "n_distinct": table.n}
        if advice is not None and not advice.degenerate:
            e["advice"] = {"chosen": advice.chosen, "auc_byteslice": advice.auc_byteslice,
                           "auc_ppvbs": advice.auc_ppvbs}
        entries.append(e)
        report.append({"column": spec.name, "layout": layout, "n_distinct": table.n,
                       "encode_s": encode_s, "advise_s": advise_s})
    manifest = {"format_version": FORMAT_VERSION, "n_rows": n_rows, "prng": PRNG_NAME,
                "lane_count": lanes.lane_count, "columns": entries}
    return Store(manifest, stored), report, advised
