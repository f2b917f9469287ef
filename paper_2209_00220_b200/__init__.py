"""B200-native ByteStore hot path: ByteSlice / PP-VBS encode, scan, lookup,
conjunctions and the layout advisor, as hand-written sm_100a CUDA behind the
C ABI in include/bytestore_b200.h.

The names re-exported here cover the reference package's whole public
surface (reference __init__.py:10-52, every layout and column kind) plus the
device-specific entry points.  Importing the
package does not touch the GPU; the first device call loads
libbytestore_b200.so and fails loudly if it (or a CUDA device) is missing.
"""

from .predicate import DEFAULT_LANES, LaneConfig, Op, Predicate, ResolvedPredicate
from .stats import LookupStats, ScanStats

__version__ = "0.1.0"

_LAZY = {
    "ResultBitVector": "bitvector", "DeviceBitVector": "bitvector",
    "bitvector_and": "bitvector", "bitvector_or": "bitvector", "popcount_vector": "bitvector",
    "ByteSliceColumn": "byteslice", "build_byteslice": "byteslice",
    "scan_byteslice": "byteslice", "lookup_byteslice": "byteslice",
    "lookup_byteslice_rows": "byteslice", "lookup_byteslice_bits": "byteslice",
    "byteslice_size_report": "byteslice",
    "VbsColumn": "vbs", "build_vbs": "vbs", "scan_vbs": "vbs", "lookup_vbs": "vbs",
    "lookup_vbs_rows": "vbs", "lookup_vbs_rows_dec": "vbs", "lookup_vbs_bits": "vbs",
    "vbs_size_report": "vbs",
    "write_store": "store", "read_store": "store", "store_bytes": "store",
    "BitPackedColumn": "bitpacked", "build_bitpacked": "bitpacked",
    "scan_bitpacked": "bitpacked", "lookup_bitpacked": "bitpacked",
    "bitpacked_size_report": "bitpacked", "VbpColumn": "vbp", "build_vbp": "vbp",
    "pad_codes": "vbp", "scan_vbp": "vbp", "lookup_vbp": "vbp", "vbp_size_report": "vbp",
    "ppe_categorical": "dictionary", "prefix_free_assignment": "dictionary",
    "ColumnKind": "dictionary", "FrequencyTable": "dictionary", "CodeAssignment": "dictionary",
    "Dictionary": "dictionary", "build_frequency_table": "dictionary",
    "ppe_numerical": "dictionary", "fixed_assignment": "dictionary",
    "compare_codes": "dictionary",
    "ZipfSpec": "datagen", "gen_zipf": "datagen", "zipf_pmf": "datagen",
    "gen_zipf_device": "datagen",
    "ProfilePoint": "advisor", "ColumnAdvice": "advisor", "advise": "advisor",
    "advise_column": "advisor", "auc": "advisor", "select_literals": "advisor",
    "LAYOUTS": "engine", "DataError": "engine", "ColumnSpec": "engine", "Schema": "engine",
    "Query": "engine", "QueryResult": "engine", "Store": "engine", "StoredColumn": "engine",
    "build_layout": "engine", "scan_layout": "engine", "lookup_decode": "engine",
    "execute": "engine", "ingest_arrays": "engine", "conj_scan": "engine",
}

__all__ = ["DEFAULT_LANES", "LaneConfig", "Op", "Predicate", "ResolvedPredicate", "ScanStats",
           "LookupStats", *_LAZY]


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib
    value = getattr(importlib.import_module(f".{mod}", __name__), name)
    globals()[name] = value
    return value
