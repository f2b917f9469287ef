"""ctypes binding of the C ABI in include/bytestore_b200.h.

This is exactly the binding a maintainer would add to the reference package
(see INTEGRATION.md): the shared library is loaded from the package
directory and every entry point is declared with its C signature.  There is
no fallback: if the library is missing or no CUDA device is present, calls
fail loudly.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int32, c_int64, c_uint8, c_uint64, c_void_p

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libbytestore_b200.so")

LANES = 32
TILE_ROWS = 1024
MAX_LEVELS = 8
MAX_CONJ = 8
STATS_WORDS = 24

OK, EINVAL, ERANGE, ENOTFOUND, ECUDA, EKEY, EINDEX = 0, 1, 2, 3, 4, 5, 6
ERR_NOTFOUND, ERR_INDEX = 1, 2  # device error word bits (err_dev)
OP_CODES = {"EQ": 0, "NE": 1, "LT": 2, "LE": 3, "GT": 4, "GE": 5, "BETWEEN": 6}
LAYOUT_BYTESLICE, LAYOUT_PPVBS = 0, 1
DEEP_PACKED, DEEP_SLICED = 0, 3
VBP_PLAIN, VBP_PADDED = 0, 1
VBP_MAX_PLANES, VBP_STATS_WORDS = 32, 66


class BsbPred(ctypes.Structure):
    _fields_ = [("op", c_int32), ("trivial", c_int32), ("code", c_uint64), ("code2", c_uint64),
                ("length", c_int32), ("length2", c_int32)]


class BsbByteSlice(ctypes.Structure):
    _fields_ = [("n_rows", c_int64), ("stride", c_int64), ("width_bits", c_int32),
                ("n_slices", c_int32), ("slices", c_void_p)]


class BsbVbs(ctypes.Structure):
    _fields_ = [("n_rows", c_int64), ("stride", c_int64), ("max_len", c_int32),
                ("deep_mode", c_int32), ("bs1", c_void_p), ("deep", c_void_p * MAX_LEVELS),
                ("exist", c_void_p * MAX_LEVELS), ("block_dir", c_void_p * MAX_LEVELS),
                ("deep_len", c_int64 * MAX_LEVELS), ("rexist", c_void_p * MAX_LEVELS),
                ("deep1_shared", c_int32), ("reserved", c_int32)]


class BsbDecode(ctypes.Structure):
    _fields_ = [("kind", c_int32), ("reserved", c_int32), ("values", c_void_p),
                ("sorted_padded", c_void_p), ("n_dict", c_int64), ("e1", c_void_p),
                ("e2", c_void_p)]


class BsbBitPacked(ctypes.Structure):
    _fields_ = [("n_rows", c_int64), ("width_bits", c_int32), ("reserved", c_int32),
                ("words", c_void_p)]


class BsbVbp(ctypes.Structure):
    _fields_ = [("n_rows", c_int64), ("w_max", c_int32), ("kind", c_int32),
                ("planes", c_void_p)]


class BsbColumnRef(ctypes.Structure):
    _fields_ = [("layout", c_int32), ("reserved", c_int32),
                ("byteslice", POINTER(BsbByteSlice)), ("vbs", POINTER(BsbVbs))]


_P = c_void_p
_SIGS = {
    "bsb_version": (c_char_p, []),
    "bsb_last_error": (c_char_p, []),
    "bsb_tune": (c_int32, [c_char_p, c_int64]),
    "bsb_stride_for": (c_int64, [c_int64]),
    "bsb_byteslice_build": (c_int32, [_P, c_int64, c_int32, _P, c_int64, _P]),
    "bsb_byteslice_build_ranks": (c_int32, [_P, c_int64, c_int32, _P, c_int64, _P]),
    "bsb_byteslice_export": (c_int32, [POINTER(BsbByteSlice), _P, _P]),
    "bsb_byteslice_scan": (c_int32, [POINTER(BsbByteSlice), POINTER(BsbPred), _P, _P, _P, _P,
                                     _P, _P]),
    "bsb_byteslice_lookup_rows": (c_int32, [POINTER(BsbByteSlice), _P, c_int64, _P, _P, _P, _P,
                                            _P, _P]),
    "bsb_vbs_plan": (c_int32, [_P, _P, c_int64, POINTER(c_int32), POINTER(c_int64), _P]),
    "bsb_vbs_build": (c_int32, [_P, _P, POINTER(BsbVbs), _P]),
    "bsb_vbs_export_bs1": (c_int32, [POINTER(BsbVbs), _P, _P]),
    "bsb_vbs_export_level": (c_int32, [POINTER(BsbVbs), c_int32, _P, _P, _P]),
    "bsb_vbs_scan": (c_int32, [POINTER(BsbVbs), POINTER(BsbPred), _P, _P, _P, _P, _P, _P]),
    "bsb_vbs_lookup_rows": (c_int32, [POINTER(BsbVbs), _P, c_int64, _P, _P, _P, c_int64, _P, _P,
                                      _P, _P, _P]),
    "bsb_byteslice_lookup_bits": (c_int32, [POINTER(BsbByteSlice), _P, POINTER(BsbDecode), _P,
                                            _P, _P, _P, _P]),
    "bsb_vbs_lookup_bits": (c_int32, [POINTER(BsbVbs), _P, POINTER(BsbDecode), _P, _P, _P, _P,
                                      _P]),
    "bsb_vbs_lookup_rows_dec": (c_int32, [POINTER(BsbVbs), _P, c_int64, POINTER(BsbDecode), _P,
                                          _P, _P, _P, _P]),
    "bsb_rows_sort": (c_int32, [_P, c_int64, c_int64, _P, _P, POINTER(c_int32), _P]),
    "bsb_rows_bucket": (c_int32, [_P, c_int64, c_int64, _P, _P, _P]),
    "bsb_byteslice_lookup_pairs": (c_int32, [POINTER(BsbByteSlice), _P, _P, _P, c_int64, _P, _P,
                                             _P, _P, _P, _P]),
    "bsb_vbs_lookup_pairs_dec": (c_int32, [POINTER(BsbVbs), _P, _P, _P, c_int64,
                                           POINTER(BsbDecode), _P, _P, _P, _P, _P]),
    "bsb_byteslice_lookup_rows_auto": (c_int32, [POINTER(BsbByteSlice), _P, c_int64, _P, _P, _P,
                                                 _P, _P, _P]),
    "bsb_vbs_lookup_rows_dec_auto": (c_int32, [POINTER(BsbVbs), _P, c_int64, POINTER(BsbDecode),
                                               _P, _P, _P, _P, _P]),
    "bsb_scatter": (c_int32, [_P, _P, c_int64, c_int32, _P, _P]),
    "bsb_bits_to_rows": (c_int32, [_P, c_int64, _P, POINTER(c_int64), _P]),
    "bsb_bits_to_rows_async": (c_int32, [_P, c_int64, c_int64, _P, _P, _P]),
    "bsb_bits_to_rows_at": (c_int32, [_P, c_int64, c_int64, _P, _P, _P, _P]),
    "bsb_bits_combine": (c_int32, [c_int32, _P, _P, _P, c_int64, _P]),
    "bsb_bits_popcount": (c_int32, [_P, c_int64, _P, _P]),
    "bsb_conj_scan": (c_int32, [c_int32, POINTER(BsbColumnRef), POINTER(BsbPred), _P, _P, _P,
                                _P]),
    "bsb_freq_table": (c_int32, [_P, c_int64, _P, _P, _P, POINTER(c_int64), _P]),
    "bsb_encode_rows": (c_int32, [_P, c_int64, _P, c_int64, _P, _P]),
    "bsb_ppe_numerical_host": (c_int32, [_P, c_int64, _P, _P]),
    "bsb_gather_codes": (c_int32, [_P, c_int64, _P, _P, _P, _P, _P]),
    "bsb_zipf_from_uniform": (c_int32, [_P, c_int64, _P, c_int64, _P, _P]),
    "bsb_stats_layout": (None, [POINTER(c_int32)] * 5),
    "bsb_bitpacked_words_for": (c_int64, [c_int64, c_int32]),
    "bsb_bitpacked_build": (c_int32, [_P, c_int64, c_int32, _P, _P]),
    "bsb_bitpacked_scan": (c_int32, [POINTER(BsbBitPacked), POINTER(BsbPred), _P, _P, _P, _P]),
    "bsb_bitpacked_lookup_bits": (c_int32, [POINTER(BsbBitPacked), _P, POINTER(BsbDecode), _P,
                                            _P, _P, _P, _P]),
    "bsb_vbp_build": (c_int32, [_P, c_int64, c_int32, _P, _P]),
    "bsb_vbp_scan": (c_int32, [POINTER(BsbVbp), POINTER(BsbPred), _P, _P, _P, _P, _P, _P]),
    "bsb_vbp_lookup_bits": (c_int32, [POINTER(BsbVbp), _P, POINTER(BsbDecode), _P, _P, _P, _P,
                                      _P]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None


class NativeLibraryMissing(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    """Load (once) and declare the C ABI.  Raises if the library is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeLibraryMissing(
            f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the device path)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().bsb_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = ""):
    """Map a C status to the reference's exception types (header comment)."""
    if rc == OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc in (EINVAL, ERANGE):
        raise ValueError(msg)
    if rc == ENOTFOUND:
        raise LookupError(msg)
    if rc == EKEY:
        raise KeyError(msg)
    if rc == EINDEX:
        raise IndexError(msg)
    raise RuntimeError(f"CUDA error in {msg}")


def ptr(t) -> int:
    """Device pointer of a torch tensor (or None -> NULL)."""
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


__all__ = ["load", "check", "ptr", "stream_ptr", "BsbPred", "BsbByteSlice", "BsbVbs",
           "BsbColumnRef", "BsbDecode", "EXPORTED_SYMBOLS", "c_double", "c_int64", "c_int32", "c_uint8",
           "c_uint64"]
