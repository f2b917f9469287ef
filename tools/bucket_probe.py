"""Stage timings of the bucket-ordered row-id gather (diagnostic):
bsb_rows_bucket alone, the pair lookups alone, the direct gathers, per
bucket-bits setting (bsb_tune pair_bits).

    python tools/bucket_probe.py [log2n] [bits,bits,...]
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2209_00220_b200 import _lib  # noqa: E402
from paper_2209_00220_b200 import ColumnKind, Dictionary, FrequencyTable, ZipfSpec  # noqa: E402
from paper_2209_00220_b200.byteslice import build_byteslice  # noqa: E402
from paper_2209_00220_b200.datagen import gen_zipf_device  # noqa: E402
from paper_2209_00220_b200.device import stream  # noqa: E402
from paper_2209_00220_b200.dictionary import freq_table_and_ranks  # noqa: E402
from paper_2209_00220_b200.vbs import build_vbs  # noqa: E402


def timed(fn, steps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / steps * 1e3


def main():
    log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
    bits_list = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [13, 10, 7]
    lib = _lib.load()
    n, m = 1 << log2n, 1 << (log2n - 4)
    codes = torch.from_numpy(np.random.default_rng(3).integers(0, 1 << 24, n, dtype=np.int64)).cuda()
    col_b = build_byteslice(codes, 24)
    raw_b = codes.to(torch.int32)
    del codes
    vals = gen_zipf_device(ZipfSpec(1.0, 20, n, seed=4))
    raw_v = vals.to(torch.int32)
    u, c, ranks = freq_table_and_ranks(vals)
    d = Dictionary.build(FrequencyTable(u.cpu().numpy(), c.cpu().numpy(), ColumnKind.NUMERIC),
                         "prefix_preserving")
    cv, lv = d.row_codes_device(ranks)
    col_v = build_vbs(cv, lv)
    del cv, lv, ranks, vals
    dec = d.dev_decoder
    ids = torch.from_numpy(np.random.default_rng(5).integers(0, n, m)).cuda()
    srt = torch.sort(ids).values
    pairs = torch.empty(m, dtype=torch.int64, device="cuda")
    o32 = torch.empty(m, dtype=torch.int32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = stream()

    def bucket():
        lib.bsb_rows_bucket(ids.data_ptr(), m, n, pairs.data_ptr(), None, s)

    def bs_pairs():
        lib.bsb_byteslice_lookup_pairs(col_b.desc_ref, pairs.data_ptr(), None, None, m, None, None, None,
                                       o32.data_ptr(), err.data_ptr(), s)

    def vbs_pairs():
        lib.bsb_vbs_lookup_pairs_dec(col_v.desc_ref, pairs.data_ptr(), None, None, m, ctypes.byref(dec), None,
                                     None, o32.data_ptr(), err.data_ptr(), s)

    def bs_rows(t):
        return lambda: lib.bsb_byteslice_lookup_rows(col_b.desc_ref, t.data_ptr(), m, None, None,
                                                     None, o32.data_ptr(), err.data_ptr(), s)

    def vbs_rows(t):
        return lambda: lib.bsb_vbs_lookup_rows_dec(col_v.desc_ref, t.data_ptr(), m,
                                                   ctypes.byref(dec), None, None, o32.data_ptr(),
                                                   err.data_ptr(), s)

    print(f"rows 2^{log2n}, ids 2^{log2n - 4}; times in us")
    if "--nodirect" not in sys.argv:
      print("direct  bs unsorted %.1f  sorted %.1f | vbs unsorted %.1f sorted %.1f" % (
          timed(bs_rows(ids)), timed(bs_rows(srt)), timed(vbs_rows(ids)), timed(vbs_rows(srt))))
    for bits in bits_list:
        lib.bsb_tune(b"pair_bits", bits)
        tb = timed(bucket)
        t1 = timed(bs_pairs)
        assert torch.equal(o32, raw_b[ids])
        t2 = timed(vbs_pairs)
        assert torch.equal(o32, raw_v[ids])
        print(f"pair_bits {bits:2d}: bucket {tb:.1f}  bs_pairs {t1:.1f} (total {tb + t1:.1f})  "
              f"vbs_pairs {t2:.1f} (total {tb + t2:.1f})")
    assert int(err.item()) == 0


if __name__ == "__main__":
    main()
