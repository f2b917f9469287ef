"""Diagnostics: cfg1 scan (2^24 rows, w=16, LT 6554) per-launch device time
on 16 rotated replicas (eager and graph), and the ScanStats path time for
the cfg2 windows (PP-VBS SLICED row-parallel stats kernel, ByteSlice stats
variant) vs the plain scan.

    python tools/misc_probe.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2209_00220_b200.byteslice import build_byteslice, scan_byteslice  # noqa: E402
from paper_2209_00220_b200.predicate import Op, Predicate, ResolvedPredicate  # noqa: E402
from paper_2209_00220_b200.vbs import scan_vbs  # noqa: E402


def ev_time(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    torch.cuda.set_device(0)
    n = 1 << 24
    codes = np.random.default_rng(1).integers(0, 65536, n)
    reps = [build_byteslice(codes, 16) for _ in range(16)]
    pred = ResolvedPredicate.compare(Op.LT, 6554, 2)
    it = [0]

    def one():
        c = reps[it[0] % 16]
        it[0] += 1
        scan_byteslice(c, pred)
    print(f"cfg1 scan public API eager: {ev_time(one, 64):.2f} us")
    data = bench.build_cfg2(1 << 28)
    wins = bench.window_bounds(data["table"].values, data["table"].weights, 1 << 28)
    for p, lo, hi in wins:
        for name, col, d, fn in (("ppvbs", data["col_v"], data["d_ppe"], scan_vbs),
                                 ("byteslice", data["col_b"], data["d_fix"], scan_byteslice)):
            rp = d.encode_literal(Predicate("c", Op.BETWEEN, lo, hi))
            t_scan = ev_time(lambda: fn(col, rp), 10)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(3):
                fn(col, rp)[1].materialize()
            t_stats = (time.perf_counter() - t0) / 3 * 1e6
            # the stats call alone on the device (C ABI, events; no host copies)
            import ctypes
            from paper_2209_00220_b200 import _lib
            lib = _lib.load()
            nb = col.n_blocks
            stw = torch.zeros(_lib.STATS_WORDS, dtype=torch.int64, device="cuda")
            dep = torch.zeros(nb, dtype=torch.int8, device="cuda")
            out = torch.empty(nb, dtype=torch.int32, device="cuda")
            cnt = torch.empty(1, dtype=torch.int64, device="cuda")
            cp = rp.to_c()
            f = lib.bsb_vbs_scan if name == "ppvbs" else lib.bsb_byteslice_scan
            t_dev = ev_time(lambda: f(col.desc_ref, ctypes.byref(cp), None, out.data_ptr(),
                                      cnt.data_ptr(), stw.data_ptr(), dep.data_ptr(),
                                      _lib.stream_ptr()), 5)
            print(f"cfg2 p={p} {name}: scan {t_scan:.1f} us, stats (wall) {t_stats:.1f} us "
                  f"= {t_stats / t_scan:.1f}x; stats call on the device {t_dev:.1f} us "
                  f"= {t_dev / t_scan:.1f}x")


if __name__ == "__main__":
    main()
