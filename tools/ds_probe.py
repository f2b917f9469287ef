"""Time the cfg2 PP-VBS BETWEEN windows under several bsb_tune settings
(diagnostic; one column build, CUDA events around each scan, L2 flushed
between reps).  Every setting must return the same words as the first.

    python tools/ds_probe.py "ds_enable=0" "ds_unroll=1,ds_prefetch=3" ...
"""
import ctypes
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2209_00220_b200 import _lib  # noqa: E402
from paper_2209_00220_b200.device import stream as cur_stream  # noqa: E402
from paper_2209_00220_b200.predicate import Op, Predicate  # noqa: E402


def main(settings, reps=20, log2n=28, layout="ppvbs", scan_lib=None):
    torch.cuda.set_device(0)
    lib = _lib.load()
    n = 1 << log2n
    data = bench.build_cfg2(n)
    col = data["col_v"] if layout == "ppvbs" else data["col_b"]
    d = data["d_ppe"] if layout == "ppvbs" else data["d_fix"]
    slib = lib if scan_lib is None else scan_lib
    fn = slib.bsb_vbs_scan if layout == "ppvbs" else slib.bsb_byteslice_scan
    if scan_lib is not None:  # another build: same C ABI for the scans
        for name in ("bsb_vbs_scan", "bsb_byteslice_scan"):
            getattr(slib, name).restype = getattr(lib, name).restype
            getattr(slib, name).argtypes = getattr(lib, name).argtypes
    wins = bench.window_bounds(data["table"].values, data["table"].weights, n)
    preds = [d.encode_literal(Predicate("c", Op.BETWEEN, lo, hi)).to_c() for _, lo, hi in wins]
    out = torch.empty(-(-n // 32), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ref = {}
    for setting in settings:
        for kv in filter(None, setting.split(",")):
            k, v = kv.split("=")
            assert slib.bsb_tune(k.encode(), int(v)) == 0, kv
        row = []
        for wi, cp in enumerate(preds):
            ts = []
            for r in range(reps + 2):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                rc = fn(col.desc_ref, ctypes.byref(cp), None, out.data_ptr(), cnt.data_ptr(),
                        None, None, cur_stream())
                e1.record()
                assert rc == 0, _lib.load().bsb_last_error()
                e1.synchronize()
                if r >= 2:
                    ts.append(e0.elapsed_time(e1) * 1000)
            h = int(torch.sum(out.to(torch.int64) * 2654435761 % 1000003).item())
            ref.setdefault(wi, (int(cnt.item()), h))
            assert ref[wi] == (int(cnt.item()), h), (setting, wi)
            row.append(statistics.median(ts))
        print(f"{setting:40s}", " ".join(f"{t:7.1f}" for t in row), flush=True)


if __name__ == "__main__":
    args = sys.argv[1:]
    scan_lib = None
    if args and args[0].startswith("--lib="):  # scans from another build of the library
        import ctypes
        scan_lib = ctypes.CDLL(os.path.abspath(args[0][len("--lib="):]))
        args = args[1:]
    layout = "ppvbs"
    if args and args[0] in ("ppvbs", "byteslice"):
        layout, args = args[0], args[1:]
    main(args or [""], layout=layout, scan_lib=scan_lib)
