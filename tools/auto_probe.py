"""Host time and device time of the row-id lookup entry points (diagnostic)."""
import os, sys, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2209_00220_b200 import _lib
from paper_2209_00220_b200.byteslice import build_byteslice
from paper_2209_00220_b200.device import stream

lib = _lib.load()
n = 1 << 28
m = 1 << (int(sys.argv[1]) if len(sys.argv) > 1 else 24)
codes = torch.from_numpy(np.random.default_rng(3).integers(0, 1 << 24, n, dtype=np.int64)).cuda()
col = build_byteslice(codes, 24)
del codes
ids = torch.from_numpy(np.random.default_rng(5).integers(0, n, m)).cuda()
srt = torch.sort(ids).values
o32 = torch.empty(m, dtype=torch.int32, device="cuda")
err = torch.zeros(1, dtype=torch.int32, device="cuda")
s = stream()
for name, t in (("sorted", srt), ("unsorted", ids)):
    for label, fn in (
        ("rows       ", lambda: lib.bsb_byteslice_lookup_rows(col.desc_ref, t.data_ptr(), m, None, None, None, o32.data_ptr(), err.data_ptr(), s)),
        ("auto       ", lambda: lib.bsb_byteslice_lookup_rows_auto(col.desc_ref, t.data_ptr(), m, None, None, None, o32.data_ptr(), err.data_ptr(), s)),
        ("auto + sync", lambda: lib.bsb_byteslice_lookup_rows_auto(col.desc_ref, t.data_ptr(), m, None, None, None, o32.data_ptr(), None, s)),
    ):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        host, dev = [], []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            t0 = time.perf_counter()
            fn()
            host.append((time.perf_counter() - t0) * 1e6)
            e1.record()
            e1.synchronize()
            dev.append(e0.elapsed_time(e1) * 1e3)
        print(f"{name:9s} {label}: host {np.median(host):7.1f} us  device {np.median(dev):7.1f} us")
