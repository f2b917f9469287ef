"""Where the cfg1 scan's ~10 us go (diagnostic).  Each case is 16 rotated
2^24-row replicas captured as one CUDA graph; per-replica microseconds:
  scan      bsb_byteslice_scan as bench.py times it (count memset + kernel)
  scan_nocount  the same call with count = NULL (words only, as the reference's scan)
  persistent*   the same with the small-column kernel off (bsb_tune bs_small=0)
  kernel    the scan kernel alone (bsb_tune scan_nomemset: count not zeroed)
  zero_count  a torch fill of the 8-byte count (a kernel node, not a memset)
  read      torch sum over the replica's planes (a plain streaming read of
            the same 2 x 16 MB + padding)
  popc_plane1  bsb_bits_popcount over plane 1 (16 MB streaming read, + count memset)
  empty     a 1-element torch add (launch floor)

    python tools/cfg1_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2209_00220_b200 import _lib  # noqa: E402
from paper_2209_00220_b200.byteslice import build_byteslice  # noqa: E402
from paper_2209_00220_b200.predicate import Op, ResolvedPredicate  # noqa: E402


def graph_us(body, reps=20):
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=cap):
        for i in range(16):
            body(i, cap.cuda_stream)
    torch.cuda.current_stream().wait_stream(cap)
    g.replay()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000 / reps / 16


def main():
    import ctypes
    torch.cuda.set_device(0)
    lib = _lib.load()
    n, w = 1 << 24, 16
    codes = np.random.default_rng(1).integers(0, 65536, n)
    reps = [build_byteslice(codes, w) for _ in range(16)]
    cp = ResolvedPredicate.compare(Op.LT, 6554, 2).to_c()
    outs = [torch.empty(n // 32, dtype=torch.int32, device="cuda") for _ in reps]
    cnts = [torch.zeros(1, dtype=torch.int64, device="cuda") for _ in reps]
    one = torch.zeros(1, device="cuda")
    planes = [r.planes.view(torch.int64) for r in reps]

    def scan(i, s):
        _lib.check(lib.bsb_byteslice_scan(reps[i].desc_ref, ctypes.byref(cp), None,
                                          outs[i].data_ptr(), cnts[i].data_ptr(), None, None,
                                          s), "scan")

    def scan_nc(i, s):
        _lib.check(lib.bsb_byteslice_scan(reps[i].desc_ref, ctypes.byref(cp), None,
                                          outs[i].data_ptr(), None, None, None, s), "scan")

    rows = {"scan": graph_us(scan), "scan_nocount": graph_us(scan_nc)}
    lib.bsb_tune(b"pdl", 0)
    rows["scan_nocount_nopdl"] = graph_us(scan_nc)
    lib.bsb_tune(b"pdl", -1)
    lib.bsb_tune(b"bs_small", 0)
    rows["persistent"] = graph_us(scan)
    rows["persistent_nocount"] = graph_us(scan_nc)
    lib.bsb_tune(b"bs_small", -1)
    if lib.bsb_tune(b"scan_nomemset", 1) == 0:
        rows["kernel"] = graph_us(scan)
        lib.bsb_tune(b"scan_nomemset", -1)
    rows["zero_count"] = graph_us(lambda i, s: cnts[i].zero_())
    rows["read"] = graph_us(lambda i, s: planes[i].sum())
    # bsb_bits_popcount over the first plane (16 MB): our own streaming read
    rows["popc_plane1"] = graph_us(lambda i, s: _lib.check(lib.bsb_bits_popcount(
        reps[i].planes.data_ptr(), n * 8, cnts[i].data_ptr(), s), "popc"))
    rows["empty"] = graph_us(lambda i, s: one.add_(1))
    print({k: (round(v, 2) if isinstance(v, float) else v) for k, v in rows.items()})


if __name__ == "__main__":
    main()
