"""Masked PP-VBS scans on ONE cfg5 segment (diagnostic): the AND's legs
(z0 under u0&u1, z1 under u0&u1&z0) and z1 under seeded random masks of
several densities, with the compacted kernel (ds_masked=0), the
block-masked one (ds_masked=1) and the scan-whole + AND cost (unmasked
scan).  Words are checked equal across kernels and against the unmasked
words AND the mask.

    python tools/masked_probe.py [--reps=10]
"""
import ctypes
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench_cfg5 as C  # noqa: E402
from paper_2209_00220_b200 import _lib  # noqa: E402


def main(argv):
    reps = 10
    cfgs = [0]
    only = 0
    for a in argv:
        if a.startswith("--reps="):
            reps = int(a[7:])
        elif a.startswith("--cases="):
            only = int(a[8:])
        elif a.startswith("--cfgs="):
            cfgs = [int(x) for x in a[7:].split(",")]
    torch.cuda.set_device(0)
    lib = _lib.load()
    tab = C.Cfg5Table(1, 0, 1 << 29, only_segments=[0], keep_raw=False)
    step = C.Cfg5Step(tab, 1)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    sp = _lib.stream_ptr()
    for q in ("u0", "u1", "z0", "z1"):
        fn, args = step.calls(q, 0)
        _lib.check(fn(*args, sp), q)
    torch.cuda.synchronize()
    W = {q: step.words[q][0].clone() for q in ("u0", "u1", "z0", "z1")}
    nb = W["z1"].numel()
    out = torch.empty_like(W["z1"])
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")

    def timed(q, mask):
        col = tab.cols[q][0]
        ts = []
        for r in range(reps + 2):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            rc = lib.bsb_vbs_scan(col.desc_ref, ctypes.byref(step.cpreds[q]),
                                  None if mask is None else mask.data_ptr(), out.data_ptr(),
                                  cnt.data_ptr(), None, None, sp)
            e1.record()
            e1.synchronize()
            assert rc == 0, rc
            if r >= 2:
                ts.append(e0.elapsed_time(e1) * 1000)
        return statistics.median(ts), out.clone()

    m1 = W["u0"] & W["u1"]
    m2 = m1 & W["z0"]
    g = torch.Generator(device="cuda").manual_seed(7)
    cases = [("z0 | u0&u1", "z0", m1), ("z1 | u0&u1&z0", "z1", m2)]
    for p in (0.001, 0.0075, 0.02, 0.05, 0.2, 0.5):
        bits = torch.rand(nb * 32, generator=g, device="cuda") < p
        w = (bits.view(nb, 32).to(torch.int64) << torch.arange(32, device="cuda")).sum(1)
        cases.append((f"z1 | rand {p * 100:g}%", "z1", w.to(torch.int32)))
    if only:
        cases = cases[:only]
    for name, q, mask in cases:
        dens = int(np.bitwise_count(mask.cpu().numpy().view(np.uint32)).sum()) / (nb * 32)
        t_un, w_un = timed(q, None)
        row = {"whole": t_un}
        ref = w_un & mask
        for k in [("c", c) for c in cfgs] + [("b", 0)]:
            lib.bsb_tune(b"ds_masked", 0 if k[0] == "c" else 1)
            lib.bsb_tune(b"dsm_cfg", k[1])
            t, w = timed(q, mask)
            assert torch.equal(w, ref), f"{name} {k}: words differ"
            row[k] = t
        lib.bsb_tune(b"ds_masked", 0)
        lib.bsb_tune(b"dsm_cfg", cfgs[0])
        print(f"{name:>18} dens={dens:.4f}  whole {row['whole']:6.1f}  compacted " +
              " ".join(f"[{c}] {row[('c', c)]:6.1f}" for c in cfgs) +
              f"  block-masked {row[('b', 0)]:6.1f} us", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
