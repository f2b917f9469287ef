"""Time the cfg5 queries on ONE 2^29-row segment per column (diagnostic).

Each query's C ABI call is timed with CUDA events (L2 flushed before every
rep); with --lib=PATH a second build of libbytestore_b200.so is timed on the
same columns and must return the same words.  bsb_tune settings can be
given as k=v,k=v.

    python tools/cfg5_probe.py [--lib=other.so] [--reps=20] ["tune=1,..."]
"""
import ctypes
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench_cfg5 as C  # noqa: E402
from paper_2209_00220_b200 import _lib  # noqa: E402


def main(argv):
    reps = 20
    libs = [("this", None)]
    settings = []
    for a in argv:
        if a.startswith("--lib="):
            libs.append((a[6:], a[6:]))
        elif a.startswith("--reps="):
            reps = int(a[7:])
        else:
            settings.append(a)
    torch.cuda.set_device(0)
    base = _lib.load()
    tab = C.Cfg5Table(1, 0, 1 << 29, only_segments=[0], keep_raw=True)
    step = C.Cfg5Step(tab, 1)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    words = {}
    for name, path in libs:
        lib = base if path is None else ctypes.CDLL(os.path.abspath(path))
        if path is not None:
            for fn in ("bsb_vbs_scan", "bsb_byteslice_scan", "bsb_conj_scan", "bsb_tune"):
                getattr(lib, fn).restype = getattr(base, fn).restype
                getattr(lib, fn).argtypes = getattr(base, fn).argtypes
        for setting in settings or [""]:
            for kv in filter(None, setting.split(",")):
                k, v = kv.split("=")
                assert lib.bsb_tune(k.encode(), int(v)) == 0, kv
            row = {}
            for q in C.QUERIES:
                fn, args = step.calls(q, 0)
                fn = getattr(lib, fn.__name__)
                ts = []
                for r in range(reps + 2):
                    flush.zero_()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    rc = fn(*args, _lib.stream_ptr())
                    e1.record()
                    e1.synchronize()
                    assert rc == 0, rc
                    if r >= 2:
                        ts.append(e0.elapsed_time(e1) * 1000)
                w = step.words[q][0].clone()
                if q in words:
                    assert torch.equal(words[q], w), f"{name} {setting} {q}: words differ"
                else:
                    words[q] = w
                row[q] = statistics.median(ts)
            print(f"{name:>12} {setting:>24} " +
                  " ".join(f"{q}={row[q]:7.1f}us" for q in C.QUERIES), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
