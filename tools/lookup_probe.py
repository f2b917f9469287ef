"""Run the cfg3 lookup measurements alone (diagnostic; for ncu launch lists).

    python tools/lookup_probe.py [steps] [log2n]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1].startswith("--lib="):  # another build, all symbols
        from paper_2209_00220_b200 import _lib
        _lib.load(os.path.abspath(sys.argv.pop(1)[len("--lib="):]))
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    log2n = int(sys.argv[2]) if len(sys.argv) > 2 else 28
    only = sys.argv[3] if len(sys.argv) > 3 else None
    for k, v in bench.measure_lookups(steps, log2n, only).items():
        print(k, json.dumps(v))
