"""Run one of bench_cfgs' measurements alone (diagnostic).

    python tools/cfg_probe.py cfg1|cfg4|cfg5
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench_cfgs  # noqa: E402

if __name__ == "__main__":
    for name in sys.argv[1:]:
        print(name, json.dumps(getattr(bench_cfgs, f"measure_{name}")()), flush=True)
