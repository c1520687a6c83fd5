"""Repeated drop-in calls on one read-only RMAT edge array (what the
reference's harness does with a frozen Graph, bench.py:176-179): call 1
stages (chunk-sorted, sweep 1 streamed behind the copy), call 2 upgrades the
resident graph in place to layout 6, later calls run from HBM.

    python tools/frozen_probe.py [--scale 28] [--calls 5]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2311_02811_b200 import _lib, engine, graphgen, run_contour  # noqa: E402
from paper_2311_02811_b200.engine import make_schedule  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=28)
    ap.add_argument("--calls", type=int, default=5)
    args = ap.parse_args()
    ctx = _lib.Context(0)
    n, m = graphgen.rmat_device(ctx, args.scale, 16, 1)
    e = graphgen.read_edges(ctx, 8)
    ctx.close()
    e.flags.writeable = False
    ts, layouts, first = [], [], None
    for _ in range(args.calls):
        t = time.perf_counter()
        lab, st = run_contour((n, e), make_schedule("c2"))
        ts.append(round(time.perf_counter() - t, 3))
        layouts.append(engine._context(0).layout_info()["layout"])
        if first is None:
            first = lab
        elif not np.array_equal(lab, first):
            raise SystemExit("labels differ between calls")
        del lab
    print(json.dumps({"scale": args.scale, "m": int(m), "call_s": ts, "layout": layouts,
                      "edges_per_s_last": int(m) / ts[-1]}))


if __name__ == "__main__":
    main()
