"""The forest config (configs[3]) on the relabeled layout with the rows of each
relabel block interleaved (CC_OPT_RELABEL_INTERLEAVE), development aid:
device time, sweeps, cc_verify per stride.

    python tools/forest_probe.py [--strides 0,8,32,128] [--block 24] [--runs 3] [--components N]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2311_02811_b200 import _lib, engine, graphgen  # noqa: E402
from paper_2311_02811_b200.engine import make_schedule  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--strides", default="0,8,32,128")
    ap.add_argument("--blocks", default="24")
    ap.add_argument("--runs", type=int, default=3)
    ap.add_argument("--components", type=int, default=0, help="0: the full config")
    args = ap.parse_args()
    spec = dict(graphgen.CONFIGS["forest"])
    if args.components:
        spec["components"] = args.components
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = _lib.Context(0, stream.cuda_stream)
    n, host = graphgen.make(spec, 1, elem_bytes=8)
    engine.stage_graph(ctx, n, host, "input")
    del host
    sched = make_schedule("c2")
    for blk in [int(x) for x in args.blocks.split(",")]:
        for st_ in [int(x) for x in args.strides.split(",")]:
            ctx.set_option(_lib.CC_OPT_RELABEL_INTERLEAVE, st_)
            ctx.set_option(_lib.CC_OPT_RELABEL_BLOCK, blk)
            _lib.check(ctx.lib.cc_reorder_edges(ctx.handle, engine.LAYOUTS["relabel"]))
            engine.run_staged(ctx, sched, count_changes=False, sweep_times=False)
            runs = [engine.run_staged(ctx, sched, count_changes=False, sweep_times=True)[1]
                    for _ in range(args.runs)]
            best = min(runs, key=lambda s: s.device_seconds)
            print(json.dumps({"n": n, "block": blk, "stride": st_,
                              "layout": ctx.layout_info()["layout"],
                              "device_ms": round(best.device_seconds * 1e3, 2),
                              "sweeps": [s.sweeps_executed for s in runs],
                              "sweep_ms": [round(t * 1e3, 2) for t in best.sweep_seconds],
                              "verify": engine.verify_staged(ctx)}), flush=True)


if __name__ == "__main__":
    main()
