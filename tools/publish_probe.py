"""A/B of bitmap publishing (CC_OPT_BITS_PUBLISH: the delta-packed bitmap
sweeps set a vertex's bit when a row leaves it at the root label) on RMAT in
the bench's layout: whole runs (graph loop: device ms, sweeps), host-loop
sweep times (then the whole host-loop run's device ms), the
split / rebuild schedule with it, and the uniting check (CC_OPT_CHECK_UNITE)
-- DESIGN 5.31, 5.32.

    python tools/publish_probe.py [--scale 28] [--runs 12] [--publish 0,1,2,0,1]
                                  [--splits -1] [--rebuilds -1]
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
    ap.add_argument("--scale", type=int, default=28)
    ap.add_argument("--runs", type=int, default=12)
    ap.add_argument("--seeds", default="1")
    ap.add_argument("--publish", default="0,1,2,0,1")
    ap.add_argument("--splits", default="-1")
    ap.add_argument("--rebuilds", default="-1")
    ap.add_argument("--canon", default="1")
    ap.add_argument("--shortcut", default="1", help="pointer-jumping passes after each sweep")
    ap.add_argument("--unite", default="0", help="CC_OPT_CHECK_UNITE values")
    ap.add_argument("--defer", default="-1", help="CC_OPT_BITS_DEFER values")
    ap.add_argument("--opts", default="", help="extra options, NAME=V[,NAME=V...] (CC_OPT_ names)")
    ap.add_argument("--item-rows", type=int, default=0, help="CC_OPT_ITEM_ROWS before the layout")
    ap.add_argument("--split-shortcut", default="0",
                    help="pointer-jumping passes before each bitmap part")
    args = ap.parse_args()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = _lib.Context(0, stream.cuda_stream)
    sched = make_schedule("c2")
    ints = lambda s: [int(x) for x in s.split(",")]
    for seed in ints(args.seeds):
        graphgen.rmat_device(ctx, args.scale, 16, seed)
        for name, val in [kv.split("=") for kv in args.opts.split(",") if kv]:
            ctx.set_option(getattr(_lib, "CC_OPT_" + name), int(val))
        if args.item_rows:
            ctx.set_option(_lib.CC_OPT_ITEM_ROWS, args.item_rows)
        engine.apply_layout(ctx, "l2_tiled_check")
        for canon in ints(args.canon):
            ctx.set_option(_lib.CC_OPT_CANON_SWEEP, canon)
            for split in ints(args.splits):
                ctx.set_option(_lib.CC_OPT_SPLIT_SWEEP, split)
                for rebuild in ints(args.rebuilds):
                    ctx.set_option(_lib.CC_OPT_SPLIT_REBUILD, rebuild)
                    for pub, sc, un, ss, df in [(p, k, q, z, d) for p in ints(args.publish)
                                                for k in ints(args.shortcut)
                                                for q in ints(args.unite)
                                                for z in ints(args.split_shortcut)
                                                for d in ints(args.defer)]:
                        ctx.set_option(_lib.CC_OPT_BITS_DEFER, df)
                        ctx.set_option(_lib.CC_OPT_SPLIT_SHORTCUT, ss)
                        ctx.set_option(_lib.CC_OPT_BITS_PUBLISH, pub)
                        ctx.set_option(_lib.CC_OPT_CHECK_UNITE, un)
                        ctx.set_option(_lib.CC_OPT_SHORTCUT, sc)
                        engine.run_staged(ctx, sched, count_changes=False, early_check=True,
                                          sweep_times=False)
                        dev, sweeps = [], []
                        for _ in range(args.runs):
                            _, st = engine.run_staged(ctx, sched, count_changes=False,
                                                      early_check=True, sweep_times=False)
                            dev.append(round(st.device_seconds * 1e3, 2))
                            sweeps.append(st.sweeps_executed)
                        host = []
                        for _ in range(3):
                            _, st = engine.run_staged(ctx, sched, count_changes=False,
                                                      early_check=True, sweep_times=True,
                                                      host_loop=True)
                            host.append([round(x * 1e3, 2) for x in st.sweep_seconds] +
                                        [round(st.device_seconds * 1e3, 2)])
                        print(json.dumps({"scale": args.scale, "seed": seed, "canon": canon,
                                          "split": split, "rebuild": rebuild, "publish": pub, "shortcut": sc, "unite": un, "split_shortcut": ss, "defer": df,
                                          "run_ms": dev, "sweeps": sweeps,
                                          "hostloop_sweep_ms": host,
                                          "verify": engine.verify_staged(ctx)}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
