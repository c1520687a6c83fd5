"""Full-size runs of the BASELINE configs on one B200: device time, sweeps,
the device certificate (cc_verify) and -- where host RAM allows -- exact
equality with a CPU checker.

    python tools/scale_check.py forest rmat28 grid4096 [--no-oracle]

Prints one JSON line per config.  The checker is the sequential oracle for
grid4096 and the multi-threaded union-find checker (same output contract as
rem_union_find) for forest / rmat28.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2311_02811_b200 import _lib, engine, graphgen  # noqa: E402
from paper_2311_02811_b200.engine import make_schedule  # noqa: E402


def run(cfg, args):
    spec = (dict(kind="rmat", scale=int(cfg[5:]), edgefactor=16) if cfg.startswith("rmat:")
            else graphgen.CONFIGS[cfg])
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = _lib.Context(0, stream.cuda_stream)
    ctx.set_option(_lib.CC_OPT_SWEEP_VARIANT, args.variant)
    ctx.set_option(_lib.CC_OPT_BUCKET_PIPE, args.pipe)
    ctx.set_option(_lib.CC_OPT_ITEM_ORDER, args.item_order)
    ctx.set_option(_lib.CC_OPT_ITEM_ROWS, args.item_rows)
    ctx.set_option(_lib.CC_OPT_SORT_CHUNK, args.sort_chunk)
    ctx.set_option(_lib.CC_OPT_BUCKET_SHIFT, args.bshift)
    ctx.set_option(_lib.CC_OPT_TILE_SPLIT, args.tsplit)
    if args.store_mode >= 0:
        ctx.set_option(_lib.CC_OPT_STORE_MODE_ATOMIC, args.store_mode)
    ctx.set_option(_lib.CC_OPT_TILE_SHIFT, args.tshift)
    ctx.set_option(_lib.CC_OPT_SWEEP_CTAS, args.sweep_ctas)
    rec = {"store_mode": args.store_mode, "first_scatter": args.first_scatter, "host_loop": args.host_loop,
           "shortcut": args.shortcut, "tsplit": args.tsplit, "tshift": args.tshift, "seed": args.seed, "early_check": args.early_check, "sort_chunk": args.sort_chunk, "bshift": args.bshift, "config": cfg, "variant": args.variant, "pipe": args.pipe,
           "item_order": args.item_order, "item_rows": args.item_rows,
           "sweep_ctas": args.sweep_ctas}
    t0 = time.perf_counter()
    host = None
    if spec["kind"] == "rmat":
        n, m = graphgen.rmat_device(ctx, spec["scale"], spec["edgefactor"], args.seed)
        if args.runs:
            ctx.set_option(_lib.CC_OPT_SORT_CHUNK, -(-m // args.runs))
            rec["runs"] = args.runs
        lay = engine.resolve_layout(args.layout, m, n)
        t1 = time.perf_counter()
        engine.apply_layout(ctx, lay)
    else:
        n, host = graphgen.make(spec, 1, elem_bytes=8)
        m = host.shape[0]
        lay = engine.resolve_layout(args.layout, m, n)
        t1 = time.perf_counter()
        engine.stage_graph(ctx, n, host, lay)
    torch.cuda.synchronize()
    rec.update(n=int(n), m_input=int(m), layout=lay, layout_s=round(time.perf_counter() - t1, 3),
               prep_s=round(time.perf_counter() - t0, 2))
    sched = make_schedule("c2")
    shortcuts = [int(x) for x in str(args.shortcut).split(",")]
    for sc in shortcuts[:-1]:  # extra shortcut settings: timing lines only
        ctx.set_option(_lib.CC_OPT_SHORTCUT, sc)
        runs = [engine.run_staged(ctx, sched, count_changes=False, early_check=args.early_check,
                                  host_loop=bool(args.host_loop))[1] for _ in range(args.repeats)]
        best = min(runs, key=lambda s: s.device_seconds)
        print(json.dumps(dict(rec, shortcut=sc, n=int(n), m_input=int(m), layout=lay,
                              device_s=best.device_seconds,
                              sweeps=[s.sweeps_executed for s in runs],
                              sweep_ms=[round(t * 1e3, 3) for t in best.sweep_seconds],
                              verify=engine.verify_staged(ctx))), flush=True)
    ctx.set_option(_lib.CC_OPT_SHORTCUT, shortcuts[-1])
    rec["shortcut"] = shortcuts[-1]
    runs = []
    for _ in range(args.repeats):
        _, st = engine.run_staged(ctx, sched, count_changes=False, early_check=args.early_check,
                                  first_scatter=bool(args.first_scatter),
                                  host_loop=bool(args.host_loop))
        runs.append(st)
    best = min(runs, key=lambda s: s.device_seconds)
    rec.update(device_s=best.device_seconds, edges_per_s=m / best.device_seconds,
               sweeps=[s.sweeps_executed for s in runs],
               sweep_ms=[round(t * 1e3, 3) for t in best.sweep_seconds],
               b_sweep_gbs=(8 * m + 4 * n) / (sum(best.sweep_seconds) /
                                              len(best.sweep_seconds)) / 1e9)
    rec["verify"] = engine.verify_staged(ctx)
    if not args.no_oracle:
        from oracle import oracle
        labels = np.empty(n, dtype=np.int64)
        _lib.check(ctx.lib.cc_read_labels(ctx.handle, ctypes_ptr(labels), 8))
        ctx.close()
        if host is None:
            t1 = time.perf_counter()
            _, host = graphgen.rmat(spec["scale"], spec["edgefactor"], 1, elem_bytes=4)
            rec["host_gen_s"] = round(time.perf_counter() - t1, 1)
        t1 = time.perf_counter()
        if cfg == "grid4096":
            exp = oracle.rem_union_find(n, host)
            rec["checker"] = "sequential oracle (rem_union_find restatement)"
        else:
            exp = oracle.parallel_components(n, host)
            rec["checker"] = "multi-threaded union-find (rem_union_find output contract)"
        rec["checker_s"] = round(time.perf_counter() - t1, 1)
        rec["exact"] = bool(np.array_equal(labels, exp))
        rec["components"] = int(np.count_nonzero(exp == np.arange(n)))
        del exp, labels
    else:
        ctx.close()
    del host
    print(json.dumps(rec), flush=True)


def ctypes_ptr(a):
    import ctypes
    return ctypes.c_void_p(a.ctypes.data)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--no-oracle", action="store_true")
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--layout", default="auto")
    ap.add_argument("--variant", type=int, default=12)
    ap.add_argument("--pipe", type=int, default=2)
    ap.add_argument("--item-order", type=int, default=0)
    ap.add_argument("--item-rows", type=int, default=1 << 18)
    ap.add_argument("--sort-chunk", type=int, default=1 << 23)
    ap.add_argument("--bshift", type=int, default=15)
    ap.add_argument("--early-check", type=int, default=0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--tsplit", type=int, default=2)
    ap.add_argument("--shortcut", default="1", help="comma list: pointer-jumping passes per sweep")
    ap.add_argument("--first-scatter", type=int, default=0)
    ap.add_argument("--store-mode", type=int, default=-1)
    ap.add_argument("--host-loop", type=int, default=0)
    ap.add_argument("--tshift", type=int, default=24)
    ap.add_argument("--sweep-ctas", type=int, default=0)
    ap.add_argument("--runs", type=int, default=0, help="bucketed run-major: runs (sets sort chunk)")
    args = ap.parse_args()
    for cfg in args.configs:
        run(cfg, args)


if __name__ == "__main__":
    main()
