"""Sweep-1 time of the order-2 sweep variants (CC_OPT_SWEEP_VARIANT) x CTAs
per SM on an RMAT graph staged in the bench's layout (development aid).

    python tools/sweep1_variants.py [--scale 28] [--variants 18,19,20,21] [--ctas 0,3,4] [--runs 3]

Host-driven runs with per-sweep device times; prints one JSON line per
(variant, ctas): sweep-1 ms (median), run ms, sweeps, and labels checked
with cc_verify.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2311_02811_b200 import _lib, engine, graphgen  # noqa: E402
from paper_2311_02811_b200.engine import make_schedule  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=28)
    ap.add_argument("--variants", default="18,19,20,21")
    ap.add_argument("--ctas", default="0")
    ap.add_argument("--runs", type=int, default=3)
    ap.add_argument("--layout", default="auto")
    ap.add_argument("--split", default="-1", help="comma list of CC_OPT_SPLIT_SWEEP (-1 auto)")
    ap.add_argument("--rebuild", default="-1", help="comma list of CC_OPT_SPLIT_REBUILD (-1 auto)")
    ap.add_argument("--shortcut", type=int, default=-1, help="CC_OPT_SPLIT_SHORTCUT (-1: default)")
    ap.add_argument("--masks", default="", help="';'-separated lists of bitmap-part start windows "
                    "(CC_OPT_SPLIT_MASK), e.g. 4,6,8,11;3,5,8,12")
    args = ap.parse_args()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = _lib.Context(0, stream.cuda_stream)
    n, m = graphgen.rmat_device(ctx, args.scale, 16, 1)
    layout = engine.resolve_layout(args.layout, m, n)
    engine.apply_layout(ctx, layout)
    print(json.dumps({"layout_info": ctx.layout_info()}), flush=True)
    if args.shortcut >= 0:
        ctx.set_option(_lib.CC_OPT_SPLIT_SHORTCUT, args.shortcut)
    sched = make_schedule("c2")
    combos = [(v, c_, sp, rb) for v in [int(x) for x in args.variants.split(",")]
              for c_ in [int(x) for x in args.ctas.split(",")]
              for sp in [int(x) for x in args.split.split(",")]
              for rb in [int(x) for x in args.rebuild.split(",")]]
    masks = [sum(1 << int(w) for w in grp.split(",")) for grp in args.masks.split(";") if grp]
    if masks:
        combos = [(combos[0][0], combos[0][1], -1, -1, mk) for mk in masks]
    else:
        combos = [cb + (0,) for cb in combos]
    for var, ctas, split, rebuild, mask in combos:
        if True:
            ctx.set_option(_lib.CC_OPT_SPLIT_MASK, mask)
            ctx.set_option(_lib.CC_OPT_SPLIT_SWEEP, split)
            ctx.set_option(_lib.CC_OPT_SPLIT_REBUILD, rebuild)
            ctx.set_option(_lib.CC_OPT_SWEEP_VARIANT, var)
            ctx.set_option(_lib.CC_OPT_SWEEP_CTAS, ctas)
            kw = dict(count_changes=False, early_check=True, sweep_times=True, host_loop=True)
            engine.run_staged(ctx, sched, **kw)
            s1, run, sweeps = [], [], []
            for _ in range(args.runs):
                _, st = engine.run_staged(ctx, sched, **kw)
                s1.append(st.sweep_seconds[0] * 1e3)
                run.append(st.device_seconds * 1e3)
                sweeps.append(st.sweeps_executed)
            ok = ctypes_verify(ctx)
            b_sweep = 8 * m + 4 * n
            med = statistics.median(s1)
            print(json.dumps({"scale": args.scale, "layout": layout, "variant": var,
                              "ctas": ctas, "split": split, "rebuild": rebuild,
                              "mask": [w for w in range(64) if (mask >> w) & 1], "sweep1_ms": round(med, 3),
                              "sweep1_all": [round(x, 2) for x in s1],
                              "run_ms": [round(x, 2) for x in run], "sweeps": sweeps,
                              "frac": round(b_sweep / (med * 1e-3) / 6.55e12, 4),
                              "verify": ok}), flush=True)
    ctx.close()


def ctypes_verify(ctx):
    import ctypes
    r = ctypes.c_int(-1)
    _lib.check(ctx.lib.cc_verify(ctx.handle, ctypes.byref(r)))
    return r.value


if __name__ == "__main__":
    main()
