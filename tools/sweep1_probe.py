"""How often one sweep converges RMAT-28 (check passes after sweep 1), by
shortcut passes per sweep and layout -- DESIGN 5.19.

    python tools/sweep1_probe.py [--scale 28] [--runs 8] [--shortcuts 1,2,3]
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
    ap.add_argument("--runs", type=int, default=8)
    ap.add_argument("--shortcuts", default="1,2,3")
    ap.add_argument("--layout", default="l2_tiled_check")
    ap.add_argument("--split", default="2")
    ap.add_argument("--ctas", default="0")
    ap.add_argument("--seeds", default="1")
    ap.add_argument("--scales", default=None)
    args = ap.parse_args()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = _lib.Context(0, stream.cuda_stream)
    scales = [int(x) for x in (args.scales or str(args.scale)).split(",")]
    combos = [(sc_, sd, sp) for sc_ in scales for sd in [int(x) for x in args.seeds.split(",")]
              for sp in [int(x) for x in args.split.split(",")]]
    for scale, seed, split in combos:
        args.scale = scale
        ctx.set_option(_lib.CC_OPT_TILE_SPLIT, split)
        n, m = graphgen.rmat_device(ctx, args.scale, 16, seed)
        engine.apply_layout(ctx, args.layout)
        for ctas in [int(x) for x in args.ctas.split(",")]:
            ctx.set_option(_lib.CC_OPT_SWEEP_CTAS, ctas)
            for sc in [int(x) for x in args.shortcuts.split(",")]:
                ctx.set_option(_lib.CC_OPT_SHORTCUT, sc)
                sched = make_schedule("c2")
                engine.run_staged(ctx, sched, count_changes=False, early_check=True,
                                  sweep_times=False)
                sweeps, dev = [], []
                for _ in range(args.runs):
                    _, st = engine.run_staged(ctx, sched, count_changes=False, early_check=True,
                                              sweep_times=False)
                    sweeps.append(st.sweeps_executed)
                    dev.append(st.device_seconds)
                print(json.dumps({"scale": args.scale, "seed": seed, "layout": args.layout,
                                  "split": split,
                                  "ctas": ctas, "shortcut": sc, "sweeps": sweeps,
                                  "ms": [round(x * 1e3, 2) for x in dev],
                                  "verify": engine.verify_staged(ctx)}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
