"""A/B of the bitmap sweeps over the canonical copy (each undirected pair
once, CC_OPT_CANON_SWEEP) vs the dst-bucketed check copy on RMAT in the
bench's layout: whole runs (graph loop: device ms, sweeps), the host-loop
sweep times, and how often one sweep converges -- DESIGN 5.31.

    python tools/canon_sweep_probe.py [--scale 28] [--runs 12] [--seeds 1]
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
    ap.add_argument("--canon", default="0,1,2,0,1")
    ap.add_argument("--splits", default="-1")
    args = ap.parse_args()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = _lib.Context(0, stream.cuda_stream)
    sched = make_schedule("c2")
    for seed in [int(x) for x in args.seeds.split(",")]:
        graphgen.rmat_device(ctx, args.scale, 16, seed)
        engine.apply_layout(ctx, "l2_tiled_check")
        for split in [int(x) for x in args.splits.split(",")]:
            ctx.set_option(_lib.CC_OPT_SPLIT_SWEEP, split)
            for canon in [int(x) for x in args.canon.split(",")]:
                ctx.set_option(_lib.CC_OPT_CANON_SWEEP, canon)
                engine.run_staged(ctx, sched, count_changes=False, early_check=True,
                                  sweep_times=False)
                dev, sweeps = [], []
                for _ in range(args.runs):
                    _, st = engine.run_staged(ctx, sched, count_changes=False, early_check=True,
                                              sweep_times=False)
                    dev.append(round(st.device_seconds * 1e3, 2))
                    sweeps.append(st.sweeps_executed)
                host = []
                for _ in range(3):
                    _, st = engine.run_staged(ctx, sched, count_changes=False, early_check=True,
                                              sweep_times=True, host_loop=True)
                    host.append([round(x * 1e3, 2) for x in st.sweep_seconds])
                print(json.dumps({"scale": args.scale, "seed": seed, "split": split,
                                  "canon_sweep": canon, "run_ms": dev, "sweeps": sweeps,
                                  "hostloop_sweep_ms": host,
                                  "verify": engine.verify_staged(ctx)}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
