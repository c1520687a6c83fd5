"""Probe (development aid): work-item order of the dst-bucketed layout vs the
number of sweeps RMAT needs -- does a src-major item order (every bucket's
j-th src slice together) converge in one sweep like chunk-sorted rows?

    python tools/order_probe.py [--scales 20,21,22,23] [--seeds 1,2,3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2311_02811_b200 import _lib, engine, graphgen  # noqa: E402
from paper_2311_02811_b200.engine import make_schedule  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scales", default="20,21,22,23")
    ap.add_argument("--seeds", default="1,2,3")
    ap.add_argument("--orders", default="0,3")
    ap.add_argument("--item-rows", default="65536,131072,262144")
    ap.add_argument("--layouts", default="dst_bucketed")
    ap.add_argument("--nosmem", default="0", help="comma list: 1 = dst labels from global memory")
    ap.add_argument("--runs", default="1", help="comma list: input-order runs (item order 1/2)")
    ap.add_argument("--checks", default="0,1")
    ap.add_argument("--bshifts", default="15")
    a = ap.parse_args()
    sched = make_schedule("c2")
    for scale in map(int, a.scales.split(",")):
        for seed in map(int, a.seeds.split(",")):
            stream = torch.cuda.current_stream().cuda_stream
            ctx = _lib.Context(0, stream)
            _, m = graphgen.rmat_device(ctx, scale, 16, seed)
            for layout in a.layouts.split(","):
                for order, rows, nosmem, nruns, bsh in [
                        (o, r, ns, ru, bs) for o in map(int, a.orders.split(","))
                        for r in map(int, a.item_rows.split(","))
                        for ns in map(int, a.nosmem.split(","))
                        for ru in map(int, a.runs.split(","))
                        for bs in map(int, a.bshifts.split(","))]:
                    if True:
                        ctx.set_option(_lib.CC_OPT_BUCKET_SHIFT, bsh)
                        ctx.set_option(_lib.CC_OPT_SORT_CHUNK, -(-m // nruns) if nruns > 1 else 1 << 23)
                        ctx.set_option(_lib.CC_OPT_BUCKET_NOSMEM, nosmem)
                        ctx.set_option(_lib.CC_OPT_ITEM_ORDER, order)
                        ctx.set_option(_lib.CC_OPT_ITEM_ROWS, rows)
                        engine.apply_layout(ctx, layout)
                        torch.cuda.synchronize()
                        for check in [bool(int(x)) for x in a.checks.split(",")]:
                            for _ in range(2):
                                engine.run_staged(ctx, sched, count_changes=False,
                                                  early_check=check, sweep_times=False)
                            runs = [engine.run_staged(ctx, sched, count_changes=False,
                                                      early_check=check)[1] for _ in range(3)]
                            best = min(runs, key=lambda s: s.device_seconds)
                            ok = engine.verify_staged(ctx) == 0
                            print(f"scale={scale} seed={seed} {layout} order={order} "
                                  f"item_rows={rows} nosmem={nosmem} runs={nruns} bshift={bsh} check={int(check)} "
                                  f"ms={best.device_seconds * 1e3:.3f} "
                                  f"sweeps={[s.sweeps_executed for s in runs]} "
                                  f"sweep_ms={[round(t * 1e3, 3) for t in best.sweep_seconds]} "
                                  f"verified={ok}", flush=True)
            ctx.close()


if __name__ == "__main__":
    main()
