"""Quick per-sweep timing matrix for kernel/layout variants (development aid).

    python tools/explore.py [--layouts a,b] [--stores 0,1] [config ...]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2311_02811_b200 import _lib, engine, graphgen  # noqa: E402
from paper_2311_02811_b200.engine import make_schedule  # noqa: E402


def prepare(cfg, layout, chunk, bshift=15, item_rows=1 << 18, bthreads=1024, tshift=23,
            tsplit=1):
    ctx = _lib.Context(0, torch.cuda.current_stream().cuda_stream)
    ctx.set_option(_lib.CC_OPT_SORT_CHUNK, chunk)
    ctx.set_option(_lib.CC_OPT_TILE_SHIFT, tshift)
    ctx.set_option(_lib.CC_OPT_TILE_SPLIT, tsplit)
    ctx.set_option(_lib.CC_OPT_BUCKET_NOSMEM, int(os.environ.get("CC_NOSMEM", "0")))
    ctx.set_option(_lib.CC_OPT_SWEEP_VARIANT, int(os.environ.get("CC_VARIANT", "12")))
    ctx.set_option(_lib.CC_OPT_BUCKET_SHIFT, bshift)
    ctx.set_option(_lib.CC_OPT_ITEM_ROWS, item_rows)
    ctx.set_option(_lib.CC_OPT_BUCKET_THREADS, bthreads)
    spec = graphgen.CONFIGS[cfg]
    if spec["kind"] == "rmat":
        graphgen.rmat_device(ctx, spec["scale"], spec["edgefactor"], 1)
    else:
        n, e = graphgen.make(spec, 1, elem_bytes=4)
        engine.stage_graph(ctx, n, e)
    ts = []
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.check(ctx.lib.cc_reorder_edges(ctx.handle, engine.LAYOUTS[layout]))
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return ctx, min(ts)


def measure(ctx, sched, reps=3, **kw):
    for _ in range(2):
        engine.run_staged(ctx, sched, count_changes=False, sweep_times=False, **kw)
    best, runs = None, []
    for _ in range(reps):
        _, st = engine.run_staged(ctx, sched, count_changes=False, **kw)
        runs.append(st)
        if best is None or st.device_seconds < best.device_seconds:
            best = st
    best.mean_ms = 1e3 * sum(s.device_seconds for s in runs) / len(runs)
    best.sweep_hist = sorted(s.sweeps_executed for s in runs)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["rmat22", "grid4096", "er"])
    ap.add_argument("--layouts", default="input")
    ap.add_argument("--stores", default="1")
    ap.add_argument("--chunk", type=int, default=1 << 23)
    ap.add_argument("--atomic", type=int, default=1)
    ap.add_argument("--bshift", type=int, default=15)
    ap.add_argument("--item-rows", type=int, default=1 << 18)
    ap.add_argument("--bthreads", type=int, default=1024)
    ap.add_argument("--no-fs", action="store_true")
    ap.add_argument("--shortcut", default="0")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--tshift", type=int, default=23)
    ap.add_argument("--tsplit", default="1")
    a = ap.parse_args()
    for cfg in a.configs:
        for layout, tsplit in [(lay, int(t)) for lay in a.layouts.split(",")
                               for t in a.tsplit.split(",")]:
            ctx, tr = prepare(cfg, layout, a.chunk, a.bshift, a.item_rows, a.bthreads, a.tshift,
                              tsplit)
            print(f"# {cfg} layout={layout} tsplit={tsplit} tshift={a.tshift} chunk={a.chunk}",
                  flush=True)
            for sm in map(int, a.stores.split(",")):
                ctx.set_option(_lib.CC_OPT_STORE_MODE_ATOMIC if a.atomic else
                               _lib.CC_OPT_STORE_MODE_PLAIN, sm)
                for sc in map(int, a.shortcut.split(",")):
                    ctx.set_option(_lib.CC_OPT_SHORTCUT, sc)
                    for fs in ((False,) if a.no_fs else (False, True)):
                        st = measure(ctx, make_schedule("c2", atomic=bool(a.atomic)), a.reps,
                                     early_check=False, first_scatter=fs)
                        print(f"{cfg:9s} layout={layout:12s} reorder={tr*1e3:6.2f}ms store={sm} "
                              f"shortcut={sc} first_scatter={fs:d} "
                              f"best={st.device_seconds*1e3:8.3f}ms mean={st.mean_ms:8.3f}ms "
                              f"sweeps={st.sweep_hist} "
                              f"sweep_ms={[round(t*1e3,3) for t in st.sweep_seconds]}",
                              flush=True)
            ctx.close()


if __name__ == "__main__":
    main()
