"""Where the RMAT-28 drop-in call's time goes (DESIGN 5.20): staging alone,
the default one-shot layout, and chunk-sorted staging with sweep 1 streamed
behind the copy.

    python tools/e2e28_probe.py [--scale 28]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_02811_b200 import _lib, engine, graphgen, run_contour  # noqa: E402
from paper_2311_02811_b200.engine import make_schedule  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=28)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--cases", default="stage_input,stage_chunk,auto,chunk_sorted,auto_nocount,chunk_nocount")
    ap.add_argument("--host-sub", default="0", help="comma list of CC_OPT_HOST_SUB (0: default)")
    ap.add_argument("--host-nt", default="0", help="comma list of CC_OPT_HOST_NT")
    args = ap.parse_args()
    ctx = _lib.Context(0)
    n, m = graphgen.rmat_device(ctx, args.scale, 16, 1)
    t = time.perf_counter()
    e = graphgen.read_edges(ctx, 8)
    print(json.dumps({"read_edges_s": round(time.perf_counter() - t, 2), "bytes": e.nbytes}),
          flush=True)
    _lib.check(ctx.lib.cc_run(ctx.handle, None, 0, 0, None, 8, None)) if False else None
    # reference labels from a device-resident run
    engine.apply_layout(ctx, engine.resolve_layout("auto", m, n))
    ref = np.empty(n, dtype=np.int64)
    engine.run_staged(ctx, make_schedule("c2"), count_changes=False, labels_out=ref)
    ctx.close()
    del ctx
    sched = make_schedule("c2")
    combos = [(case, hs, nt) for hs in args.host_sub.split(",") for nt in args.host_nt.split(",")
              for case in args.cases.split(",")]
    for case, hs, nt in combos:
        c0 = engine._context(0)
        if int(hs):
            c0.set_option(_lib.CC_OPT_HOST_SUB, int(hs))
        c0.set_option(_lib.CC_OPT_HOST_NT, int(nt))
        ts, extra = [], {}
        for _ in range(args.reps):
            c2 = engine._context(0)
            t = time.perf_counter()
            if case in ("host_nolabels", "host_labels", "host_labels32"):
                out = None
                if case == "host_labels":
                    out = np.empty(n, dtype=np.int64)
                elif case == "host_labels32":
                    out = np.empty(n, dtype=np.int32)
                t = time.perf_counter()
                _, st = engine.run_host(c2, n, e, sched, count_changes=False, labels_out=out)
                extra = {"sweeps": st.sweeps_executed, "device_s": round(st.device_seconds, 3)}
            elif case == "stage_input":
                engine.stage_graph(c2, n, e, "input")
            elif case == "stage_chunk":
                engine.stage_graph(c2, n, e, "chunk_sorted")
            else:
                layout = {"auto": "auto", "chunk_sorted": "chunk_sorted", "auto_nocount": "auto",
                          "chunk_nocount": "chunk_sorted"}[case]
                lab, st = run_contour((n, e), sched, layout=layout,
                                      count_changes="nocount" not in case)
                torch.cuda.synchronize()
                ts.append(round(time.perf_counter() - t, 3))  # (the check below is untimed)
                extra = {"sweeps": st.sweeps_executed, "by": st.converged_by,
                         "sweep_ms": [round(x * 1e3, 1) for x in st.sweep_seconds],
                         "exact": bool(np.array_equal(lab, ref))}
                del lab
                continue
            torch.cuda.synchronize()
            ts.append(round(time.perf_counter() - t, 3))
        print(json.dumps({"case": case, "host_sub": int(hs), "host_nt": int(nt), "s": ts,
                          **extra}), flush=True)


if __name__ == "__main__":
    main()
