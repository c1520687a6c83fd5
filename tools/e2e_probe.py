"""Break the end-to-end leg of bench.py into its parts (development aid):
pinned H2D staging, the solve, the label read-back."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_02811_b200 import _lib, engine, graphgen  # noqa: E402
from paper_2311_02811_b200.engine import make_schedule  # noqa: E402


def timed(stream, fn, reps=5):
    out = []
    for i in range(reps + 2):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        if i >= 2:
            out.append((a.elapsed_time(b), (time.perf_counter() - t0) * 1e3))
    return [round(sum(x[k] for x in out) / len(out), 3) for k in (0, 1)]


def main():
    layout = sys.argv[1] if len(sys.argv) > 1 else "chunk_sorted"
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = _lib.Context(0, stream.cuda_stream)
    t = torch.empty((1 << 27, 2), dtype=torch.int32, pin_memory=True)
    n, _ = graphgen.rmat(22, 16, 1, elem_bytes=4, out=t.numpy())
    e = t.numpy()
    lab64 = torch.empty(n, dtype=torch.int64, pin_memory=True).numpy()
    lab32 = torch.empty(n, dtype=torch.int32, pin_memory=True).numpy()
    sched = make_schedule("c2")
    kw = dict(count_changes=False, early_check=True, sweep_times=False)
    print("stage          [event ms, wall ms]", timed(stream, lambda: engine.stage_graph(ctx, n, e, layout)))
    print("run (no out)   ", timed(stream, lambda: engine.run_staged(ctx, sched, **kw)))
    print("run + int64 out", timed(stream, lambda: engine.run_staged(ctx, sched, labels_out=lab64, **kw)))
    print("run + int32 out", timed(stream, lambda: engine.run_staged(ctx, sched, labels_out=lab32, **kw)))

    def full():
        engine.stage_graph(ctx, n, e, layout)
        engine.run_staged(ctx, sched, labels_out=lab64, **kw)
    print("stage+run+out  ", timed(stream, full))
    d = torch.empty(e.size, dtype=torch.int32, device="cuda")
    tt = torch.from_numpy(e.reshape(-1))
    print("raw H2D 1 GiB  ", timed(stream, lambda: d.copy_(tt, non_blocking=True)))
    ctx.close()


if __name__ == "__main__":
    main()
