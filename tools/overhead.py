"""Host overhead of one cc_run (development aid): wall time per call vs the
device time of the run, for the graph loop with/without per-sweep records."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2311_02811_b200 import _lib, engine, graphgen  # noqa: E402
from paper_2311_02811_b200.engine import make_schedule  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "rmat22"
    layout = sys.argv[2] if len(sys.argv) > 2 else "chunk_sorted"
    check = len(sys.argv) > 3 and sys.argv[3] == "check"
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = _lib.Context(0, stream.cuda_stream)
    spec = graphgen.CONFIGS[cfg]
    if spec["kind"] == "rmat":
        n, m = graphgen.rmat_device(ctx, spec["scale"], spec["edgefactor"], 1)
        engine.apply_layout(ctx, layout)
    else:
        n, e = graphgen.make(spec, 1, elem_bytes=4)
        engine.stage_graph(ctx, n, e)
    sched = make_schedule("c2")
    for times in (True, False):
        for _ in range(3):
            engine.run_staged(ctx, sched, count_changes=False, early_check=check,
                              sweep_times=times)
        walls, devs = [], []
        for _ in range(20):
            t0 = time.perf_counter()
            _, st = engine.run_staged(ctx, sched, count_changes=False, early_check=check,
                                      sweep_times=times)
            walls.append(time.perf_counter() - t0)
            devs.append(st.device_seconds)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(20):
            engine.run_staged(ctx, sched, count_changes=False, early_check=check,
                              sweep_times=times)
        ev1.record(stream)
        torch.cuda.synchronize()
        print(f"{cfg} sweep_times={times}: wall/run {1e3*sum(walls)/20:.3f} ms, device/run "
              f"{1e3*sum(devs)/20:.3f} ms, events/run {ev0.elapsed_time(ev1)/20:.3f} ms", flush=True)
    # raw C call, no Python wrapper work
    import ctypes
    st = _lib.CCStats()
    sc = engine._cc_schedule(sched)
    t0 = time.perf_counter()
    for _ in range(20):
        _lib.check(ctx.lib.cc_run(ctx.handle, ctypes.byref(sc), _lib.CC_RUN_EARLY_CHECK if check else 0,
                                  n + 2, None, 8, ctypes.byref(st)))
    print(f"{cfg} raw cc_run: wall/run {1e3*(time.perf_counter()-t0)/20:.3f} ms, "
          f"device {1e3*st.converge_seconds:.3f} ms", flush=True)


if __name__ == "__main__":
    main()
