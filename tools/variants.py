"""Per-variant device time on the staged configs (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2311_02811_b200 import _lib, engine, graphgen  # noqa: E402
from paper_2311_02811_b200.engine import make_schedule  # noqa: E402


def main():
    cfgs = sys.argv[1:] or ["rmat22", "grid4096"]
    for cfg in cfgs:
        ctx = _lib.Context(0, torch.cuda.current_stream().cuda_stream)
        spec = graphgen.CONFIGS[cfg]
        if spec["kind"] == "rmat":
            n, m = graphgen.rmat_device(ctx, spec["scale"], spec["edgefactor"], 1)
            engine.apply_layout(ctx, engine.resolve_layout("auto", m, n))
        else:
            n, e = graphgen.make(spec, 1, elem_bytes=4)
            engine.stage_graph(ctx, n, e)
        for v, sync in (("C-2", False), ("C-1", False), ("C-m", False), ("C-11mm", False),
                        ("C-1m1m", False), ("C-2", True), ("C-Syn", True), ("C-m", True)):
            sched = make_schedule(v, 1024, sync=sync)
            kw = dict(count_changes=sync, early_check=sync)
            engine.run_staged(ctx, sched, **kw)
            best = None
            for _ in range(3):
                _, st = engine.run_staged(ctx, sched, **kw)
                if best is None or st.device_seconds < best.device_seconds:
                    best = st
            print(f"{cfg:9s} {v:7s} sync={sync:d} {best.device_seconds*1e3:9.3f} ms "
                  f"sweeps={best.sweeps_executed} "
                  f"sweep_ms={[round(t*1e3, 3) for t in best.sweep_seconds][:12]}", flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
