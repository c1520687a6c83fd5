"""Run one config through the host loop so ncu can see every sweep launch
(development aid): python tools/profile_config.py forest [layout]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2311_02811_b200 import _lib, engine, graphgen  # noqa: E402
from paper_2311_02811_b200.engine import make_schedule  # noqa: E402


def main():
    cfg = sys.argv[1]
    layout = sys.argv[2] if len(sys.argv) > 2 else "auto"
    ctx = _lib.Context(0, torch.cuda.current_stream().cuda_stream)
    ctx.set_option(_lib.CC_OPT_SWEEP_VARIANT, int(os.environ.get("CC_VARIANT", "12")))
    ctx.set_option(_lib.CC_OPT_BUCKET_PIPE, int(os.environ.get("CC_PIPE", "1")))
    spec = graphgen.CONFIGS[cfg]
    if spec["kind"] == "rmat":
        n, m = graphgen.rmat_device(ctx, spec["scale"], spec["edgefactor"], 1)
        lay = engine.resolve_layout(layout, m, n)
        engine.apply_layout(ctx, lay)
    else:
        n, e = graphgen.make(spec, 1, elem_bytes=8)
        lay = engine.resolve_layout(layout, e.shape[0], n)
        engine.stage_graph(ctx, n, e, lay)
        del e
    for name, val in [kv.split("=") for kv in os.environ.get("CC_OPTS", "").split(",") if kv]:
        ctx.set_option(getattr(_lib, "CC_OPT_" + name), int(val))  # e.g. CC_OPTS=BITS_DEFER=4
    check = os.environ.get("CC_CHECK", "0") == "1"
    _, st = engine.run_staged(ctx, make_schedule("c2"), count_changes=False, early_check=check,
                              host_loop=True)
    print(cfg, lay, st.sweeps_executed, [round(t * 1e3, 2) for t in st.sweep_seconds])


if __name__ == "__main__":
    main()
