"""Variance of the RMAT-28 drop-in call's parts (DESIGN 5.20): staging of
the pageable int64 rows alone, and reading the 2^28 int64 labels back into a
fresh numpy array, repeated."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2311_02811_b200 import _lib, engine, graphgen, run_contour  # noqa: E402
from paper_2311_02811_b200.engine import make_schedule  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    ctx = _lib.Context(0)
    n, m = graphgen.rmat_device(ctx, 28, 16, 1)
    e = graphgen.read_edges(ctx, 8)
    ctx.close()
    c2 = engine._context(0)
    st, rd, rc, st8 = [], [], [], []
    for _ in range(reps):  # alternating: 7-byte packed rows / uint32 pairs on the link
        for pack, out in ((1, st), (0, st8)):
            c2.set_option(_lib.CC_OPT_LINK_PACK, pack)
            t = time.perf_counter()
            engine.stage_graph(c2, n, e, "input")
            out.append(round(time.perf_counter() - t, 3))
    c2.set_option(_lib.CC_OPT_LINK_PACK, 1)
    for _ in range(reps):
        t = time.perf_counter()
        lab = np.empty(n, dtype=np.int64)
        _lib.check(c2.lib.cc_read_labels(c2.handle, lab.ctypes.data, 8))
        rd.append(round(time.perf_counter() - t, 3))
        del lab
    for _ in range(reps):
        t = time.perf_counter()
        lab, _ = run_contour((n, e), make_schedule("c2"))
        rc.append(round(time.perf_counter() - t, 3))
        del lab
    print(json.dumps({"stage_input_uint32_pairs_s": st8, "stage_input_packed_s": st,
                      "read_labels_fresh_s": rd, "run_contour_s": rc}))


if __name__ == "__main__":
    main()
