"""Probe (development aid): the default drop-in call run_contour(g, schedule)
(exact changed_per_sweep + early check, the reference's semantics) from host
memory vs the bench's e2e path (count_changes=False) on RMAT-22."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_02811_b200 import graphgen, make_schedule, run_contour  # noqa: E402


def main():
    n, e = graphgen.rmat(22, 16, 1, elem_bytes=4)
    pe = torch.empty((e.shape[0], 2), dtype=torch.int32, pin_memory=True)
    pe.numpy()[:] = e
    for label, kw in (("default (count_changes=True, early_check=True)", {}),
                      ("count_changes=False, early_check=True", dict(count_changes=False)),
                      ("count_changes=False, early_check=False",
                       dict(count_changes=False, early_check=False))):
        frozen = e.astype(np.int64)
        frozen.flags.writeable = False  # as the reference's Graph.edges (graph.py:82-83)
        for src, arr in (("pinned", pe.numpy()), ("pageable int64", e.astype(np.int64)),
                         ("frozen int64, repeat", frozen)):
            for _ in range(2):
                run_contour((n, arr), make_schedule("c2"), **kw)
            ts = []
            for _ in range(5):
                t0 = time.perf_counter()
                labels, st = run_contour((n, arr), make_schedule("c2"), **kw)
                ts.append(time.perf_counter() - t0)
            print(f"{label:48s} {src:15s} wall {1e3 * min(ts):7.2f} ms  sweeps "
                  f"{st.sweeps_executed} changed {st.changed_per_sweep} by {st.converged_by}",
                  flush=True)


if __name__ == "__main__":
    main()
