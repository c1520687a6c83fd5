"""GPU FastSV baseline.

``fastsv(g)`` mirrors /root/reference/pkg/src/minmapcc/baselines.py:81-131:
synchronous stochastic + aggressive hooking and shortcutting until the
grandparent array stops changing, returning normalized labels and an
IterationStats whose per-iteration counts equal the reference's (atomic-min
proposals are order-independent).  Gives the paper's "speedup vs FastSV"
comparison on the same device and the same staged edges.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .engine import IterationStats, _context, _unpack_graph, stage_graph


def fastsv_staged(ctx: _lib.Context, labels_out: np.ndarray | None = None,
                  sweep_times: bool = True, cap: int | None = None):
    n = ctx.n
    cap = n + 2 if cap is None else int(cap)
    capacity = max(1, min(cap, 1 << 16))
    changed = np.zeros(capacity, dtype=np.int64)
    secs = np.zeros(capacity, dtype=np.float64)
    st = _lib.CCStats()
    st.capacity = capacity
    st.changed_per_sweep = changed.ctypes.data_as(_lib._I64P)
    st.sweep_seconds = secs.ctypes.data_as(_lib._DBLP)
    out, eb = None, 8
    if labels_out is not None:
        out, eb = ctypes.c_void_p(labels_out.ctypes.data), labels_out.dtype.itemsize
    _lib.check(ctx.lib.cc_fastsv(ctx.handle, cap, out, eb, ctypes.byref(st),
                                 _lib.CC_RUN_SWEEP_TIMES if sweep_times else 0))
    k = int(st.sweeps_executed)
    return labels_out, IterationStats(
        sweeps_executed=k, sweeps_until_stable=int(st.sweeps_until_stable),
        changed_per_sweep=[int(x) for x in changed[:min(k, capacity)]],
        converged_by="grandparent-stable",
        sweep_seconds=secs[:min(k, capacity)].tolist(), device_seconds=float(st.converge_seconds))


def fastsv(g, *, device: int = 0, layout: str = "auto"):
    """baselines.py:81-131 on the GPU: (labels int64, IterationStats)."""
    n, edges = _unpack_graph(g)
    ctx = _context(device)
    stage_graph(ctx, n, edges, layout)
    labels = np.empty(n, dtype=np.int64)
    _, stats = fastsv_staged(ctx, labels)
    return labels, stats
