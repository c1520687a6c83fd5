"""Drop-in host mirror of the reference engine's hot-path API.

Mirrors /root/reference/pkg/src/minmapcc/engine.py: the same ``Schedule``,
``make_schedule``, ``IterationStats`` and ``run_contour(g, schedule,
threads=1, seed=None)`` signature and return types, so the reference's
callers (bench.py:136-137, cli.py:126, its tests) can import
``run_contour``/``make_schedule`` from here instead.  Every sweep runs on the
B200 through libcontour.so (include/contour.h); there is no CPU path.
"""

from __future__ import annotations

import ctypes
import threading
import weakref
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .errors import IterationCapExceeded

__all__ = [
    "LabelArray", "Schedule", "IterationStats", "ForestDiagnostics", "VARIANTS",
    "canonical_variant", "conditional_min_assign", "make_schedule", "run_contour", "mm_order",
    "early_convergence_check", "forest_diagnostics", "IterationCapExceeded", "stage_graph",
]

LabelArray = np.ndarray  # (n,) int64, as engine.py:44

VARIANTS = ("C-Syn", "C-1", "C-2", "C-m", "C-11mm", "C-1m1m")  # engine.py:46
_ORDERED_VARIANTS = {"C-m", "C-11mm", "C-1m1m"}                 # engine.py:48
_VARIANT_CODE = {v: i for i, v in enumerate(VARIANTS)}          # include/contour.h CC_VAR_*


@dataclass(frozen=True)
class Schedule:
    """Per-iteration operator orders plus execution-mode flags (engine.py:51-74)."""

    variant: str
    high_order: int = 1024
    warmup: int = 2
    sync: bool = False
    atomic: bool = True

    def order_for(self, sweep: int) -> int:
        v = self.variant
        if v in ("C-2", "C-Syn"):
            return 2
        if v == "C-1":
            return 1
        if v == "C-m":
            return self.high_order
        if v == "C-11mm":
            return 1 if sweep <= self.warmup else self.high_order
        if v == "C-1m1m":
            return 1 if sweep % 2 == 1 else self.high_order
        raise ValueError(f"unknown variant '{v}'")


@dataclass
class IterationStats:
    """Sweep accounting for one run (engine.py:77-90).

    ``sweep_seconds`` are CUDA-event device times per sweep.  With
    ``count_changes=False`` the entries of ``changed_per_sweep`` are -1 for
    "changed, not counted" and 0 for the final no-change sweep.
    ``device_seconds`` (extra) is the device time from label init to the
    compressed labels.
    """

    sweeps_executed: int
    sweeps_until_stable: int
    changed_per_sweep: list = field(default_factory=list)
    converged_by: str = "change-flag"
    sweep_seconds: list = field(default_factory=list)
    device_seconds: float = 0.0


_ALIAS = {  # engine.py:108-115
    "csyn": "C-Syn", "c-syn": "C-Syn", "c1": "C-1", "c-1": "C-1", "c2": "C-2", "c-2": "C-2",
    "cm": "C-m", "c-m": "C-m", "c11mm": "C-11mm", "c-11mm": "C-11mm",
    "c1m1m": "C-1m1m", "c-1m1m": "C-1m1m",
}


def canonical_variant(name: str) -> str:
    canon = _ALIAS.get(name.strip().lower())
    if canon is None:
        raise ValueError(f"unknown variant '{name}' (choose from {', '.join(VARIANTS)})")
    return canon


def make_schedule(variant: str, high_order: int = 1024, warmup: int = 2, *,
                  sync: Optional[bool] = None, atomic: bool = True) -> Schedule:
    """engine.py:125-152, same validation and ValueError messages."""
    canon = canonical_variant(variant)
    if canon in _ORDERED_VARIANTS and high_order < 2:
        raise ValueError(f"{canon} requires high_order >= 2, got {high_order}")
    if warmup < 1:
        raise ValueError(f"warmup must be >= 1, got {warmup}")
    if canon == "C-Syn":
        if sync is False:
            raise ValueError("C-Syn always runs synchronously")
        sync = True
    elif sync is None:
        sync = False
    return Schedule(variant=canon, high_order=high_order, warmup=warmup, sync=sync, atomic=atomic)


def _cc_schedule(s: Schedule) -> _lib.CCSchedule:
    return _lib.CCSchedule(_VARIANT_CODE[canonical_variant(s.variant)], int(s.high_order),
                           int(s.warmup), int(bool(s.sync)), int(bool(s.atomic)))


_tls = threading.local()


def _context(device: int) -> _lib.Context:
    """One cached context per (caller thread, device) -- SPEC.md:212 reentrancy."""
    cache = getattr(_tls, "ctx", None)
    if cache is None:
        cache = _tls.ctx = {}
    ctx = cache.get(device)
    if ctx is None:
        ctx = cache[device] = _lib.Context(device)
    return ctx


def _unpack_graph(g):
    if isinstance(g, tuple) and len(g) == 2:
        n, edges = g
    else:
        n, edges = g.n, g.edges  # the duck-typed contract of engine.py:268-270
    return int(n), edges


LAYOUTS = {"input": 0, "src_sorted": 1, "chunk_sorted": 2, "dst_bucketed": 3, "l2_tiled": 4,
           "hybrid": 5, "l2_tiled_check": 6, "relabel": 7}
AUTO_SORT_MIN_ROWS = 1 << 16


AUTO_L2_LABEL_BYTES = 96 << 20  # the 126 MB L2 holds the labels plus the edge stream's lines


AUTO_HYBRID_MIN_DEGREE = 8  # rows per vertex from which the bucketed copy pays (measured)


def resolve_layout(layout: str, m: int, n: int = 0, resident: bool = True,
                   copies: bool = True, counted: bool = True) -> str:
    """"auto": input order below 2^16 rows (ER n=65,536, 524,282 rows: 0.088 ms
    per run chunk-sorted vs 0.11 ms in input order); while the label array fits
    comfortably in L2, chunk-sorted staging (it hides under the host->device
    copy, ~2x faster sweeps) -- plus, for graphs staged once and run from HBM
    (``resident``) with >= 8 rows per vertex and m < 2^31, the dst-bucketed
    copy of the hybrid layout (later sweeps and the early check gather dst
    labels from shared memory: RMAT-20..23 12-17 % faster per run; grid and
    ER are slower with it).  Label arrays beyond L2: L2-window tiles, with
    the bitmap check copy for resident dense graphs (m >= 4n, RMAT-28: 57 vs
    77-83 ms per run, DESIGN 5.19); one-shot runs from host memory
    (``resident=False``) of dense graphs stay chunk-sorted, so sweep 1
    streams behind the copy and the tiling (0.5 s at RMAT-28) is skipped
    (DESIGN 5.20).  ``copies=False``: no extra copy of the rows (the
    multi-GPU shards: their fused exchange walks one row array).
    ``counted=False`` (the graph will be run without exact change counts,
    ``run_staged(count_changes=False)``): dense resident graphs of at least
    2^20 vertices get layout 6 also while their labels fit in L2 -- with
    n/16-vertex windows their sweep 1 is split and the run ends on the uniting
    check (RMAT-22 0.51 vs 0.82 ms per run on the hybrid layout, DESIGN 5.35);
    counted runs keep the hybrid layout (plain check: 0.82 vs 1.28 ms)."""
    if layout == "auto":
        if m < AUTO_SORT_MIN_ROWS:
            return "input"
        if 4 * n > AUTO_L2_LABEL_BYTES:
            if not resident:
                return "chunk_sorted" if m >= 4 * n else "l2_tiled"
            if m >= 4 * n:
                return "l2_tiled_check" if copies else "l2_tiled"
            # sparse (the forest): first-appearance relabeling, which falls
            # back to the tiles when the input order carries no locality
            return "relabel" if copies and m < (1 << 31) else "l2_tiled"
        if resident and copies and m < (1 << 31) and m >= AUTO_HYBRID_MIN_DEGREE * n:
            return "l2_tiled_check" if (not counted and n >= (1 << 20)) else "hybrid"
        return "chunk_sorted"
    if layout not in LAYOUTS:
        raise ValueError(f"unknown edge layout '{layout}'")
    return layout


def _host_edges(edges) -> np.ndarray:
    e = np.asarray(edges)
    if e.size == 0:
        e = np.zeros((0, 2), dtype=np.int64)
    if e.ndim != 2 or e.shape[1] != 2:
        raise ValueError("edges must be a sequence of (u, v) pairs")
    if e.dtype not in (np.int32, np.int64):
        e = e.astype(np.int64)
    return np.ascontiguousarray(e)


def apply_layout(ctx: _lib.Context, layout: str) -> None:
    """Reorder rows already staged in HBM (e.g. generated on device) into
    ``layout``; "hybrid" = chunk-sorted rows plus a dst-bucketed copy."""
    if layout == "hybrid":
        _lib.check(ctx.lib.cc_reorder_edges(ctx.handle, LAYOUTS["chunk_sorted"]))
    if LAYOUTS[layout]:
        _lib.check(ctx.lib.cc_reorder_edges(ctx.handle, LAYOUTS[layout]))


def stage_graph(ctx: _lib.Context, n: int, edges, layout: str = "auto",
                copies: bool = True) -> None:
    """Stage an (m, 2) edge array (numpy int32/int64 on the host, or a CUDA
    tensor) as packed uint32 SoA in HBM, with the graph.py:73-79 range check.

    ``layout`` is the staging-time edge order -- the analogue of the
    reference building CSR at Graph construction (graph.py:80,109-122):
    "input" keeps the caller's order, "chunk_sorted" radix-sorts every 2^23-row
    chunk by src as it lands (overlapped with the next chunk's copy),
    "src_sorted" sorts all rows by src afterwards, "auto" picks."""
    ctx.staged = None  # the context's edges change: no resident graph to reuse
    m_rows = int(edges.shape[0]) if hasattr(edges, "shape") and len(edges.shape) == 2 \
        else len(edges)
    layout = resolve_layout(layout, m_rows, n, copies=copies)
    ctx.set_option(_lib.CC_OPT_STAGE_LAYOUT, 2 if layout in ("chunk_sorted", "hybrid") else 0)
    lib = ctx.lib
    if hasattr(edges, "data_ptr") and getattr(edges, "is_cuda", False):
        import torch
        if edges.dtype not in (torch.int32, torch.int64):
            raise ValueError("edges must be int32 or int64")
        e = edges.reshape(-1, 2)
        if e.device.index != ctx.device:  # a tensor on another GPU: copy it over first
            e = e.to(torch.device("cuda", ctx.device))
        e = e.contiguous()
        # the library stages on its own stream: wait for the work that produced
        # the tensor (torch's current stream of its device, e.g. a
        # torch.randint just before this call) before it reads the rows
        torch.cuda.current_stream(e.device).synchronize()
        if e.data_ptr() != edges.data_ptr():
            torch.cuda.current_stream(edges.device).synchronize()
        eb = e.element_size()
        _lib.check(lib.cc_stage_edges_device(ctx.handle, ctypes.c_void_p(e.data_ptr()), eb,
                                             e.shape[0], n))
        m = e.shape[0]
    else:
        e = _host_edges(edges)
        m = e.shape[0]
        _lib.check(lib.cc_stage_edges(ctx.handle, ctypes.c_void_p(e.ctypes.data),
                                      e.dtype.itemsize, m, n))
    ctx.n, ctx.m = n, m
    if layout in ("src_sorted", "dst_bucketed", "l2_tiled", "hybrid", "l2_tiled_check",
                  "relabel"):
        _lib.check(lib.cc_reorder_edges(ctx.handle, LAYOUTS[layout]))


def run_staged(ctx: _lib.Context, schedule: Schedule, *, count_changes: bool = True,
               early_check: bool = True, sweep_times: bool = True, cap: Optional[int] = None,
               labels_out: Optional[np.ndarray] = None, first_scatter: bool = False,
               host_loop: bool = False):
    """cc_run on already-staged edges; returns (labels or None, IterationStats).

    Async runs without ``count_changes``/``early_check``/``first_scatter``
    execute the whole convergence loop as one CUDA-graph launch unless
    ``host_loop`` forces the per-sweep host loop."""
    n = ctx.n
    call = _RunCall(n, schedule, count_changes, early_check, sweep_times, cap, labels_out,
                    first_scatter, host_loop)
    _lib.check(ctx.lib.cc_run(ctx.handle, ctypes.byref(call.sched), call.flags, call.cap,
                              call.out_ptr, call.eb, ctypes.byref(call.st)))
    return labels_out, call.stats()


class _RunCall:
    """Arguments and stats buffers of one cc_run / cc_run_host call."""

    def __init__(self, n, schedule, count_changes, early_check, sweep_times, cap, labels_out,
                 first_scatter=False, host_loop=False):
        self.cap = n + 2 if cap is None else int(cap)  # engine.py:275
        capacity = max(1, min(self.cap, 1 << 12 if not count_changes else 1 << 16))
        # the library writes entries [0, sweeps_executed) -- no need to clear
        self.changed = np.empty(capacity, dtype=np.int64)
        self.secs = np.empty(capacity, dtype=np.float64)
        st = _lib.CCStats()
        st.capacity = capacity
        st.changed_per_sweep = self.changed.ctypes.data_as(_lib._I64P)
        st.sweep_seconds = self.secs.ctypes.data_as(_lib._DBLP)
        self.st = st
        self.flags = ((_lib.CC_RUN_EARLY_CHECK if early_check else 0)
                      | (_lib.CC_RUN_COUNT_CHANGES if count_changes else 0)
                      | (_lib.CC_RUN_SWEEP_TIMES if sweep_times else 0)
                      | (_lib.CC_RUN_FIRST_SCATTER if first_scatter else 0)
                      | (_lib.CC_RUN_HOST_LOOP if host_loop else 0))
        self.sched = _cc_schedule(schedule)
        self.out_ptr, self.eb = None, 8
        if labels_out is not None:
            if labels_out.dtype not in (np.int64, np.uint32, np.int32) or labels_out.size != n:
                raise ValueError("labels_out must be a length-n int64/int32/uint32 array")
            self.eb = labels_out.dtype.itemsize
            self.out_ptr = ctypes.c_void_p(labels_out.ctypes.data)

    def stats(self) -> IterationStats:
        st, changed, secs = self.st, self.changed, self.secs
        capacity = st.capacity
        return _stats_from(st, changed, secs, capacity)


def run_host(ctx: _lib.Context, n: int, edges, schedule: Schedule, *, layout: str = "auto",
             count_changes: bool = True, early_check: bool = True, sweep_times: bool = True,
             cap: Optional[int] = None, labels_out: Optional[np.ndarray] = None,
             first_scatter: bool = False, host_loop: bool = False):
    """Stage host edges and run in ONE call (cc_run_host): for asynchronous
    runs in input / chunk-sorted order, sweep 1 runs chunk by chunk right
    behind the host-to-device copy, so the transfer hides it (with exact
    counts too: sweep 1 started from the identity, so its change count is the
    number of cells with L[x] != x); every other case stages, then runs,
    exactly as stage_graph + run_staged.  Returns (labels_out, IterationStats)."""
    ctx.staged = None
    e = _host_edges(edges)
    m = e.shape[0]
    layout = resolve_layout(layout, m, n, resident=False)
    if layout not in ("input", "chunk_sorted"):
        stage_graph(ctx, n, e, layout)
        return run_staged(ctx, schedule, count_changes=count_changes, early_check=early_check,
                          sweep_times=sweep_times, cap=cap, labels_out=labels_out,
                          first_scatter=first_scatter, host_loop=host_loop)
    ctx.set_option(_lib.CC_OPT_STAGE_LAYOUT, 2 if layout == "chunk_sorted" else 0)
    call = _RunCall(n, schedule, count_changes, early_check, sweep_times, cap, labels_out,
                    first_scatter, host_loop)
    _lib.check(ctx.lib.cc_run_host(ctx.handle, ctypes.c_void_p(e.ctypes.data), e.dtype.itemsize,
                                   m, n, ctypes.byref(call.sched), call.flags, call.cap,
                                   call.out_ptr, call.eb, ctypes.byref(call.st)))
    ctx.n, ctx.m = n, m
    return labels_out, call.stats()


def _stats_from(st, changed, secs, capacity) -> IterationStats:
    k = int(st.sweeps_executed)
    cnt = changed[:min(k, capacity)].tolist() + [-1] * max(0, k - capacity)
    sec = secs[:min(k, capacity)].tolist() + [0.0] * max(0, k - capacity)
    stats = IterationStats(
        sweeps_executed=k, sweeps_until_stable=int(st.sweeps_until_stable),
        changed_per_sweep=[int(x) for x in cnt],
        converged_by="early-check" if st.converged_by == 1 else "change-flag",
        sweep_seconds=sec, device_seconds=float(st.converge_seconds))
    return stats


def verify_staged(ctx: _lib.Context) -> int:
    """cc_verify on the device labels of the last run: 0 = valid final
    labelling (per edge L[u]==L[v], L[L[x]]==L[x], L[x]<=x); else a bitmask
    (1 edge disagreement, 2 non-root label, 4 label above its vertex)."""
    r = ctypes.c_int(0)
    _lib.check(ctx.lib.cc_verify(ctx.handle, ctypes.byref(r)))
    return r.value


def loop_check(ctx: _lib.Context) -> bool:
    """The early convergence check (engine.py:331-348) exactly as the device
    loop runs it after a changing sweep, on the context's current labels."""
    ok = ctypes.c_int(0)
    _lib.check(ctx.lib.cc_loop_check(ctx.handle, ctypes.byref(ok)))
    return bool(ok.value)


def _frozen(edges) -> bool:
    """True only for an edge array that cannot change behind our back: not
    writeable itself and every array it views is read-only and owns its
    memory (a read-only view of a writeable base, or a read-only memory map
    of a file, can still change)."""
    if not isinstance(edges, np.ndarray) or edges.flags.writeable:
        return False
    a = edges
    while isinstance(a, np.ndarray) and a.base is not None:
        a = a.base
        if not isinstance(a, np.ndarray) or a.flags.writeable:
            return False  # a foreign buffer (mmap, bytes, ...) or a writeable base
    return True


def _array_key(edges):
    return (edges.ctypes.data, edges.shape, edges.strides, edges.dtype.str)


def run_contour(g, schedule: Schedule, threads: int = 1, seed: Optional[int] = None, *,
                device: int = 0, count_changes: bool = True, early_check: bool = True,
                sweep_times: bool = True, layout: str = "auto",
                first_scatter: bool = False,
                host_loop: bool = False, devices=None,
                cadence: int = 1) -> tuple[LabelArray, IterationStats]:
    """Run minimum-mapping sweeps to convergence on the GPU (engine.py:248-328).

    ``g`` is anything with ``.n`` and ``.edges`` ((m, 2) int32/int64 pairs,
    numpy or CUDA tensor), or an ``(n, edges)`` tuple.  ``threads`` and
    ``seed`` are validated as in the reference but do not change GPU
    semantics (every sweep already runs on all SMs).  Returns int64 labels
    (every entry the minimum vertex ID of its component) and IterationStats.
    Raises IterationCapExceeded after n+2 sweeps, ValueError on bad input.

    ``count_changes=False`` (no exact per-sweep counts; ``changed_per_sweep``
    then holds -1 for a changing sweep) is the fast path: the whole loop is one
    CUDA-graph launch, and on layout 6 an asynchronous C-2 run ends on the
    uniting early check (CC_OPT_CHECK_UNITE, DESIGN 5.32): rows whose labels
    still differ after a sweep are united and pointer jumping finishes the
    labels -- same labels, ``converged_by == "early-check"``.

    ``devices`` (a list of CUDA device ordinals, more than one) shards the
    edge rows over those GPUs inside this process -- label replicas merged by
    an element-wise MIN every ``cadence`` local sweeps (distributed.py; one
    process per GPU with torch.distributed is the multi-node-ready form).
    Asynchronous schedules: ``changed_per_sweep`` holds -1 for the sweeps of
    changing rounds and 0 for the last round's (with ``cadence`` k > 1 the
    last round has k no-write sweeps, so executed = until_stable + k).
    Synchronous schedules shard deterministically (shadow lowering per
    shard, MIN all-reduce of the shadows, commit): every IterationStats
    field equals the single-device run's.
    """
    if threads < 1:
        raise ValueError("threads must be >= 1")
    n, edges = _unpack_graph(g)
    if n < 0:
        raise ValueError("vertex count must be non-negative")
    if devices is not None and len(devices) > 1:
        from .distributed import run_in_process
        if schedule.sync:  # deterministic: the same per-sweep results as one device
            labels, (k, until, changed, by) = run_in_process(
                n, edges, schedule, devices, layout=layout, early_check=early_check)
            return labels, IterationStats(
                sweeps_executed=k, sweeps_until_stable=until, changed_per_sweep=changed,
                converged_by=by, sweep_seconds=[0.0] * k, device_seconds=0.0)
        labels, sweeps, rounds = run_in_process(n, edges, schedule, devices, cadence=cadence,
                                                layout=layout)
        k = max(1, int(cadence))
        changed = [-1] * (rounds - 1) + [0]
        return labels, IterationStats(
            sweeps_executed=sweeps, sweeps_until_stable=max(0, sweeps - k),
            changed_per_sweep=[c for c in changed for _ in range(k)],
            converged_by="change-flag", sweep_seconds=[0.0] * sweeps, device_seconds=0.0)
    if devices is not None and len(devices) == 1:
        device = int(devices[0])
    ctx = _context(device)
    labels = np.empty(n, dtype=np.int64)
    # A read-only edge array (the reference's Graph freezes its arrays,
    # graph.py:82-83) cannot change between calls: the graph staged by the
    # previous call on this context stays resident and is reused -- as the
    # device layout for resident graphs (resolve_layout(resident=True)).
    frozen = _frozen(edges)
    if frozen and ctx.staged is not None and ctx.staged[0]() is edges and \
            ctx.staged[1:3] == (n, layout) and ctx.staged[4] == _array_key(edges):
        if ctx.staged[3]:  # upgrade the streamed layout once (+ the hybrid's bucketed copy)
            _lib.check(ctx.lib.cc_reorder_edges(ctx.handle, LAYOUTS[ctx.staged[3]]))
            ctx.staged = ctx.staged[:3] + (None,) + ctx.staged[4:]
        _, stats = run_staged(ctx, schedule, count_changes=count_changes,
                              early_check=early_check, sweep_times=sweep_times,
                              labels_out=labels, first_scatter=first_scatter,
                              host_loop=host_loop)
        return labels, stats
    if hasattr(edges, "data_ptr") and getattr(edges, "is_cuda", False):
        stage_graph(ctx, n, edges, layout)
        _, stats = run_staged(ctx, schedule, count_changes=count_changes,
                              early_check=early_check, sweep_times=sweep_times,
                              labels_out=labels, first_scatter=first_scatter,
                              host_loop=host_loop)
    else:
        _, stats = run_host(ctx, n, edges, schedule, layout=layout, count_changes=count_changes,
                            early_check=early_check, sweep_times=sweep_times, labels_out=labels,
                            first_scatter=first_scatter, host_loop=host_loop)
        if frozen:
            m = int(edges.shape[0])
            staged = resolve_layout(layout, m, n, resident=False)
            want = resolve_layout(layout, m, n, resident=True)
            upgrade = None
            if want != staged:
                # only layouts reachable from the staged order in place (the
                # L2-window tiles are built from rows in any order; the hybrid's
                # bucketed copy needs the chunk-sorted rows)
                upgrade = want if (staged, want) in (("chunk_sorted", "hybrid"),
                                                     ("chunk_sorted", "l2_tiled_check"),
                                                     ("chunk_sorted", "l2_tiled")) else None
            # a weak reference: the cache must not keep the caller's array alive
            ctx.staged = (weakref.ref(edges), n, layout, upgrade, _array_key(edges))
    return labels, stats


def early_convergence_check(g, labels, parallel: bool = False, *, device: int = 0) -> bool:
    """True iff the labels are idempotent (L[L[x]] == L[x]) and both endpoints
    of every edge agree -- engine.py:331-348, evaluated on the device
    (cc_write_labels + cc_early_check).  ``parallel`` is accepted for the
    reference's signature; the device check is always parallel.  Labels must
    lie in 0..n-1 (ValueError otherwise; numpy indexing in the reference would
    fail or wrap on such input)."""
    n, edges = _unpack_graph(g)
    lab = np.asarray(labels)
    if lab.shape[0] != n:
        raise ValueError("label array length does not match vertex count")  # engine.py:339-340
    if n == 0:
        return True
    if lab.dtype not in (np.int64, np.int32):
        lab = lab.astype(np.int64)
    lab = np.ascontiguousarray(lab)
    ctx = _context(device)
    stage_graph(ctx, n, edges, "input")
    _lib.check(ctx.lib.cc_write_labels(ctx.handle, ctypes.c_void_p(lab.ctypes.data),
                                       lab.dtype.itemsize))
    ok = ctypes.c_int(0)
    _lib.check(ctx.lib.cc_early_check(ctx.handle, ctypes.byref(ok)))
    return bool(ok.value)


_cas_lock = threading.Lock()


def conditional_min_assign(labels: np.ndarray, cells, value: int, atomic: bool = False) -> bool:
    """Lower every referenced cell holding more than ``value`` to it; True if
    any changed (engine.py:158-189).  The scalar host form of the update the
    device sweeps apply (``lower`` in csrc/kernels.cuh); ``atomic`` makes
    each lowering a compare-and-swap, so concurrent callers never lose one."""
    changed = False
    for i in cells:
        if atomic:
            with _cas_lock:  # the CAS retry loop collapses to one locked compare
                if labels[i] > value:
                    labels[i] = value
                    changed = True
        elif labels[i] > value:
            labels[i] = value
            changed = True
    return changed


@dataclass
class ForestDiagnostics:
    """Pointer-graph structure v -> labels[v] (engine.py:92-105): the roots,
    each root's tree height, label-class sizes, number of label values."""

    roots: np.ndarray
    heights: dict
    class_sizes: dict
    merged_min_count: int


def forest_diagnostics(labels) -> ForestDiagnostics:
    """Roots, per-root tree heights and label-class sizes of a pointer graph
    (engine.py:373-405).  Host-side diagnostics, not part of the run: depths
    by pointer doubling (O(n log depth) gathers); a cycle raises
    IterationCapExceeded as in the reference."""
    lab = np.asarray(labels, dtype=np.int64)
    n = lab.shape[0]
    if n and (lab.min() < 0 or lab.max() >= n):
        raise ValueError("labels reference vertices outside 0..n-1")
    idx = np.arange(n, dtype=np.int64)
    # jump[x] = 2^k-th ancestor, dist[x] = steps taken to reach it (stops at roots)
    jump = lab.copy()
    dist = (jump != idx).astype(np.int64)
    for _ in range(64):
        nxt = jump[jump]
        if np.array_equal(nxt, jump):
            break
        dist = dist + dist[jump]
        jump = nxt
    else:
        raise IterationCapExceeded("cycle detected in pointer graph")
    if n and np.any(lab[jump] != jump):
        raise IterationCapExceeded("cycle detected in pointer graph")
    roots = np.flatnonzero(lab == idx)
    height = np.zeros(n, dtype=np.int64)
    if n:
        np.maximum.at(height, jump, dist)
    values, counts = np.unique(lab, return_counts=True)
    return ForestDiagnostics(roots=roots, heights={int(r): int(height[r]) for r in roots},
                             class_sizes={int(v): int(c) for v, c in zip(values, counts)},
                             merged_min_count=int(values.size))


def mm_order(target: np.ndarray, read: np.ndarray, w: int, v: int, order: int,
             atomic: bool = False) -> bool:
    """Single-edge order-h update (engine.py:209-231) executed by the device
    edge routines.  ``target is read`` is the asynchronous (in-place) form."""
    if order < 1:
        raise ValueError("operator order must be >= 1")
    if w == v:
        return False
    inplace = target is read
    r = np.ascontiguousarray(read, dtype=np.int64)
    t = r if inplace else np.ascontiguousarray(target, dtype=np.int64).copy()
    out = np.empty_like(r) if inplace else t
    if inplace:
        out[:] = r
    ch = ctypes.c_int(0)
    lib = _lib.load()
    _lib.check(lib.cc_mm_order(r.ctypes.data_as(_lib._I64P), out.ctypes.data_as(_lib._I64P),
                               r.size, int(w), int(v), int(order), int(inplace),
                               ctypes.byref(ch)))
    target[:] = out
    return bool(ch.value)
