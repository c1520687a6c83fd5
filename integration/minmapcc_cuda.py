"""minmapcc/_cuda.py -- the module a minmapcc maintainer adds to run the hot
path on a B200 through libcontour.so (INTEGRATION.md "Option B").

It binds the C-ABI of include/contour.h with ctypes and nothing else (no
import of this repo's Python package): ``run_contour_cuda(g, schedule)``
replaces the body of minmapcc.engine.run_contour (engine.py:248-328) --
same arguments, same (labels, IterationStats) result, same exceptions.
integration/apply_option_b.py installs it into a copy of an installed
minmapcc together with the dispatch line in engine.run_contour;
tests/test_gpu_reference_dropin.py runs the reference's own harness through
it.
"""
import ctypes
import os

import numpy as np

from .errors import IterationCapExceeded

_VAR = {"C-Syn": 0, "C-1": 1, "C-2": 2, "C-m": 3, "C-11mm": 4, "C-1m1m": 5}
_EARLY_CHECK, _COUNT_CHANGES, _SWEEP_TIMES = 1, 2, 4  # cc_run flags


class _Sched(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in ("variant", "high_order", "warmup", "sync", "atomic")]


class _Stats(ctypes.Structure):
    _fields_ = [("executed", ctypes.c_int64), ("until_stable", ctypes.c_int64),
                ("converged_by", ctypes.c_int32), ("compress_rounds", ctypes.c_int32),
                ("capacity", ctypes.c_int64), ("changed", ctypes.POINTER(ctypes.c_int64)),
                ("seconds", ctypes.POINTER(ctypes.c_double)), ("total", ctypes.c_double)]


_lib = None
_ctx = ctypes.c_void_p()


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(os.environ["MINMAPCC_CONTOUR_LIB"])  # path to libcontour.so
        lib.cc_create.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
        lib.cc_create.restype = ctypes.c_int
        lib.cc_run_host.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                    ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(_Sched),
                                    ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                                    ctypes.POINTER(_Stats)]
        lib.cc_run_host.restype = ctypes.c_int
        lib.cc_last_error.restype = ctypes.c_char_p
        _lib = lib
    return _lib


def _check(rc):
    if rc == 0:
        return
    msg = _lib.cc_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise IterationCapExceeded(msg)
    raise RuntimeError(msg)


def run_contour_cuda(g, schedule):
    """engine.run_contour(g, schedule) on the GPU: early check after every
    changing sweep and exact changed_per_sweep, as the reference loop."""
    from .engine import IterationStats
    lib = _load()
    if not _ctx.value:
        _check(lib.cc_create(int(os.environ.get("MINMAPCC_CUDA_DEVICE", "0")), None,
                             ctypes.byref(_ctx)))
    edges = np.ascontiguousarray(g.edges)  # (m, 2) int64 (graph.py:66); read-only is fine
    if edges.size == 0:
        edges = np.zeros((0, 2), dtype=np.int64)
    n, m = int(g.n), int(edges.shape[0])
    cap = n + 2  # engine.py:275
    k = max(1, min(cap, 1 << 16))
    changed, secs = np.zeros(k, np.int64), np.zeros(k, np.float64)
    st = _Stats(capacity=k, changed=changed.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                seconds=secs.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    s = _Sched(_VAR[schedule.variant], schedule.high_order, schedule.warmup,
               int(schedule.sync), int(schedule.atomic))
    labels = np.empty(n, np.int64)
    _check(lib.cc_run_host(_ctx, edges.ctypes.data, edges.itemsize, m, n, ctypes.byref(s),
                           _EARLY_CHECK | _COUNT_CHANGES | _SWEEP_TIMES, cap,
                           labels.ctypes.data if n else None, 8, ctypes.byref(st)))
    e = int(st.executed)
    return labels, IterationStats(sweeps_executed=e, sweeps_until_stable=int(st.until_stable),
                                  changed_per_sweep=changed[:e].tolist(),
                                  converged_by="early-check" if st.converged_by else "change-flag",
                                  sweep_seconds=secs[:e].tolist())
