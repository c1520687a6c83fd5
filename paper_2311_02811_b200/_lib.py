"""ctypes binding of libcontour.so (include/contour.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, the product entry points raise.
"""

from __future__ import annotations

import ctypes
import os

from .errors import IterationCapExceeded

_PKG = os.path.dirname(os.path.abspath(__file__))
# CONTOUR_LIB: another build of the library (A/B runs of two builds on one box)
LIB_PATH = os.environ.get("CONTOUR_LIB") or os.path.join(_PKG, "lib", "libcontour.so")

CC_OK, CC_EINVAL, CC_ECAP, CC_ECUDA = 0, 1, 2, 3
CC_RUN_EARLY_CHECK, CC_RUN_COUNT_CHANGES, CC_RUN_SWEEP_TIMES = 1, 2, 4
CC_RUN_FIRST_SCATTER, CC_RUN_HOST_LOOP = 8, 16

CC_OPT_STORE_MODE_PLAIN, CC_OPT_STORE_MODE_ATOMIC, CC_OPT_SORT_CHUNK = 1, 2, 3
CC_OPT_STAGE_LAYOUT, CC_OPT_BUCKET_SHIFT, CC_OPT_ITEM_ROWS, CC_OPT_BUCKET_THREADS = 4, 5, 6, 7
CC_OPT_TILE_SHIFT, CC_OPT_SHORTCUT, CC_OPT_TILE_SPLIT, CC_OPT_BUCKET_NOSMEM = 8, 9, 10, 11
CC_OPT_SWEEP_VARIANT = 12
CC_OPT_BUCKET_PIPE = 13
CC_OPT_ITEM_ORDER = 14
CC_OPT_WARP_TRANSPOSE = 15
CC_OPT_SWEEP_CTAS = 16
CC_OPT_CHECK_SHIFT = 17
CC_OPT_FLAT_BITS = 18
CC_OPT_HOST_SUB = 19
CC_OPT_HOST_NT = 20
CC_OPT_CHECK_PACK = 21
CC_OPT_LINK_PACK = 22
CC_OPT_SPLIT_SWEEP = 23
CC_OPT_SPLIT_REBUILD = 24
CC_OPT_SPLIT_MASK = 26
CC_OPT_CANON_CHECK = 27
CC_OPT_CANON_SPAN_BITS = 28
CC_OPT_CANON_GROUP_WINDOWS = 29
CC_OPT_RELABEL_INTERLEAVE = 30
CC_OPT_RELABEL_BLOCK = 31
CC_OPT_SPLIT_SHORTCUT = 32
CC_OPT_CANON_SWEEP = 33
CC_OPT_BITS_PUBLISH = 34
CC_OPT_CHECK_UNITE = 35
CC_OPT_BITS_DEFER = 36
STORE_PLAIN, STORE_RED, STORE_CHECK_PLAIN, STORE_CHECK_RED = 0, 1, 2, 3

_I64P = ctypes.POINTER(ctypes.c_int64)
_U32P = ctypes.POINTER(ctypes.c_uint32)
_DBLP = ctypes.POINTER(ctypes.c_double)


class CCSchedule(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int32), ("high_order", ctypes.c_int32),
                ("warmup", ctypes.c_int32), ("sync", ctypes.c_int32), ("atomic", ctypes.c_int32)]


class CCStats(ctypes.Structure):
    _fields_ = [("sweeps_executed", ctypes.c_int64), ("sweeps_until_stable", ctypes.c_int64),
                ("converged_by", ctypes.c_int32), ("compress_rounds", ctypes.c_int32),
                ("capacity", ctypes.c_int64), ("changed_per_sweep", _I64P),
                ("sweep_seconds", _DBLP), ("converge_seconds", ctypes.c_double)]


# name -> (restype, argtypes); every symbol declared in include/contour.h
SIGNATURES = {
    "cc_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    "cc_destroy": (None, [ctypes.c_void_p]),
    "cc_last_error": (ctypes.c_char_p, []),
    "cc_version": (ctypes.c_int, []),
    "cc_layout_info": (ctypes.c_int, [ctypes.c_void_p, _I64P, ctypes.c_int]),
    "cc_stage_edges": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                      ctypes.c_int64, ctypes.c_int64]),
    "cc_stage_edges_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                             ctypes.c_int64, ctypes.c_int64]),
    "cc_attach_soa": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_int64, ctypes.c_int64]),
    "cc_attach_labels": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "cc_labels_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    "cc_run": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(CCSchedule), ctypes.c_int,
                              ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                              ctypes.POINTER(CCStats)]),
    "cc_run_host": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                   ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(CCSchedule),
                                   ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                                   ctypes.POINTER(CCStats)]),
    "cc_init_labels": (ctypes.c_int, [ctypes.c_void_p]),
    "cc_sweep": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
    "cc_sweep_numbered": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int64, ctypes.POINTER(ctypes.c_int)]),
    "cc_reorder_edges": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "cc_set_option": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64]),
    "cc_fold_flag": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "cc_sync_sweep": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
    "cc_sync_commit": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]),
    "cc_shadow_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    "cc_compress": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)]),
    "cc_shortcut": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "cc_early_check": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)]),
    "cc_read_labels": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]),
    "cc_read_edges": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                     ctypes.c_int64, ctypes.c_int64]),
    "cc_write_labels": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]),
    "cc_loop_check": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)]),
    "cc_verify": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)]),
    "cc_synchronize": (ctypes.c_int, [ctypes.c_void_p]),
    "cc_mm_order": (ctypes.c_int, [_I64P, _I64P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                   ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
    "cc_gen_rmat_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                          ctypes.c_uint32, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int64, ctypes.c_int64]),
    "cc_gen_rmat_host": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                                        ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                        ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                                        ctypes.c_int]),
    "cc_gen_grid_host": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_uint32,
                                        ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p,
                                        ctypes.c_int, _I64P, ctypes.c_int]),
    "cc_gen_er_host": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                      ctypes.c_void_p, ctypes.c_int, _I64P]),
    "cc_gen_forest_host": (ctypes.c_int, [_I64P, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                          ctypes.c_void_p, ctypes.c_int, _I64P, ctypes.c_int]),
    "cc_ipc_get_handle": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "cc_ipc_open": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.POINTER(ctypes.c_uint64)]),
    "cc_ipc_close": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64]),
    "cc_set_peers": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64),
                                    ctypes.c_int]),
    "cc_fastsv": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                                 ctypes.POINTER(CCStats), ctypes.c_int]),
    "cc_parse_edges": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int64, ctypes.c_int, _I64P,
                                      ctypes.c_int64, _I64P, _I64P, ctypes.POINTER(ctypes.c_int),
                                      ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_int64,
                                      _I64P]),
    "cc_ingest_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "cc_ingest_destroy": (None, [ctypes.c_void_p]),
    "cc_ingest_parse": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int64,
                                       ctypes.c_int, ctypes.c_int64, ctypes.c_int, _I64P, _I64P,
                                       ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                       _I64P]),
    "cc_ingest_parse_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                              ctypes.c_int, ctypes.c_int64, ctypes.c_int, _I64P,
                                              _I64P, ctypes.POINTER(ctypes.c_int),
                                              ctypes.POINTER(ctypes.c_int), _I64P]),
    "cc_ingest_finish": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_int64, _I64P, _I64P,
                                        ctypes.POINTER(ctypes.c_int)]),
    "cc_ingest_result": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p),
                                        ctypes.POINTER(ctypes.c_void_p)]),
    "cc_ingest_copy": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
}

_lib = None


def load():
    """Load libcontour.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2311_02811_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error() -> str:
    msg = load().cc_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    if rc == CC_OK:
        return
    msg = last_error() or what
    if rc == CC_EINVAL:
        raise ValueError(msg)
    if rc == CC_ECAP:
        raise IterationCapExceeded(msg)
    raise RuntimeError(f"CUDA error in libcontour: {msg}")


class Context:
    """Owns one cc_ctx (device buffers, streams) on one CUDA device."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self.lib = load()
        self.device = device
        h = ctypes.c_void_p()
        check(self.lib.cc_create(device, ctypes.c_void_p(stream or 0), ctypes.byref(h)),
              "cc_create")
        self.handle = h
        self.staged = None  # run_contour's resident-graph key (engine._resident)
        self.n = 0
        self.m = 0

    def set_option(self, option: int, value: int) -> None:
        check(self.lib.cc_set_option(self.handle, option, value), "cc_set_option")

    def layout_info(self) -> dict:
        """cc_layout_info: layout code, check-copy format and bytes per pass."""
        import numpy as np
        out = np.zeros(14, dtype=np.int64)
        check(self.lib.cc_layout_info(self.handle, out.ctypes.data_as(_I64P), 14), "cc_layout_info")
        return {"layout": int(out[0]), "check_format": int(out[1]), "check_bytes": int(out[2]),
                "items": int(out[3]), "m": int(out[4]), "canon_rows": int(out[5]),
                "canon_bytes": int(out[6]), "canon_status": int(out[7]),
                "canon_side_groups": int(out[8]), "windows": int(out[9]),
                "split_windows": int(out[10]), "split_parts": int(out[11]),
                "uniting_check": bool(out[12]), "split_parts_canonical": bool(out[13])}

    def close(self):
        if getattr(self, "handle", None):
            self.lib.cc_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
