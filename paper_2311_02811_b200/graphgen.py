"""Seeded synthetic inputs for BASELINE.json's five configs.

Definitions: oracle/gen.py (numpy specification; tests/test_gen.py checks
these generators against it bit for bit).  Host generators are
multi-threaded C++ in libcontour.so; RMAT also has a device generator that
writes the packed SoA edge arrays straight into HBM (needed at scale 28,
where the int32 edge list is 69 GB).
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np

from . import _lib

STREAM_FSIZE = 5
_GOLD = 0x9E3779B97F4A7C15
_M64 = (1 << 64) - 1


def _mix(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z ^ (z >> np.uint64(30))
        z = z * np.uint64(0xBF58476D1CE4E5B9)
        z = z ^ (z >> np.uint64(27))
        z = z * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _key(seed: int, stream: int) -> np.uint64:
    return _mix(np.array([((seed * _GOLD) + stream + 1) & _M64], dtype=np.uint64))[0]


def rmat_thresholds(a=0.57, b=0.19, c=0.19):
    return (int(a * 2 ** 32), int((a + b) * 2 ** 32), int((a + b + c) * 2 ** 32))


def _threads() -> int:
    return max(1, os.cpu_count() or 1)


def _alloc(m: int, elem_bytes: int) -> np.ndarray:
    return np.empty((m, 2), dtype=np.int32 if elem_bytes == 4 else np.int64)


def rmat(scale: int, edgefactor: int = 16, seed: int = 1, symmetrize: bool = True,
         permute: bool = True, elem_bytes: int = 8, row_lo: int = 0, row_hi=None,
         out: np.ndarray | None = None):
    """Kronecker/RMAT (a, b, c) = (.57, .19, .19): returns (n, edges)."""
    n = 1 << scale
    rows = (2 if symmetrize else 1) * edgefactor * n
    hi = rows if row_hi is None else int(row_hi)
    e = _alloc(hi - row_lo, elem_bytes) if out is None else out
    tA, tAB, tABC = rmat_thresholds()
    _lib.check(_lib.load().cc_gen_rmat_host(scale, edgefactor, seed, tA, tAB, tABC,
                                            int(symmetrize), int(permute), row_lo, hi,
                                            ctypes.c_void_p(e.ctypes.data),
                                            e.dtype.itemsize, _threads()))
    return n, e


def grid(rows: int, cols: int, p: float = 0.55, seed: int = 1, permute: bool = True,
         elem_bytes: int = 8):
    lib = _lib.load()
    m = ctypes.c_int64(0)
    thr = int(p * 2 ** 32)
    _lib.check(lib.cc_gen_grid_host(rows, cols, thr, seed, int(permute), None, elem_bytes,
                                    ctypes.byref(m), _threads()))
    e = _alloc(m.value, elem_bytes)
    _lib.check(lib.cc_gen_grid_host(rows, cols, thr, seed, int(permute),
                                    ctypes.c_void_p(e.ctypes.data), elem_bytes, ctypes.byref(m),
                                    _threads()))
    return rows * cols, e


def erdos_renyi(n: int, pairs: int, seed: int = 1, elem_bytes: int = 8):
    lib = _lib.load()
    m = ctypes.c_int64(0)
    _lib.check(lib.cc_gen_er_host(n, pairs, seed, None, elem_bytes, ctypes.byref(m)))
    e = _alloc(m.value, elem_bytes)
    _lib.check(lib.cc_gen_er_host(n, pairs, seed, ctypes.c_void_p(e.ctypes.data), elem_bytes,
                                  ctypes.byref(m)))
    return n, e


def forest_sizes(components: int, seed: int = 1, lo: int = 2, hi: int = 100_000) -> np.ndarray:
    """Sizes floor(exp(U(ln lo, ln hi))), U from the high 53 bits of draw c."""
    k = _key(seed, STREAM_FSIZE)
    with np.errstate(over="ignore"):
        idx = np.arange(components, dtype=np.uint64)
        d = _mix(k + (idx + np.uint64(1)) * np.uint64(_GOLD))
    U = (d >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    s = np.floor(np.exp(math.log(lo) + U * (math.log(hi) - math.log(lo)))).astype(np.int64)
    return np.clip(s, lo, hi)


def forest(components: int, seed: int = 1, isolated_frac: float = 0.2, elem_bytes: int = 8):
    sizes = np.ascontiguousarray(forest_sizes(components, seed))
    T = int(sizes.sum())
    n = T + int(round(T * isolated_frac / (1.0 - isolated_frac)))
    lib = _lib.load()
    m = ctypes.c_int64(0)
    sp = sizes.ctypes.data_as(_lib._I64P)
    _lib.check(lib.cc_gen_forest_host(sp, components, n, seed, None, elem_bytes,
                                      ctypes.byref(m), _threads()))
    e = _alloc(m.value, elem_bytes)
    _lib.check(lib.cc_gen_forest_host(sp, components, n, seed, ctypes.c_void_p(e.ctypes.data),
                                      elem_bytes, ctypes.byref(m), _threads()))
    return n, e


def rmat_device(ctx: _lib.Context, scale: int, edgefactor: int = 16, seed: int = 1,
                symmetrize: bool = True, permute: bool = True, row_lo: int = 0, row_hi=None):
    """Generate RMAT rows [row_lo, row_hi) on the device into ctx's SoA arrays."""
    n = 1 << scale
    rows = (2 if symmetrize else 1) * edgefactor * n
    hi = rows if row_hi is None else int(row_hi)
    tA, tAB, tABC = rmat_thresholds()
    _lib.check(ctx.lib.cc_gen_rmat_device(ctx.handle, scale, edgefactor, seed, tA, tAB, tABC,
                                          int(symmetrize), int(permute), row_lo, hi))
    ctx.n, ctx.m = n, hi - row_lo
    return n, hi - row_lo


def read_edges(ctx: _lib.Context, elem_bytes: int = 8, row_lo: int = 0, row_hi=None,
               out: np.ndarray | None = None) -> np.ndarray:
    """The context's staged rows [row_lo, row_hi) as a host (rows, 2) array
    (cc_read_edges) -- e.g. an RMAT-28 edge list generated on the device in a
    second, handed to host-side callers as the reference's int64 pairs."""
    hi = ctx.m if row_hi is None else int(row_hi)
    e = _alloc(hi - row_lo, elem_bytes) if out is None else out
    if e.shape != (hi - row_lo, 2) or e.dtype.itemsize != elem_bytes or \
            not e.flags.c_contiguous:
        raise ValueError("out must be a C-contiguous (rows, 2) array of elem_bytes")
    _lib.check(ctx.lib.cc_read_edges(ctx.handle, ctypes.c_void_p(e.ctypes.data), elem_bytes,
                                     row_lo, hi))
    return e


# BASELINE.json configs (DESIGN.md "Inputs" documents every deviation)
CONFIGS = {
    "er": dict(kind="er", n=65536, pairs=524288),
    "rmat22": dict(kind="rmat", scale=22, edgefactor=16),
    "grid4096": dict(kind="grid", rows=4096, cols=4096, p=0.55),
    "forest": dict(kind="forest", components=200_000),
    "rmat28": dict(kind="rmat", scale=28, edgefactor=16),
}


def make(cfg: dict, seed: int = 1, elem_bytes: int = 8):
    k = cfg["kind"]
    if k == "er":
        return erdos_renyi(cfg["n"], cfg["pairs"], seed, elem_bytes)
    if k == "rmat":
        return rmat(cfg["scale"], cfg.get("edgefactor", 16), seed, elem_bytes=elem_bytes)
    if k == "grid":
        return grid(cfg["rows"], cfg["cols"], cfg.get("p", 0.55), seed, elem_bytes=elem_bytes)
    if k == "forest":
        return forest(cfg["components"], seed, elem_bytes=elem_bytes)
    raise ValueError(k)
