"""Graph ingestion: edge-list and Matrix Market text to
the (n, (m,2) int64 edges) input contract of run_contour.

With ``device=k`` the text goes to GPU k once and everything after the
Matrix Market header runs there (``cc_ingest_*`` in libcontour.so, csrc/
ingest.inc): newline split, tokenising, canonical rows, densification and
sorted de-duplication; ``edges`` (and ``id_map``) are then int64 CUDA
tensors that ``run_contour`` stages device-to-device.

Same semantics and error messages as the reference loaders
(/root/reference/pkg/src/minmapcc/graph.py:149-197 ``load_edge_list`` and
graph.py:203-274 ``load_matrix_market``: canonical (min, max) rows, optional
ID densification by ascending original ID, sorted de-duplication); the line
tokenizer is the multi-threaded C++ ``cc_parse_edges`` in libcontour.so.
"""

from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass
from pathlib import Path
from typing import Optional

import numpy as np

from . import _lib
from .errors import EdgeListParseError, MatrixMarketFormatError

CC_PARSE_TOKENS, CC_PARSE_NONINT, CC_PARSE_NEGATIVE, CC_PARSE_RANGE = -1, -2, -3, -4


@dataclass(frozen=True)
class LoadedGraph:
    """The duck-typed graph contract of run_contour (engine.py:268-270)."""

    n: int
    edges: np.ndarray                    # (m, 2) int64 (a CUDA tensor with device=)
    id_map: Optional[np.ndarray] = None  # dense ID -> original external ID
    name: str = ""

    @property
    def m(self) -> int:
        return int(self.edges.shape[0])


def _read_bytes(source) -> bytes:
    if isinstance(source, (str, Path)):
        with open(source, "rb") as fh:
            return fh.read()
    if hasattr(source, "read"):
        data = source.read()
        return data.encode() if isinstance(data, str) else data
    return "".join(source).encode()  # iterable of lines


def _parse(buf: bytes, mode: int, bound: int = 0):
    """-> (rows int64 (m,2) or None, err_line, err_code, err_tokens, err_vals)."""
    lib = _lib.load()
    m = ctypes.c_int64(0)
    line, tok = ctypes.c_int64(0), ctypes.c_int(0)
    code = ctypes.c_int(0)
    vals = np.zeros(2, dtype=np.int64)
    vp = vals.ctypes.data_as(_lib._I64P)
    threads = os.cpu_count() or 1
    rc = lib.cc_parse_edges(buf, len(buf), mode, None, 0, ctypes.byref(m), ctypes.byref(line),
                            ctypes.byref(code), ctypes.byref(tok), threads, bound, vp)
    if rc != 0:
        if code.value == 0:
            _lib.check(rc)
        return None, line.value, code.value, tok.value, (int(vals[0]), int(vals[1]))
    rows = np.empty((m.value, 2), dtype=np.int64)
    if m.value:
        _lib.check(lib.cc_parse_edges(buf, len(buf), mode,
                                      rows.ctypes.data_as(_lib._I64P), m.value,
                                      ctypes.byref(m), ctypes.byref(line), ctypes.byref(code),
                                      ctypes.byref(tok), threads, bound, vp))
    return rows, 0, 0, 0, (0, 0)


_INGEST = {}
_INGEST_LOCK = threading.Lock()


def _device_index(device) -> int:
    if isinstance(device, int):
        return device
    s = str(device)
    if s == "cuda":
        return 0
    if s.startswith("cuda:"):
        return int(s.split(":", 1)[1])
    raise ValueError(f"device must be a CUDA device index or 'cuda:k', got {device!r}")


class _Ingest:
    """One cc_ingest handle (device buffers of the parser) per device."""

    def __init__(self, device: int):
        self.lib = _lib.load()
        self.device = device
        h = ctypes.c_void_p()
        _lib.check(self.lib.cc_ingest_create(device, ctypes.byref(h)), "cc_ingest_create")
        self.handle = h
        self.lock = threading.Lock()

    def __del__(self):
        try:
            if self.handle:
                self.lib.cc_ingest_destroy(self.handle)
        except Exception:
            pass


def _ingest_handle(device: int) -> _Ingest:
    with _INGEST_LOCK:
        h = _INGEST.get(device)
        if h is None:
            h = _INGEST[device] = _Ingest(device)
        return h


def _parse_device(h: _Ingest, buf, mode: int, bound: int = 0):
    """Device parse -> (m or None, err_line, err_code, err_tokens, err_vals)."""
    m = ctypes.c_int64(0)
    line, tok, code = ctypes.c_int64(0), ctypes.c_int(0), ctypes.c_int(0)
    vals = np.zeros(2, dtype=np.int64)
    vp = vals.ctypes.data_as(_lib._I64P)
    if hasattr(buf, "data_ptr") and getattr(buf, "is_cuda", False):
        import torch
        if buf.dtype != torch.uint8 or not buf.is_contiguous():
            raise ValueError("text on the device must be a contiguous uint8 CUDA tensor")
        if buf.device.index != h.device:
            buf = buf.to(torch.device("cuda", h.device))
        torch.cuda.current_stream(buf.device).synchronize()
        rc = h.lib.cc_ingest_parse_device(h.handle, ctypes.c_void_p(buf.data_ptr()), buf.numel(),
                                          mode, bound, 1, ctypes.byref(m), ctypes.byref(line),
                                          ctypes.byref(code), ctypes.byref(tok), vp)
    else:
        rc = h.lib.cc_ingest_parse(h.handle, buf, len(buf), mode, bound, 1, ctypes.byref(m),
                                   ctypes.byref(line), ctypes.byref(code), ctypes.byref(tok), vp)
    if rc != 0:
        if code.value == 0:
            _lib.check(rc)
        return None, line.value, code.value, tok.value, (int(vals[0]), int(vals[1]))
    return m.value, 0, 0, 0, (0, 0)


def _finish_device(h: _Ingest, remap: bool, dedupe: bool, n_given: int):
    """Densify / de-duplicate on the device -> (n, edges, id_map) CUDA tensors."""
    import torch
    n, m, has_map = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int(0)
    _lib.check(h.lib.cc_ingest_finish(h.handle, int(remap), int(dedupe), n_given, ctypes.byref(n),
                                      ctypes.byref(m), ctypes.byref(has_map)), "cc_ingest_finish")
    dev = torch.device("cuda", h.device)
    edges = torch.empty((m.value, 2), dtype=torch.int64, device=dev)
    id_map = torch.empty(n.value, dtype=torch.int64, device=dev) if has_map.value else None
    # the copy runs on the handle's stream: order it after torch's allocations
    torch.cuda.current_stream(dev).synchronize()
    _lib.check(h.lib.cc_ingest_copy(
        h.handle, ctypes.c_void_p(edges.data_ptr() if m.value else 0),
        ctypes.c_void_p(id_map.data_ptr() if id_map is not None and n.value else 0)),
        "cc_ingest_copy")
    return int(n.value), edges, id_map


def _canonicalize(edges: np.ndarray) -> np.ndarray:  # graph.py:133-139
    if edges.shape[0] == 0:
        return edges
    return np.column_stack([np.minimum(edges[:, 0], edges[:, 1]),
                            np.maximum(edges[:, 0], edges[:, 1])])


def _sorted_unique(x: np.ndarray) -> np.ndarray:
    """np.unique(x) for 1-D integers by sort + neighbour compare (numpy 2's
    hash-based unique is several times slower on tens of millions of IDs)."""
    s = np.sort(x, axis=None)
    if s.size == 0:
        return s
    keep = np.empty(s.size, dtype=bool)
    keep[0] = True
    np.not_equal(s[1:], s[:-1], out=keep[1:])
    return s[keep]


def _dedupe_sorted(edges: np.ndarray) -> np.ndarray:  # graph.py:142-146
    if edges.shape[0] == 0:
        return edges
    if int(edges.max()) < (1 << 31):
        # np.unique(edges, axis=0) sorts rows as byte records; one packed
        # (u << 32 | v) key per row sorts in the same (lexicographic) order
        key = _sorted_unique((edges[:, 0].astype(np.int64) << 32) | edges[:, 1])
        return np.column_stack([key >> 32, key & 0xFFFFFFFF])
    return np.unique(edges, axis=0)


def _edge_list_error(line: int, code: int, tok: int) -> EdgeListParseError:
    if code == CC_PARSE_TOKENS:
        return EdgeListParseError(f"line {line}: expected two vertex IDs, got {tok} tokens")
    if code == CC_PARSE_NONINT:
        return EdgeListParseError(f"line {line}: non-integer token")
    return EdgeListParseError(f"line {line}: negative vertex ID")


def load_edge_list(source, *, dedupe: bool = True, remap: bool = True,
                   name: str = "", device=None) -> LoadedGraph:
    """graph.py:149-197.  ``device``: parse and densify on that GPU; the
    source may then also be a uint8 CUDA tensor holding the text."""
    if device is not None:
        h = _ingest_handle(_device_index(device))
        src = source if getattr(source, "is_cuda", False) else _read_bytes(source)
        with h.lock:
            m, line, code, tok, _ = _parse_device(h, src, 0)
            if m is None:
                raise _edge_list_error(line, code, tok)
            if m == 0:  # graph.py:183-184
                n, edges, id_map = _finish_device(h, False, False, 0)
                return LoadedGraph(0, edges, None, name)
            n, edges, id_map = _finish_device(h, remap, dedupe, -1)
        return LoadedGraph(n, edges, id_map, name)
    rows, line, code, tok, _ = _parse(_read_bytes(source), 0)
    if rows is None:
        if code == CC_PARSE_TOKENS:
            raise EdgeListParseError(f"line {line}: expected two vertex IDs, got {tok} tokens")
        if code == CC_PARSE_NONINT:
            raise EdgeListParseError(f"line {line}: non-integer token")
        raise EdgeListParseError(f"line {line}: negative vertex ID")
    if rows.shape[0] == 0:
        return LoadedGraph(0, np.zeros((0, 2), dtype=np.int64), None, name)
    edges = _canonicalize(rows)
    id_map = None
    if remap:
        ids = _sorted_unique(edges)
        if ids[0] == 0 and ids[-1] == ids.size - 1:
            n = int(ids.size)
        else:  # densify by ascending original ID
            edges = np.searchsorted(ids, edges).astype(np.int64)
            id_map = ids
            n = int(ids.size)
    else:
        n = int(edges.max()) + 1
    if dedupe:
        edges = _dedupe_sorted(edges)
    return LoadedGraph(n, np.ascontiguousarray(edges, dtype=np.int64), id_map, name)


_MM_FIELDS = {"pattern", "real", "integer", "double"}
_MM_SYMMETRIES = {"general", "symmetric"}


def load_matrix_market(source, name: str = "", device=None) -> LoadedGraph:
    """graph.py:203-274.  ``device``: the entry lines are parsed, canonicalised
    and de-duplicated on that GPU (header and size line on the host)."""
    buf = _read_bytes(source)
    pos = 0

    def next_line():
        nonlocal pos
        if pos >= len(buf):
            return None
        nl = buf.find(b"\n", pos)
        end = len(buf) if nl < 0 else nl
        line = buf[pos:end].decode("utf-8", errors="replace")
        pos = len(buf) if nl < 0 else nl + 1
        return line

    header = next_line()
    if header is None:
        raise MatrixMarketFormatError("empty input: missing MatrixMarket header")
    tokens = header.strip().split()
    if len(tokens) != 5 or tokens[0].lower() != "%%matrixmarket":
        raise MatrixMarketFormatError("missing '%%MatrixMarket' header line")
    _, obj, fmt, fld, sym = (t.lower() for t in tokens)
    if obj != "matrix" or fmt != "coordinate":
        raise MatrixMarketFormatError(f"unsupported format '{obj} {fmt}' (need matrix coordinate)")
    if fld not in _MM_FIELDS:
        raise MatrixMarketFormatError(f"unsupported field '{fld}'")
    if sym not in _MM_SYMMETRIES:
        raise MatrixMarketFormatError(f"unsupported symmetry '{sym}'")
    dims = None
    while dims is None:
        raw = next_line()
        if raw is None:
            raise MatrixMarketFormatError("missing size line")
        line = raw.strip()
        if not line or line.startswith("%"):
            continue
        parts = line.split()
        if len(parts) != 3:
            raise MatrixMarketFormatError("size line must hold 'rows cols nnz'")
        try:
            nrows, ncols, nnz = (int(p) for p in parts)
        except ValueError as exc:
            raise MatrixMarketFormatError("non-integer size line") from exc
        if nrows != ncols:
            raise MatrixMarketFormatError(f"adjacency matrix must be square, got {nrows}x{ncols}")
        dims = (nrows, ncols, nnz)
    n = dims[0]
    # bound -1 when n == 0 so every entry is out of range, as in the reference
    if device is not None:
        h = _ingest_handle(_device_index(device))
        with h.lock:
            m, line, code, tok, vals = _parse_device(h, buf[pos:], 1, n if n > 0 else -1)
            if m is None:
                raise _mm_entry_error(code, vals, n)
            if m != dims[2]:
                raise MatrixMarketFormatError(f"declared {dims[2]} entries but found {m}")
            n, edges, _ = _finish_device(h, False, True, n)
        return LoadedGraph(n, edges, None, name)
    rows, line, code, tok, vals = _parse(buf[pos:], 1, n if n > 0 else -1)
    if rows is None:
        raise _mm_entry_error(code, vals, n)
    if rows.shape[0] != dims[2]:
        raise MatrixMarketFormatError(f"declared {dims[2]} entries but found {rows.shape[0]}")
    edges = _dedupe_sorted(_canonicalize(rows - 1))
    return LoadedGraph(n, np.ascontiguousarray(edges.reshape(-1, 2), dtype=np.int64), None, name)


def _mm_entry_error(code: int, vals, n: int) -> MatrixMarketFormatError:
    if code == CC_PARSE_TOKENS:
        return MatrixMarketFormatError("entry line must hold at least two indices")
    if code == CC_PARSE_RANGE:
        return MatrixMarketFormatError(f"entry ({vals[0]},{vals[1]}) outside 1..{n}")
    return MatrixMarketFormatError("non-integer entry indices")


def load_binary_edges(path, n: int, dtype=np.int32, name: str = "") -> LoadedGraph:
    """Raw little-endian (m, 2) pairs of ``dtype`` (no text parsing); the
    edges keep file order and are not canonicalised (run_contour accepts
    any orientation, self-loops and duplicates)."""
    data = np.fromfile(path, dtype=dtype)
    if data.size % 2:
        raise ValueError("binary edge file holds an odd number of IDs")
    return LoadedGraph(int(n), data.reshape(-1, 2), None, name)
