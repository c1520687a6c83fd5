"""Probe: sweep 1 split into a chunk-sorted prefix (flat kernel) followed by a
dst-bucketed remainder (shared-memory slice kernel) -- does one such sweep
still converge RMAT, and what does it cost?  (development aid)

    python tools/prefix_probe.py [--scales 20,21,22,23] [--seeds 1,2,3] [--fracs 0,1,2,4,16]

frac f = prefix rows f/16 of m (0: all rows bucketed, 16: all rows flat).
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_2311_02811_b200 import _lib, graphgen  # noqa: E402


def ctx_for(src, dst, n, layout, chunk, stream, labels=None):
    c = _lib.Context(0, stream)
    c.set_option(_lib.CC_OPT_SORT_CHUNK, chunk)
    m = src.numel()
    _lib.check(c.lib.cc_attach_soa(c.handle, ctypes.c_void_p(src.data_ptr()),
                                   ctypes.c_void_p(dst.data_ptr()), m, n))
    if labels is not None:
        _lib.check(c.lib.cc_attach_labels(c.handle, ctypes.c_void_p(labels)))
    _lib.check(c.lib.cc_reorder_edges(c.handle, layout))
    c.n, c.m = n, m
    return c


def labels_ptr(c):
    p = ctypes.c_void_p()
    _lib.check(c.lib.cc_labels_device(c.handle, ctypes.byref(p)))
    return p.value


def run(parts, n, check, reps=3):
    """parts: list of contexts sharing labels (parts[0] owns them)."""
    lib = parts[0].lib
    out = []
    for _ in range(reps + 1):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        _lib.check(lib.cc_init_labels(parts[0].handle))
        torch.cuda.synchronize()
        ev[0].record()
        sweeps, part_ms = 0, []
        while True:
            sweeps += 1
            wrote = 0
            pe = []
            for c in parts:
                if c.m == 0:
                    continue
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                w = ctypes.c_int(0)
                _lib.check(lib.cc_sweep(c.handle, 2, 0, 1, 0, ctypes.byref(w)))
                e1.record()
                pe.append((e0, e1))
                wrote |= w.value
            _lib.check(lib.cc_shortcut(parts[0].handle, 1))
            torch.cuda.synchronize()
            part_ms.append([round(a.elapsed_time(b), 3) for a, b in pe])
            if not wrote:
                break
            if check:
                ok = 1
                for c in parts:
                    if c.m == 0:
                        continue
                    o = ctypes.c_int(0)
                    _lib.check(lib.cc_early_check(c.handle, ctypes.byref(o)))
                    ok &= o.value
                if ok:
                    break
        ev[1].record()
        torch.cuda.synchronize()
        out.append((sweeps, ev[0].elapsed_time(ev[1]), part_ms))
    return out[1:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scales", default="20,21,22,23")
    ap.add_argument("--seeds", default="1,2,3")
    ap.add_argument("--fracs", default="0,1,2,4,16")
    ap.add_argument("--verify", type=int, default=1)
    a = ap.parse_args()
    stream = torch.cuda.current_stream().cuda_stream
    for scale in map(int, a.scales.split(",")):
        for seed in map(int, a.seeds.split(",")):
            n, e = graphgen.rmat(scale, 16, seed, elem_bytes=4)
            m = e.shape[0]
            expect = oracle.rem_union_find(n, e) if a.verify else None
            src_all = torch.from_numpy(np.ascontiguousarray(e[:, 0])).cuda()
            dst_all = torch.from_numpy(np.ascontiguousarray(e[:, 1])).cuda()
            for f in map(int, a.fracs.split(",")):
                P = (m * f // 16) // 4 * 4
                src, dst = src_all.clone(), dst_all.clone()
                chunk = min(1 << 23, max(P, 4))
                A = ctx_for(src[:P] if P else src[:0], dst[:P] if P else dst[:0], n, 2, chunk,
                            stream)
                lab = labels_ptr(A)
                parts = [A]
                if P < m:
                    B = ctx_for(src[P:], dst[P:], n, 3, 1 << 23, stream, labels=lab)
                    parts.append(B)
                for check in (False, True):
                    res = run(parts, n, check)
                    if expect is not None:
                        got = np.empty(n, np.int64)
                        _lib.check(A.lib.cc_compress(A.handle, None))
                        _lib.check(A.lib.cc_read_labels(A.handle, ctypes.c_void_p(got.ctypes.data), 8))
                        exact = bool(np.array_equal(got, expect))
                    else:
                        exact = None
                    print(f"scale={scale} seed={seed} frac={f:2d}/16 check={check:d} "
                          f"sweeps={[r[0] for r in res]} ms={[round(r[1], 3) for r in res]} "
                          f"parts={res[0][2]} exact={exact}", flush=True)
                for c in parts[::-1]:
                    c.close()


if __name__ == "__main__":
    main()
