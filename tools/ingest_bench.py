"""Ingestion throughput: an RMAT edge list as text,
loaded by (1) the device path (text -> HBM, parse, canonicalise, densify,
de-duplicate on the GPU), (2) the host path (multi-threaded C++ tokenizer +
numpy), (3) the unmodified reference's load_edge_list (graph.py:149-197,
pure Python) on a bounded prefix of the same text.  One JSON line.

    python tools/ingest_bench.py [--scale 20] [--ef 16] [--reps 3] [--ref-lines 2000000]
"""
import argparse
import io
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import gen  # noqa: E402
from paper_2311_02811_b200 import ingest  # noqa: E402


def rmat_text(scale: int, ef: int) -> bytes:
    n, e = gen.rmat(scale, ef, 1, symmetrize=False)
    # sparse original IDs (x * 7 + 3) so that densification has work to do
    e = e * 7 + 3
    parts = []
    step = 1 << 20
    for lo in range(0, e.shape[0], step):
        blk = e[lo:lo + step]
        parts.append("\n".join(f"{u} {v}" for u, v in blk.tolist()))
    return ("# rmat edge list\n" + "\n".join(parts) + "\n").encode()


def timed(fn, reps):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        out.append(time.perf_counter() - t0)
    return r, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--ef", type=int, default=16)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--ref-lines", type=int, default=2_000_000)
    args = ap.parse_args()
    t0 = time.perf_counter()
    text = rmat_text(args.scale, args.ef)
    gen_s = time.perf_counter() - t0
    lines = text.count(b"\n")
    # device path, pageable bytes in; then the same text already in HBM
    ingest.load_edge_list(io.BytesIO(text[:1 << 20].rsplit(b"\n", 1)[0]), device=0)  # warm
    dev, dev_t = timed(lambda: ingest.load_edge_list(io.BytesIO(text), device=0), args.reps)
    tt = torch.frombuffer(bytearray(text), dtype=torch.uint8).cuda()
    _, devr_t = timed(lambda: ingest.load_edge_list(tt, device=0), args.reps)
    host, host_t = timed(lambda: ingest.load_edge_list(io.BytesIO(text)), args.reps)
    exact = bool(dev.n == host.n and np.array_equal(dev.edges.cpu().numpy(), host.edges)
                 and np.array_equal(dev.id_map.cpu().numpy(), host.id_map))
    ref = {}
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if args.ref_lines > 0 and os.path.isdir(ref_dir):
        sys.path.insert(0, ref_dir)
        try:
            import minmapcc
            cut = text.split(b"\n", args.ref_lines)
            sample = b"\n".join(cut[:args.ref_lines]).decode()
            t0 = time.perf_counter()
            minmapcc.load_edge_list(io.StringIO(sample))
            s = time.perf_counter() - t0
            ref = {"lines": args.ref_lines, "seconds": s, "lines_per_s": args.ref_lines / s,
                   "what": f"minmapcc {minmapcc.__version__} load_edge_list (unmodified, pure "
                           "Python) on the first lines of the same text"}
        except Exception as exc:  # noqa: BLE001
            ref = {"error": repr(exc)}
    best = lambda ts: min(ts)  # noqa: E731
    print(json.dumps({
        "what": "edge-list ingestion (load_edge_list: parse, canonicalise, remap, dedupe)",
        "text_bytes": len(text), "lines": lines, "rows_out": int(dev.edges.shape[0]),
        "n": dev.n, "gen_seconds": gen_s, "exact_device_vs_host": exact,
        "device_pageable_s": dev_t, "device_resident_text_s": devr_t, "host_s": host_t,
        "device_pageable_lines_per_s": lines / best(dev_t),
        "device_resident_lines_per_s": lines / best(devr_t),
        "device_resident_text_GBps": len(text) / best(devr_t) / 1e9,
        "host_lines_per_s": lines / best(host_t), "host_threads": os.cpu_count(),
        "reference": ref}))


if __name__ == "__main__":
    main()
