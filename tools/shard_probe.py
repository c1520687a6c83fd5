"""Probe (development aid): rounds of the edge-sharded exchange on one GPU.
N shards of the RMAT rows, each with its own label replica; a round = every
shard's local order-2 sweep (+ shortcut), then the element-wise MIN of the
replicas copied back to all (what the NCCL all-reduce-MIN does).  Reports per
round whether any shard wrote and whether the early check would already pass
on every shard -- i.e. how many exchange rounds a check could save.

    python tools/shard_probe.py [--scale 22] [--shards 1,2,4,8]
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2311_02811_b200 import _lib, distributed, engine, graphgen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=22)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--shards", default="1,2,4,8")
    a = ap.parse_args()
    stream = torch.cuda.current_stream().cuda_stream
    for p in map(int, a.shards.split(",")):
        n = 1 << a.scale
        total = 32 * n
        shards = []
        for r in range(p):
            ctx = _lib.Context(0, stream)
            lo, hi = distributed.shard_rows(total, r, p)
            graphgen.rmat_device(ctx, a.scale, 16, a.seed, row_lo=lo, row_hi=hi)
            _lib.check(ctx.lib.cc_reorder_edges(ctx.handle, engine.LAYOUTS["chunk_sorted"]))
            lab = torch.empty(n + 1, dtype=torch.int32, device="cuda")
            _lib.check(ctx.lib.cc_attach_labels(ctx.handle, ctypes.c_void_p(lab.data_ptr())))
            _lib.check(ctx.lib.cc_init_labels(ctx.handle))
            shards.append((ctx, lab))
        log = []
        for rnd in range(1, 20):
            wrote_any = 0
            for ctx, lab in shards:
                w = ctypes.c_int(0)
                _lib.check(ctx.lib.cc_sweep(ctx.handle, 2, 0, 1, 0, ctypes.byref(w)))
                _lib.check(ctx.lib.cc_shortcut(ctx.handle, 1))
                wrote_any |= w.value
            m = shards[0][1][:n].clone()
            for _, lab in shards[1:]:
                torch.minimum(m, lab[:n], out=m)
            for _, lab in shards:
                lab[:n].copy_(m)
            checks = []
            for ctx, _ in shards:
                ok = ctypes.c_int(0)
                _lib.check(ctx.lib.cc_early_check(ctx.handle, ctypes.byref(ok)))
                checks.append(ok.value)
            log.append((rnd, wrote_any, all(checks)))
            if not wrote_any:
                break
        print(f"scale={a.scale} shards={p}: (round, any shard wrote, check passes on all "
              f"shards after the exchange) = {log}", flush=True)
        for ctx, _ in shards[::-1]:
            ctx.close()


if __name__ == "__main__":
    main()
