"""Host->device bandwidth probe (development aid): raw pinned cudaMemcpy vs
the staging pipeline of cc_stage_edges (chunked, AoS->SoA, chunk sort)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2311_02811_b200 import _lib, engine, graphgen  # noqa: E402


def main():
    nbytes = 1 << 30
    h = torch.empty(nbytes // 4, dtype=torch.int32, pin_memory=True)
    d = torch.empty(nbytes // 4, dtype=torch.int32, device="cuda")
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    print(f"raw pinned H2D 1 GiB: {5 * nbytes / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
    n, e = graphgen.rmat(22, 16, 1, elem_bytes=4)
    pe = torch.empty((e.shape[0], 2), dtype=torch.int32, pin_memory=True)
    pe.numpy()[:] = e
    ctx = _lib.Context(0)
    for chunk in (1 << 22, 1 << 23, 1 << 24):
        ctx.set_option(_lib.CC_OPT_SORT_CHUNK, chunk)
        for layout in ("input", "chunk_sorted"):
            engine.stage_graph(ctx, n, pe.numpy(), layout)
            t0 = time.perf_counter()
            for _ in range(3):
                engine.stage_graph(ctx, n, pe.numpy(), layout)
            dt = (time.perf_counter() - t0) / 3
            print(f"stage chunk={chunk} layout={layout}: {dt*1e3:.2f} ms = "
                  f"{pe.numel() * 4 / dt / 1e9:.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
