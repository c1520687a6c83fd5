"""Fused sweep + exchange (multi-GPU design) exercised with several ranks on
ONE GPU: one process per rank, label replicas mapped into each other's
processes with CUDA IPC, every lowering sent to all replicas by the sweep
kernel, a one-word MAX all-reduce (gloo) per round.  No kernel waits on
another (the only synchronisation is the host barrier between rounds)."""

import ctypes
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_allreduce_min(t):
    import torch.distributed as dist
    c = t.cpu()
    dist.all_reduce(c, op=dist.ReduceOp.MIN)
    t.copy_(c)


def _worker(rank, world, port, cfg, q, exchange="fused"):
    import torch
    import torch.distributed as dist

    from paper_2311_02811_b200 import _lib, engine
    from paper_2311_02811_b200.distributed import (FusedShardedContour, HybridShardedContour,
                                                   PeerShard, shard_rows)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        n, e = cfg
        lo, hi = shard_rows(e.shape[0], rank, world)
        ctx = _lib.Context(0)
        engine.stage_graph(ctx, n, e[lo:hi], "chunk_sorted" if e.shape[0] > 1 << 16 else "input")
        shard = PeerShard(ctx, n, atomic=True)
        if exchange == "hybrid":
            runner = HybridShardedContour(shard, n, e.shape[0], allreduce=_gloo_allreduce_min)
        else:
            runner = FusedShardedContour(shard, n, e.shape[0])
        rounds = runner.run()
        labels = np.empty(n, dtype=np.int64)
        _lib.check(ctx.lib.cc_read_labels(ctx.handle, ctypes.c_void_p(labels.ctypes.data), 8))
        verify = engine.verify_staged(ctx)
        dist.barrier()  # peers stop writing before anyone unmaps
        shard.close()
        q.put((rank, labels, rounds, verify))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,graph,exchange",
                         [(2, "rmat", "fused"), (3, "grid", "fused"), (2, "forest", "fused"),
                          (2, "rmat", "hybrid"), (3, "grid", "hybrid"), (2, "forest", "hybrid")])
def test_fused_exchange_ranks_on_one_gpu(world, graph, exchange):
    import torch.multiprocessing as mp

    from oracle import gen, oracle
    if graph == "rmat":
        cfg = gen.rmat(15, 16, 11)
    elif graph == "grid":
        cfg = gen.grid(300, 300, 0.55, 5)
    else:
        cfg = gen.forest(20, 6)
    exp = oracle.rem_union_find(*cfg)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q, exchange))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len({r for _, _, r, _ in results}) == 1
    for _, labels, _, verify in results:
        assert np.array_equal(labels, exp)
        assert verify == 0
