"""Multi-rank host logic of the edge-sharded driver (paper_2311_02811_b200/
distributed.py) on CPU: world_size 2 over gloo, the per-rank sweep done by the
CPU oracle behind the same shard interface the CUDA shard implements.
Checks sharding, flag folding into the MIN all-reduce, termination and the
final compress give the exact union-find labels."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import gen, oracle
from paper_2311_02811_b200.distributed import (CheckedShardedContour, ShardedContour,
                                               SyncShardedContour, shard_rows)


class OracleShard:
    """CPU stand-in for CudaShard (test-only): same interface."""

    def __init__(self, n, edges):
        self.n = n
        self.edges = np.ascontiguousarray(edges, dtype=np.int64)
        self.labels = torch.zeros(n + 1, dtype=torch.int32)
        self.wrote = False

    def init(self):
        self.labels[: self.n] = torch.arange(self.n, dtype=torch.int32)

    def sweep(self, order, first=False):
        lab = self.labels[: self.n].numpy().astype(np.int64)
        L = oracle.lib()
        p = lab.ctypes.data_as(oracle._I64P)
        stores = L.oc_sweep_edges(p, p, self.edges.ctypes.data, 8, 0, self.edges.shape[0], 0,
                                  order, 1)
        self.labels[: self.n] = torch.from_numpy(lab.astype(np.int32))
        self.wrote = self.wrote or stores > 0

    def fold(self, first):
        f = 0 if self.wrote else 1
        self.labels[self.n] = f if first else min(int(self.labels[self.n]), f)
        self.wrote = False

    # synchronous mode (SyncShardedContour): lower a shadow from this shard
    def sync_sweep(self, order):
        lab = self.labels[: self.n].numpy().astype(np.int64)
        sh = lab.copy()
        L = oracle.lib()
        L.oc_sweep_edges(lab.ctypes.data_as(oracle._I64P), sh.ctypes.data_as(oracle._I64P),
                         self.edges.ctypes.data, 8, 0, self.edges.shape[0], 0, order, 1)
        self._shadow = torch.from_numpy(sh.astype(np.int32))

    def shadow(self):
        return self._shadow

    def commit(self):
        lab = self.labels[: self.n]
        changed = int((self._shadow != lab).sum())
        lab.copy_(self._shadow)
        return changed

    def check(self):
        return oracle.early_convergence_check(self.n, self.edges,
                                              self.labels[: self.n].numpy().astype(np.int64))

    # CheckedShardedContour: a numbered sweep, a shortcut pass, the loop check
    def sweep_numbered(self, order, sweep_no):
        self.sweep(order)

    def shortcut(self):
        lab = self.labels[: self.n].numpy()
        lab[:] = lab[lab]

    def loop_check(self):
        return self.check()

    def compress(self):
        lab = self.labels[: self.n].numpy()
        rounds = 0
        while True:
            nxt = lab[lab]
            if np.array_equal(nxt, lab):
                break
            lab[:] = nxt
            rounds += 1
        return rounds


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, cadence, q, checked=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, e = cfg
        lo, hi = shard_rows(e.shape[0], rank, world)
        cls = CheckedShardedContour if checked else ShardedContour
        runner = cls(OracleShard(n, e[lo:hi]), n, e.shape[0], cadence=cadence)
        rounds = runner.run()
        q.put((rank, runner.shard.labels[:n].numpy().astype(np.int64), rounds))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("graph,cadence,checked", [("rmat", 1, False), ("grid", 1, False),
                                                   ("grid", 3, False), ("forest", 2, False),
                                                   ("rmat", 1, True), ("grid", 1, True),
                                                   ("forest", 1, True)])
def test_two_rank_gloo_matches_union_find(graph, cadence, checked):
    """ShardedContour (no-write round ends the run) and CheckedShardedContour
    (one MIN exchange per sweep, the AND of the shards' early checks ends
    it) on two gloo ranks: exact labels, every rank stops at the same round."""
    if graph == "rmat":
        cfg = gen.rmat(10, 8, 3)
    elif graph == "grid":
        cfg = gen.grid(40, 40, 0.55, 2)
    else:
        cfg = gen.forest(6, 4)
    n, e = cfg
    exp = oracle.rem_union_find(n, e)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, cadence, q, checked))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rounds = {r for _, _, r in results}
    assert len(rounds) == 1  # every rank agrees when to stop
    for _, labels, _ in results:
        assert np.array_equal(labels, exp)


def _sync_worker(rank, world, port, cfg, variant, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, e = cfg
        lo, hi = shard_rows(e.shape[0], rank, world)
        runner = SyncShardedContour(OracleShard(n, e[lo:hi]), n, e.shape[0],
                                    order_for=lambda k: oracle.order_for(variant, k, 8))
        stats = runner.run()
        q.put((rank, runner.shard.labels[:n].numpy().astype(np.int64), stats))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("graph,variant,world", [("rmat", "C-2", 2), ("grid", "C-2", 3),
                                                 ("grid", "C-1", 2), ("forest", "C-m", 2)])
def test_sync_mode_shards_reproduce_single_device_counts(graph, variant, world):
    """Synchronous sweeps sharded over ranks (shadow per shard, MIN all-reduce
    of the shadows, commit) give per-sweep results identical to the
    one-device synchronous run -- the reference's."""
    cfg = {"rmat": gen.rmat(10, 8, 3), "grid": gen.grid(40, 40, 0.55, 2),
           "forest": gen.forest(6, 4)}[graph]
    n, e = cfg
    exp_labels, exp = oracle.run_contour(n, e, variant, high_order=8, sync=True)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sync_worker, args=(r, world, port, cfg, variant, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, labels, (k, until, changed, by) in results:
        assert np.array_equal(labels, exp_labels)
        assert (k, until, changed, by) == (exp.sweeps_executed, exp.sweeps_until_stable,
                                           list(exp.changed_per_sweep), exp.converged_by)


def test_shard_rows_cover_and_align():
    for total in (0, 1, 7, 1000, 1 << 20):
        for world in (1, 2, 3, 8):
            spans = [shard_rows(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
            for lo, _ in spans:
                assert lo % 4 == 0
