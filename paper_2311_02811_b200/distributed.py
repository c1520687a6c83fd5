"""Multi-GPU driver: edge-sharded sweeps, replicated labels, allreduce-MIN.

One process per GPU (torch.distributed, NCCL over NVLink 5 / NVSwitch).  Each
rank owns a contiguous shard of the edge rows (the reference's static edge
chunks per thread, engine.py:296-308, lifted to devices) and a full replica
of the n labels plus one exchange slot.  A round is ``cadence`` local sweeps
followed by an in-place ``all_reduce(labels[0:n+1], MIN)``:

* correctness: the element-wise min of valid label arrays is valid (each
  entry stays in its component and <= its index), so replicas only ever
  move toward the component minima;
* termination: slot n holds 1 if this rank's sweeps in the round lowered
  nothing, else 0, so after the MIN it is 1 iff no rank wrote -- every shard
  was then at a fixed point of the same replicated array, i.e. converged.

The per-rank compute sits behind a small shard interface so the host logic
can be exercised with gloo on CPU (tests/test_distributed_gloo.py):
``labels`` (int32 tensor, n+1), ``init()``, ``sweep(order, first)``,
``fold(first)``, ``compress()``.
"""

from __future__ import annotations

import ctypes

from . import _lib, graphgen


def _device_view(ptr: int, count: int, device: int):
    """A torch int32 view (no copy) of `count` entries of a device buffer."""
    import torch

    class _View:
        __cuda_array_interface__ = {"shape": (count,), "typestr": "<i4", "data": (ptr, False),
                                    "version": 3}
    return torch.as_tensor(_View(), device=f"cuda:{device}")


class CudaShard:
    """A rank's edge shard + label replica on its GPU (libcontour.so)."""

    def __init__(self, ctx: _lib.Context, n: int, atomic: bool = True):
        import torch
        if n >= 2 ** 31:
            raise ValueError("multi-GPU exchange uses int32 labels: n must be < 2^31")
        self.ctx = ctx
        self.n = n
        self.atomic = atomic  # Schedule.atomic: red.min (with hot-cell re-check) vs plain stores
        self.labels = torch.empty(n + 1, dtype=torch.int32, device=f"cuda:{ctx.device}")
        _lib.check(ctx.lib.cc_attach_labels(ctx.handle, ctypes.c_void_p(self.labels.data_ptr())))

    def init(self):
        _lib.check(self.ctx.lib.cc_init_labels(self.ctx.handle))

    def sweep(self, order: int, first: bool = False):
        _lib.check(self.ctx.lib.cc_sweep(self.ctx.handle, order, 0, int(self.atomic), int(first),
                                         None))

    def fold(self, first: bool):
        _lib.check(self.ctx.lib.cc_fold_flag(self.ctx.handle, int(first)))

    def shortcut(self, passes: int = 1):
        # safe before the MIN exchange: a shortcut value is a valid label and
        # the all-reduce makes the replicas identical again
        _lib.check(self.ctx.lib.cc_shortcut(self.ctx.handle, passes))

    def compress(self) -> int:
        r = ctypes.c_int(0)
        _lib.check(self.ctx.lib.cc_compress(self.ctx.handle, ctypes.byref(r)))
        return r.value

    # ---- synchronous mode (SyncShardedContour)
    def sync_sweep(self, order: int) -> None:
        _lib.check(self.ctx.lib.cc_sync_sweep(self.ctx.handle, order, None))

    def shadow(self):
        """The context's shadow labels (n entries) as a torch view, for the
        MIN all-reduce between the two halves of a synchronous sweep."""
        ptr = ctypes.c_void_p(0)
        _lib.check(self.ctx.lib.cc_shadow_device(self.ctx.handle, ctypes.byref(ptr)))
        return _device_view(ptr.value, self.n, self.ctx.device)

    def commit(self) -> int:
        c = ctypes.c_int64(0)
        _lib.check(self.ctx.lib.cc_sync_commit(self.ctx.handle, ctypes.byref(c)))
        return c.value

    def sweep_numbered(self, order: int, sweep_no: int) -> None:
        """Sweep number sweep_no of the run, laid out as cc_run would run it
        (cc_sweep_numbered); returns after the sweep finished on the device."""
        _lib.check(self.ctx.lib.cc_sweep_numbered(self.ctx.handle, order, int(self.atomic),
                                                  sweep_no, None))

    def loop_check(self) -> bool:
        """The early check as the device loop runs it on this shard's layout
        (cc_loop_check: the canonical / bitmap check copy where there is one)."""
        ok = ctypes.c_int(0)
        _lib.check(self.ctx.lib.cc_loop_check(self.ctx.handle, ctypes.byref(ok)))
        return bool(ok.value)

    def check(self) -> bool:
        """early_convergence_check on this shard's edges (and every label's
        idempotence) -- all ranks' results AND-ed give the whole graph's."""
        ok = ctypes.c_int(0)
        _lib.check(self.ctx.lib.cc_early_check(self.ctx.handle, ctypes.byref(ok)))
        return bool(ok.value)


class PeerShard:
    """A rank's shard whose order-2 sweeps write every lowering into all
    replicas at once (fused sweep + exchange, `cc_set_peers`): the label
    replicas of the other ranks are mapped through CUDA IPC, so no labels
    are reduced between sweeps -- only a one-word "did anyone lower" flag.

    Requires the context's own label buffer (not attached) and one process
    per GPU of one node (or several processes sharing a GPU in tests)."""

    def __init__(self, ctx: _lib.Context, n: int, atomic: bool = True, group=None):
        import torch.distributed as dist
        self.ctx = ctx
        self.n = n
        self.atomic = atomic
        self.group = group
        h = (ctypes.c_ubyte * 64)()
        _lib.check(ctx.lib.cc_ipc_get_handle(ctx.handle, h))
        handles = [None] * dist.get_world_size(group)
        dist.all_gather_object(handles, bytes(h), group=group)
        me = dist.get_rank(group)
        self.peer_ptrs = []
        for r, hb in enumerate(handles):
            if r == me:
                continue
            ptr = ctypes.c_uint64(0)
            buf = (ctypes.c_ubyte * 64).from_buffer_copy(hb)
            _lib.check(ctx.lib.cc_ipc_open(ctx.handle, buf, ctypes.byref(ptr)))
            self.peer_ptrs.append(ptr.value)
        arr = (ctypes.c_uint64 * max(1, len(self.peer_ptrs)))(*self.peer_ptrs)
        _lib.check(ctx.lib.cc_set_peers(ctx.handle, arr, len(self.peer_ptrs)))

    def enable(self, on: bool) -> None:
        """Route this rank's order-2 sweeps into the peers' replicas (on) or
        into the local replica only (off)."""
        if on:
            arr = (ctypes.c_uint64 * max(1, len(self.peer_ptrs)))(*self.peer_ptrs)
            _lib.check(self.ctx.lib.cc_set_peers(self.ctx.handle, arr, len(self.peer_ptrs)))
        else:
            _lib.check(self.ctx.lib.cc_set_peers(self.ctx.handle, None, 0))

    def labels_tensor(self):
        """A torch view (no copy) of the context's own n+1 int32 labels, for
        collective exchanges (NCCL all-reduce) on the same buffer the peers
        write into."""
        import torch
        ptr = ctypes.c_void_p(0)
        _lib.check(self.ctx.lib.cc_labels_device(self.ctx.handle, ctypes.byref(ptr)))

        class _View:
            __cuda_array_interface__ = {"shape": (self.n + 1,), "typestr": "<i4",
                                        "data": (ptr.value, False), "version": 3}
        return torch.as_tensor(_View(), device=f"cuda:{self.ctx.device}")

    def close(self):
        _lib.check(self.ctx.lib.cc_set_peers(self.ctx.handle, None, 0))
        for p in self.peer_ptrs:
            self.ctx.lib.cc_ipc_close(self.ctx.handle, p)
        self.peer_ptrs = []


class _HostIO:
    """Host-side input/output of a per-rank driver (the end-to-end path)."""

    def stage_host(self, edges, layout: str = "auto") -> None:
        """Stage this rank's host edge shard on its GPU (own PCIe link); the
        label buffer -- and so any peer mapping of it -- is kept."""
        from .engine import stage_graph
        # one row array: the exchange kernels walk the primary rows only
        stage_graph(self.shard.ctx, self.n, edges, layout, copies=False)

    def read_labels(self, out) -> None:
        """Copy the (converged) label replica into a host array of n
        int64/int32 entries."""
        _lib.check(self.shard.ctx.lib.cc_read_labels(
            self.shard.ctx.handle, ctypes.c_void_p(out.ctypes.data), out.dtype.itemsize))


class FusedShardedContour(_HostIO):
    """Per-rank driver of the fused exchange: init; barrier; then rounds of
    one fused order-2 sweep + a MAX all-reduce of the local "wrote" bit until
    no rank lowered anything (every replica then equals the min over all
    lowerings of all ranks, and every shard is at a fixed point of it)."""

    def __init__(self, shard: PeerShard, n: int, m_total: int, cap=None):
        self.shard = shard
        self.n = n
        self.m_total = m_total
        self.cap = n + 2 if cap is None else cap
        self.layout = "input"
        self.host_edges = None  # host copy of the shard (from_rmat keep_host)

    @classmethod
    def from_rmat(cls, scale: int, edgefactor: int, seed: int, rank: int, world: int,
                  device: int, layout: str = "auto", atomic: bool = True, group=None,
                  keep_host: bool = False):
        """This rank's contiguous row shard of the symmetrised RMAT list,
        generated on its GPU and laid out; ``keep_host``: also keep a host
        int64 copy of the shard in input order (``host_edges``, the e2e leg)."""
        import torch

        from .engine import LAYOUTS, resolve_layout
        ctx = _lib.Context(device, torch.cuda.current_stream(device).cuda_stream)
        n = 1 << scale
        total = 2 * edgefactor * n
        lo, hi = shard_rows(total, rank, world)
        graphgen.rmat_device(ctx, scale, edgefactor, seed, row_lo=lo, row_hi=hi)
        host = graphgen.read_edges(ctx, 8) if keep_host else None  # input order, pre-layout
        layout = resolve_layout(layout, hi - lo, n, copies=False)  # one row array
        if LAYOUTS[layout]:
            _lib.check(ctx.lib.cc_reorder_edges(ctx.handle, LAYOUTS[layout]))
        runner = cls(PeerShard(ctx, n, atomic, group), n, total)
        runner.layout = layout
        runner.host_edges = host
        return runner

    def _flag_any(self, wrote: int) -> bool:
        import torch
        import torch.distributed as dist
        dev = "cpu" if dist.get_backend(self.shard.group) == "gloo" else \
            f"cuda:{self.shard.ctx.device}"
        t = torch.tensor([wrote], dtype=torch.int32, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.shard.group)
        return bool(t.item())

    def run(self) -> int:
        import torch.distributed as dist
        ctx = self.shard.ctx
        _lib.check(ctx.lib.cc_init_labels(ctx.handle))
        _lib.check(ctx.lib.cc_synchronize(ctx.handle))
        dist.barrier(group=self.shard.group)  # no peer lowers into a replica before its init
        rounds = 0
        while True:
            rounds += 1
            if rounds > self.cap:
                from .errors import IterationCapExceeded
                raise IterationCapExceeded(f"no convergence after {self.cap} sweeps")
            wrote = ctypes.c_int(0)
            _lib.check(ctx.lib.cc_sweep(ctx.handle, 2, 0, int(self.shard.atomic), 0,
                                        ctypes.byref(wrote)))  # synchronises the device
            if not self._flag_any(wrote.value):
                break
        r = ctypes.c_int(0)
        _lib.check(ctx.lib.cc_compress(ctx.handle, ctypes.byref(r)))
        return rounds


class HybridShardedContour(_HostIO):
    """Dense first exchange, sparse later ones.  Sweep 1 lowers most labels:
    there a dense all-reduce-MIN of the n+1 labels (NCCL; ~2 x 4n bytes per
    rank) moves less than sending every lowering to every peer (~lowerings x
    (p-1) x 4 bytes).  Later sweeps lower few labels: there the fused sweep +
    peer red.min moves only those.  So round 1 = ``first_sweeps`` local
    sweeps (+ shortcut) folded into slot n, then one all-reduce-MIN of the
    replicas (converged if slot n == 1 after it, as in ShardedContour); from
    round 2 the FusedShardedContour protocol on the now identical replicas."""

    def __init__(self, shard: PeerShard, n: int, m_total: int, cap=None, allreduce=None,
                 first_sweeps: int = 1):
        self.shard = shard
        self.n = n
        self.m_total = m_total
        self.cap = n + 2 if cap is None else cap
        self.layout = "input"
        self.host_edges = None  # host copy of the shard (from_rmat keep_host)
        self.first_sweeps = max(1, int(first_sweeps))
        self.labels = shard.labels_tensor()
        self.allreduce = allreduce or nccl_allreduce_min(shard.group)

    @classmethod
    def from_rmat(cls, scale: int, edgefactor: int, seed: int, rank: int, world: int,
                  device: int, layout: str = "auto", atomic: bool = True, group=None,
                  keep_host: bool = False):
        base = FusedShardedContour.from_rmat(scale, edgefactor, seed, rank, world, device,
                                             layout=layout, atomic=atomic, group=group,
                                             keep_host=keep_host)
        runner = cls(base.shard, base.n, base.m_total)
        runner.layout = base.layout
        runner.host_edges = base.host_edges
        return runner

    def run(self) -> int:
        import torch
        import torch.distributed as dist
        shard, ctx = self.shard, self.shard.ctx
        lib = ctx.lib
        _lib.check(lib.cc_init_labels(ctx.handle))
        shard.enable(False)
        for k in range(self.first_sweeps):
            _lib.check(lib.cc_sweep(ctx.handle, 2, 0, int(shard.atomic), 0, None))
            _lib.check(lib.cc_fold_flag(ctx.handle, int(k == 0)))
            _lib.check(lib.cc_shortcut(ctx.handle, 1))
        _lib.check(lib.cc_synchronize(ctx.handle))
        self.allreduce(self.labels)
        rounds = 1
        if int(self.labels[self.n].item()) != 1:
            # every replica finished its all-reduce before any peer lowers into it
            torch.cuda.synchronize(ctx.device)
            dist.barrier(group=shard.group)
            shard.enable(True)
            try:
                while True:
                    rounds += 1
                    if rounds > self.cap:
                        from .errors import IterationCapExceeded
                        raise IterationCapExceeded(f"no convergence after {self.cap} sweeps")
                    wrote = ctypes.c_int(0)
                    _lib.check(lib.cc_sweep(ctx.handle, 2, 0, int(shard.atomic), 0,
                                            ctypes.byref(wrote)))
                    t = torch.tensor([wrote.value], dtype=torch.int32,
                                     device="cpu" if dist.get_backend(shard.group) == "gloo"
                                     else f"cuda:{ctx.device}")
                    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=shard.group)
                    if not int(t.item()):
                        break
            finally:
                shard.enable(False)
        r = ctypes.c_int(0)
        _lib.check(lib.cc_compress(ctx.handle, ctypes.byref(r)))
        return rounds


def shard_rows(total: int, rank: int, world: int, align: int = 4) -> tuple[int, int]:
    """Contiguous [lo, hi) of `total` rows for `rank`, boundaries aligned."""
    lo = (total * rank // world) // align * align
    hi = total if rank == world - 1 else (total * (rank + 1) // world) // align * align
    return lo, hi


def nccl_allreduce_min(group=None):
    import torch.distributed as dist

    def reduce(t):
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return reduce


class ShardedContour(_HostIO):
    """Per-rank driver.  ``allreduce`` performs the in-place MIN exchange of
    the (n+1)-slot label tensor (default: torch.distributed over the default
    NCCL/gloo group)."""

    def __init__(self, shard, n: int, m_total: int, *, order_for=lambda k: 2, cadence: int = 1,
                 group=None, cap=None, allreduce=None):
        self.shard = shard
        self.n = n
        self.m_total = m_total
        self.order_for = order_for
        self.cadence = max(1, int(cadence))
        self.allreduce = allreduce or nccl_allreduce_min(group)
        self.group = group
        self.cap = n + 2 if cap is None else cap
        self.layout = "input"
        self.host_edges = None  # host copy of the shard (from_rmat keep_host)
        self.first_scatter = False  # load-free sweep 1 (exact, but adds a sweep on RMAT)

    @classmethod
    def from_rmat(cls, scale: int, edgefactor: int, seed: int, rank: int, world: int,
                  device: int, layout: str = "auto", atomic: bool = True,
                  keep_host: bool = False, **kw):
        """Generate this rank's contiguous row shard of the symmetrised RMAT
        list on its GPU and lay it out (engine.resolve_layout); ``keep_host``
        keeps a host int64 copy of the shard in input order (``host_edges``)."""
        import torch

        from .engine import LAYOUTS, resolve_layout
        ctx = _lib.Context(device, torch.cuda.current_stream(device).cuda_stream)
        n = 1 << scale
        total = 2 * edgefactor * n
        lo, hi = shard_rows(total, rank, world)
        graphgen.rmat_device(ctx, scale, edgefactor, seed, row_lo=lo, row_hi=hi)
        host = graphgen.read_edges(ctx, 8) if keep_host else None  # input order, pre-layout
        layout = resolve_layout(layout, hi - lo, n, copies=False)  # one row array
        if LAYOUTS[layout]:
            _lib.check(ctx.lib.cc_reorder_edges(ctx.handle, LAYOUTS[layout]))
        runner = cls(CudaShard(ctx, n, atomic), n, total, **kw)
        runner.layout = layout
        runner.host_edges = host
        return runner

    def run(self) -> int:
        """Converge; returns the number of exchange rounds."""
        self.shard.init()
        sweep, rounds = 0, 0
        while True:
            rounds += 1
            for k in range(self.cadence):
                sweep += 1
                if sweep > self.cap:
                    from .errors import IterationCapExceeded
                    raise IterationCapExceeded(f"no convergence after {self.cap} sweeps")
                self.shard.sweep(self.order_for(sweep), first=(sweep == 1 and self.first_scatter))
                self.shard.fold(first=(k == 0))
                if hasattr(self.shard, "shortcut"):  # pointer jumping before the exchange
                    self.shard.shortcut()
            self.allreduce(self.shard.labels)
            if int(self.shard.labels[self.n].item()) == 1:
                break
        self.shard.compress()
        return rounds


class CheckedShardedContour(ShardedContour):
    """One exchange per sweep, ended by the early check instead of a no-write
    round: each rank lays its shard out as one GPU would (``resolve_layout``
    with row copies: on a dense graph beyond L2 the L2-window tiles + the
    delta-packed check copy + the canonical check copy), sweeps it (sweep 1
    split, later sweeps as bitmap sweeps, ``cc_sweep_numbered``), shortcuts,
    all-reduces the replicas with MIN, then runs the early check on its own
    rows (``cc_loop_check``: every edge of the shard agrees, every label is
    idempotent) and the verdicts are AND-ed (a MIN all-reduce of 0/1).  The
    replicas are identical after the MIN, so "every shard agrees" is the
    whole graph's early check (engine.py:318-320): converged.  Rounds = sweeps."""

    @classmethod
    def from_rmat(cls, scale: int, edgefactor: int, seed: int, rank: int, world: int,
                  device: int, layout: str = "auto", atomic: bool = True,
                  keep_host: bool = False, **kw):
        import torch

        from .engine import LAYOUTS, resolve_layout
        ctx = _lib.Context(device, torch.cuda.current_stream(device).cuda_stream)
        n = 1 << scale
        total = 2 * edgefactor * n
        lo, hi = shard_rows(total, rank, world)
        graphgen.rmat_device(ctx, scale, edgefactor, seed, row_lo=lo, row_hi=hi)
        host = graphgen.read_edges(ctx, 8) if keep_host else None
        layout = resolve_layout(layout, hi - lo, n)  # as one GPU would (row copies allowed)
        if layout == "hybrid":
            _lib.check(ctx.lib.cc_reorder_edges(ctx.handle, LAYOUTS["chunk_sorted"]))
        if LAYOUTS[layout]:
            _lib.check(ctx.lib.cc_reorder_edges(ctx.handle, LAYOUTS[layout]))
        runner = cls(CudaShard(ctx, n, atomic), n, total, **kw)
        runner.layout = layout
        runner.host_edges = host
        return runner

    def stage_host(self, edges, layout: str = "auto") -> None:
        """Stage this rank's host edge shard in the resident layout (with the
        check copies, as from_rmat); the attached label buffer is kept."""
        from .engine import stage_graph
        stage_graph(self.shard.ctx, self.n, edges, layout)

    def _and(self, ok: bool) -> bool:
        import torch
        import torch.distributed as dist
        dev = "cpu" if dist.get_backend(self.group) == "gloo" else f"cuda:{self.shard.ctx.device}"
        t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        return bool(int(t.item()))

    def run(self) -> int:
        shard = self.shard
        shard.init()
        rounds = 0
        while True:
            rounds += 1
            if rounds > self.cap:
                from .errors import IterationCapExceeded
                raise IterationCapExceeded(f"no convergence after {self.cap} sweeps")
            shard.sweep_numbered(self.order_for(rounds), rounds)
            shard.shortcut()
            self.allreduce(shard.labels)
            if self._and(shard.loop_check()):
                break
        shard.compress()
        return rounds


class SyncShardedContour:
    """Deterministic synchronous mode across ranks (last bullet):
    every sweep each rank lowers a shadow of the (identical) label replicas
    from its edge shard, the shadows are all-reduced with MIN -- min is
    associative, so the result is exactly the single-device synchronous
    sweep's shadow -- and committed; the change count is then the
    reference's (engine.py:288-291,309-311), identical on every rank.  The
    early check (engine.py:318-320) runs per shard and is AND-ed across
    ranks (a MIN all-reduce of the 0/1 results).  ``run`` returns
    (sweeps_executed, sweeps_until_stable, changed_per_sweep, converged_by)."""

    def __init__(self, shard, n: int, m_total: int, *, order_for=lambda k: 2,
                 early_check: bool = True, allreduce=None, group=None, cap=None):
        self.shard = shard
        self.n = n
        self.m_total = m_total
        self.order_for = order_for
        self.early_check = early_check
        self.allreduce = allreduce or nccl_allreduce_min(group)
        self.cap = n + 2 if cap is None else cap

    def run(self):
        import torch
        shard = self.shard
        shard.init()
        flag = torch.zeros(1, dtype=torch.int32, device=shard.labels.device)
        sweep, until, changed, by = 0, 0, [], "change-flag"
        while True:
            sweep += 1
            if sweep > self.cap:
                from .errors import IterationCapExceeded
                raise IterationCapExceeded(f"no convergence after {self.cap} sweeps")
            shard.sync_sweep(self.order_for(sweep))
            self.allreduce(shard.shadow())
            c = shard.commit()
            changed.append(int(c))
            if c == 0:
                break
            until = sweep
            if self.early_check:
                flag.fill_(int(shard.check()))
                self.allreduce(flag)
                if int(flag.item()) == 1:
                    by = "early-check"
                    break
        shard.compress()
        return sweep, until, changed, by


def run_in_process(n: int, edges, schedule, devices, cadence: int = 1, layout: str = "auto",
                   cap=None, early_check: bool = True):
    """``run_contour(..., devices=[...])``: the edge-sharded driver inside one
    process -- one host thread per listed device (a device may repeat: two
    shards on one GPU), each with its own context, stream and label replica;
    the MIN exchange is a host barrier + element-wise minimum of the replicas
    (gathered to the first device, copied back).  Asynchronous schedules:
    ShardedContour (a sweep of a shard is an asynchronous sweep of the whole
    edge list once the replicas are merged); returns (int64 labels, sweeps
    executed, exchange rounds).  Synchronous schedules: SyncShardedContour
    (per-sweep results identical to one device); returns (int64 labels,
    (sweeps, until_stable, changed_per_sweep, converged_by))."""
    import threading

    import numpy as np
    import torch

    from .engine import _host_edges, stage_graph

    devices = [int(d) for d in devices]
    world = len(devices)
    e = edges if (hasattr(edges, "data_ptr") and getattr(edges, "is_cuda", False)) \
        else _host_edges(edges)
    m = int(e.shape[0])
    slots = [None] * world
    barrier = threading.Barrier(world)
    out, errors, counts = {}, [], {}
    dev0 = torch.device("cuda", devices[0])

    def allreduce_for(r):
        def reduce(t):
            torch.cuda.synchronize(t.device)
            slots[r] = t
            barrier.wait()
            if r == 0:
                mn = slots[0].clone()
                for x in slots[1:]:
                    torch.minimum(mn, x.to(dev0), out=mn)
                for x in slots:
                    x.copy_(mn.to(x.device))
                for x in slots:
                    torch.cuda.synchronize(x.device)
            barrier.wait()
        return reduce

    def work(r):
        try:
            dev = devices[r]
            torch.cuda.set_device(dev)
            ctx = _lib.Context(dev)
            lo, hi = shard_rows(m, r, world)
            stage_graph(ctx, n, e[lo:hi], layout, copies=False)
            shard = CudaShard(ctx, n, atomic=schedule.atomic)
            if schedule.sync:
                runner = SyncShardedContour(shard, n, m, order_for=schedule.order_for,
                                            early_check=early_check,
                                            allreduce=allreduce_for(r), cap=cap)
            else:
                runner = ShardedContour(shard, n, m, order_for=schedule.order_for,
                                        cadence=cadence, allreduce=allreduce_for(r), cap=cap)
            rounds = runner.run()
            torch.cuda.synchronize(dev)
            counts[r] = rounds
            if r == 0:
                out[0] = shard.labels[:n].cpu().numpy().astype(np.int64)
            ctx.close()
        except Exception as exc:  # surfaced below; release the other threads
            errors.append(exc)
            barrier.abort()

    threads = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:  # the first real failure, not the barrier breaks it caused
        real = [x for x in errors if not isinstance(x, threading.BrokenBarrierError)]
        raise (real or errors)[0]
    rounds = counts[0]
    if schedule.sync:  # (sweeps, until_stable, changed_per_sweep, converged_by)
        return out[0], rounds
    return out[0], rounds * max(1, int(cadence)), rounds
