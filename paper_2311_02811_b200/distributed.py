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

    def compress(self) -> int:
        r = ctypes.c_int(0)
        _lib.check(self.ctx.lib.cc_compress(self.ctx.handle, ctypes.byref(r)))
        return r.value


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


class ShardedContour:
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
        self.cap = n + 2 if cap is None else cap
        self.layout = "input"
        self.first_scatter = False  # load-free sweep 1 (exact, but adds a sweep on RMAT)

    @classmethod
    def from_rmat(cls, scale: int, edgefactor: int, seed: int, rank: int, world: int,
                  device: int, layout: str = "auto", atomic: bool = True, **kw):
        """Generate this rank's contiguous row shard of the symmetrised RMAT
        list on its GPU and lay it out (engine.resolve_layout)."""
        import torch

        from .engine import LAYOUTS, resolve_layout
        ctx = _lib.Context(device, torch.cuda.current_stream(device).cuda_stream)
        n = 1 << scale
        total = 2 * edgefactor * n
        lo, hi = shard_rows(total, rank, world)
        graphgen.rmat_device(ctx, scale, edgefactor, seed, row_lo=lo, row_hi=hi)
        layout = resolve_layout(layout, hi - lo, n)
        if LAYOUTS[layout]:
            _lib.check(ctx.lib.cc_reorder_edges(ctx.handle, LAYOUTS[layout]))
        runner = cls(CudaShard(ctx, n, atomic), n, total, **kw)
        runner.layout = layout
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
            self.allreduce(self.shard.labels)
            if int(self.shard.labels[self.n].item()) == 1:
                break
        self.shard.compress()
        return rounds
