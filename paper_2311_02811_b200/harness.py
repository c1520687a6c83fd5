"""GPU runner for the reference's experiment harness.

Mirrors /root/reference/pkg/src/minmapcc/bench.py: the same ``PlanItem``
fields, the same CSV schema (bench.py:38-42) and ``label_checksum``
(bench.py:98-108), so GPU records sit beside the reference's CPU records;
extra columns report the device run.  Timing follows bench.py:176-179,196
(median wall time over ``repeats``; iteration statistics from the first run).
"""

from __future__ import annotations

import csv
import hashlib
import os
import statistics
import time
from dataclasses import dataclass
from pathlib import Path
from typing import IO, Callable, Iterable, Optional, Sequence, Union

import numpy as np

from . import _lib, engine
from .engine import canonical_variant, make_schedule

CSV_COLUMNS = (  # bench.py:38-42
    "graph", "n", "m", "algorithm", "variant", "sync", "atomic", "threads",
    "sweeps_until_stable", "sweeps_executed", "wall_time_ms", "components",
    "label_checksum", "oracle_match",
)
GPU_COLUMNS = ("devices", "device_ms", "edges_per_s", "hbm_fraction", "host_cores", "verified")


@dataclass(frozen=True)
class PlanItem:
    """bench.py:45-59 (``algo`` is always the GPU Contour engine here)."""

    graph: object                    # (n, edges), an object with .n/.edges, or a file path
    fmt: str = "edgelist"            # edgelist | mtx, for paths
    algo: str = "contour"
    variant: str = "c2"
    mode: str = "async"
    atomics: bool = True
    threads: int = 1
    high_order: int = 1024
    warmup: int = 2
    seed: Optional[int] = None
    name: str = ""


@dataclass(frozen=True)
class ExperimentRecord:
    graph: str
    n: int
    m: int
    algorithm: str
    variant: str
    sync: bool
    atomic: bool
    threads: int
    sweeps_until_stable: int
    sweeps_executed: int
    wall_time_ms: float
    components: int
    label_checksum: str
    oracle_match: bool
    devices: int = 1
    device_ms: float = 0.0
    edges_per_s: float = 0.0
    hbm_fraction: float = 0.0
    host_cores: int = 0
    verified: bool = False
    error: Optional[str] = None


def label_checksum(labels: np.ndarray) -> str:
    """bench.py:98-108: sha256 over "rep:size;" of the sorted (component
    minimum, size) pairs, first 16 hex digits.  ``labels`` must already be
    normalized (every entry its component minimum), as run_contour returns."""
    reps, sizes = np.unique(np.asarray(labels, dtype=np.int64), return_counts=True)
    digest = hashlib.sha256()
    for rep, size in zip(reps, sizes):
        digest.update(f"{int(rep)}:{int(size)};".encode())
    return digest.hexdigest()[:16]


def _peak_gbs() -> float:
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        import json
        with open(os.path.join(root, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return 6650.0


def _load(item: PlanItem):
    g = item.graph
    if isinstance(g, (str, Path)):
        from . import ingest
        loaded = ingest.load_matrix_market(g) if item.fmt == "mtx" else ingest.load_edge_list(g)
        return loaded.n, loaded.edges, item.name or str(g)
    if isinstance(g, tuple):
        return int(g[0]), np.asarray(g[1]), item.name or "<memory>"
    return int(g.n), g.edges, item.name or getattr(g, "name", "") or "<memory>"


def run_experiment(plan: Sequence[PlanItem], repeats: int = 3,
                   oracle: Optional[Callable[[int, np.ndarray], np.ndarray]] = None,
                   device: int = 0) -> list[ExperimentRecord]:
    """Run each plan item on the GPU (bench.py:149-201 semantics).

    ``oracle(n, edges)`` -> labels (e.g. the reference's ``rem_union_find``)
    sets ``oracle_match``; without it ``oracle_match`` is the device
    certificate ``cc_verify`` (every edge inside one label class, every label
    a root <= its vertices)."""
    if repeats < 1:
        raise ValueError("repeats must be >= 1")
    records = []
    ctx = _lib.Context(device)
    peak = _peak_gbs()
    try:
        for item in plan:
            try:
                if item.algo != "contour":
                    raise ValueError(f"GPU runner supports algo 'contour', got '{item.algo}'")
                if item.mode not in ("sync", "async"):
                    raise ValueError(f"unknown mode '{item.mode}'")
                sched = make_schedule(canonical_variant(item.variant), item.high_order,
                                      item.warmup, sync=True if item.mode == "sync" else None,
                                      atomic=item.atomics)
                if item.threads < 1:
                    raise ValueError("threads must be >= 1")
                n, edges, name = _load(item)
            except (OSError, ValueError) as exc:
                records.append(ExperimentRecord(
                    graph=item.name or str(item.graph), n=0, m=0, algorithm=item.algo,
                    variant=item.variant, sync=False, atomic=False, threads=item.threads,
                    sweeps_until_stable=0, sweeps_executed=0, wall_time_ms=0.0, components=0,
                    label_checksum="", oracle_match=False, error=str(exc)))
                continue
            m = int(np.asarray(edges).shape[0]) if not hasattr(edges, "is_cuda") else \
                int(edges.shape[0])
            labels = np.empty(n, dtype=np.int64)
            times, first_stats = [], None
            for rep in range(repeats):
                t0 = time.perf_counter()
                engine.stage_graph(ctx, n, edges)
                _, st = engine.run_staged(ctx, sched, labels_out=labels)
                times.append(time.perf_counter() - t0)
                if rep == 0:
                    first_stats = st
            verified = engine.verify_staged(ctx) == 0
            match = bool(np.array_equal(labels, oracle(n, edges))) if oracle else verified
            sweeps = [s for s in first_stats.sweep_seconds if s > 0]
            dev_s = first_stats.device_seconds
            frac = ((8 * m + 4 * n) / (sum(sweeps) / len(sweeps)) / 1e9 / peak) if sweeps else 0.0
            records.append(ExperimentRecord(
                graph=name, n=n, m=m, algorithm="contour", variant=sched.variant,
                sync=sched.sync, atomic=sched.atomic, threads=item.threads,
                sweeps_until_stable=first_stats.sweeps_until_stable,
                sweeps_executed=first_stats.sweeps_executed,
                wall_time_ms=statistics.median(times) * 1000.0,
                components=int(np.unique(labels).size), label_checksum=label_checksum(labels),
                oracle_match=match, devices=1, device_ms=dev_s * 1e3,
                edges_per_s=m / dev_s if dev_s > 0 else 0.0, hbm_fraction=frac,
                host_cores=os.cpu_count() or 1, verified=verified))
    finally:
        ctx.close()
    return records


def write_csv(records: Iterable[ExperimentRecord], sink: Union[str, Path, IO[str]],
              gpu_columns: bool = True) -> None:
    """The reference CSV schema (bench.py:204-227), plus the GPU columns."""
    if isinstance(sink, (str, Path)):
        with open(sink, "w", encoding="utf-8", newline="") as fh:
            _write(records, fh, gpu_columns)
    else:
        _write(records, sink, gpu_columns)


def _b(v: bool) -> str:
    return "true" if v else "false"


def _write(records, fh, gpu_columns):
    w = csv.writer(fh, lineterminator="\n")
    w.writerow(CSV_COLUMNS + (GPU_COLUMNS if gpu_columns else ()))
    for r in records:
        row = [r.graph, r.n, r.m, r.algorithm, r.variant, _b(r.sync), _b(r.atomic), r.threads,
               r.sweeps_until_stable, r.sweeps_executed, f"{r.wall_time_ms:.3f}", r.components,
               r.label_checksum, _b(r.oracle_match)]
        if gpu_columns:
            row += [r.devices, f"{r.device_ms:.4f}", f"{r.edges_per_s:.6g}",
                    f"{r.hbm_fraction:.4f}", r.host_cores, _b(r.verified)]
        w.writerow(row)
