"""Benchmark: Contour CC throughput (input edges/s to converged labels) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config rmat28]
                    [--impl b200|reference] [--no-cpu-baseline] [--no-e2e]

Workload (default: BASELINE.json configs[4], the north-star config): RMAT
scale 28, edgefactor 16, (a,b,c,d) = (.57,.19,.19,.05), vertices permuted,
symmetrised -> n = 268,435,456 vertices, m = 8,589,934,592 input edge rows,
seeded synthetic.  One step = one whole run of the hot
path: labels = arange(n) -> order-2 asynchronous sweeps (+ the reference's
early convergence check) until converged -> pointer-jumping compress, with
the edges resident in HBM (69 GB of edges >> the 126 MB L2, so no flush).
On the layout "auto" picks for RMAT-28 (layout 6) the early check runs in its
uniting form (DESIGN 5.32): rows whose labels still differ after sweep 1 are
united on the spot and pointer jumping finishes the labels; `plain_check` in
the line is the same K runs with the plain check (CC_OPT_CHECK_UNITE 0), and
`verified` is cc_verify's certificate of the final labels.

--gpus N without torchrun re-launches itself under torch.distributed.run with
N local ranks (one per GPU).  N > 1: the edge rows are split into N
contiguous shards (each rank generates and lays out its own), labels are
replicated; round 1 is a local sweep + an NCCL all-reduce(MIN) of the n+1
labels, later rounds the fused sweep + red.min into the peers' replicas
(DESIGN.md section 7).  Strong scaling (total work fixed); max over ranks.

`e2e`: the drop-in call a reference user makes -- run_contour((n, edges),
make_schedule("c2")) on a pageable (m, 2) int64 numpy array (graph.py:66's
dtype), labels back as a fresh int64 numpy array -- timed with the host
clock around the call, so host->device staging, layout, the run and the
label read-back are all inside.

--impl reference: the reference's own CPU implementation -- the unmodified
minmapcc package (numba) from baseline/_ref when importable, else the C
port of it under oracle/ -- on the host cores, each step a bounded sample
of the same workload (see `sample`); rank 0 only.  Neither this arm nor the
CPU baseline loads the product library: their inputs come from oracle/'s
own generator.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
import types

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CC throughput: input edges/s to converged labels; per-sweep HBM GB/s vs peak"
UNIT = "edges/s"
HBM_FALLBACK_GBS = 6650.0
REF_DIR = os.path.join(ROOT, "baseline", "_ref")
SAMPLE_ROWS = 1 << 27  # CPU legs: rows [0, 2^27) of the workload's edge list

CONFIGS = {  # BASELINE.json configs (DESIGN.md section 8 documents each deviation)
    "er": dict(kind="er", n=65536, pairs=524288, idx=0,
               label="configs[0] Erdos-Renyi n=65536, 524288 uniform pairs, self-loops dropped"),
    "rmat22": dict(kind="rmat", scale=22, edgefactor=16, idx=1,
                   label="configs[1] RMAT scale 22, edgefactor 16, (a,b,c,d)=(.57,.19,.19,.05), "
                         "vertices permuted, symmetrised"),
    "grid4096": dict(kind="grid", rows=4096, cols=4096, p=0.55, idx=2,
                     label="configs[2] 4096x4096 grid, bonds kept with p=0.55, IDs permuted"),
    "forest": dict(kind="forest", components=200_000, idx=3,
                   label="configs[3] forest of 200k paths/trees (log-uniform sizes) + 20% "
                         "isolated vertices, IDs permuted (uint32 IDs: n > 2^31)"),
    "rmat28": dict(kind="rmat", scale=28, edgefactor=16, idx=4,
                   label="configs[4] RMAT scale 28, edgefactor 16, (a,b,c,d)=(.57,.19,.19,.05), "
                         "vertices permuted, symmetrised"),
}


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="rmat28", choices=sorted(CONFIGS))
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--early-check", default="auto", choices=["auto", "on", "off"],
                   help="the reference's early convergence check after each changing sweep "
                        "(engine.py:318-320), inside the device loop.  auto: on for the hybrid "
                        "layout and for L2-window tiles (its check beats the confirming sweep "
                        "there), off on flat chunk-sorted rows (DESIGN 5.10)")
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--layout", default="auto",
                   choices=["auto", "input", "src_sorted", "chunk_sorted", "dst_bucketed",
                            "l2_tiled", "hybrid", "l2_tiled_check", "relabel"],
                   help="staging-time edge layout of the device-resident runs")
    p.add_argument("--e2e-layout", default="auto",
                   help="layout= of the e2e drop-in run_contour call")
    p.add_argument("--e2e-dtype", default="int64", choices=["int64", "int32"],
                   help="element type of the e2e host edge array (the reference's Graph "
                        "holds int64, graph.py:66)")
    p.add_argument("--first-scatter", action="store_true",
                   help="run sweep 1 as the load-free identity scatter")
    p.add_argument("--host-loop", action="store_true",
                   help="drive sweeps from the host instead of the CUDA-graph WHILE loop "
                        "(same kernels; ncu cannot see kernels inside conditional nodes)")
    p.add_argument("--no-e2e", action="store_true", help="skip the end-to-end leg")
    p.add_argument("--fastsv", type=int, default=1,
                   help="timed runs of the GPU FastSV comparison baseline (0: skip)")
    p.add_argument("--sharded", action="store_true",
                   help="use the edge-sharded driver even with one rank (plumbing check)")
    p.add_argument("--cadence", type=int, default=1,
                   help="local sweeps per MIN exchange in the NCCL-only sharded driver")
    p.add_argument("--exchange", default="checked", choices=["checked", "hybrid", "peer", "nccl"],
                   help="multi-GPU label exchange: checked (default: each rank lays its shard "
                        "out as one GPU would -- split sweep 1, bitmap sweeps, canonical "
                        "check copy -- one all-reduce-MIN of the labels per sweep, the run "
                        "ends when every shard's early check passes), hybrid (one "
                        "all-reduce-MIN after the local sweep 1, then fused red.min into the "
                        "peer replicas), peer (fused from the start, CUDA IPC) or nccl "
                        "(all-reduce-MIN every --cadence local sweeps)")
    p.add_argument("--clock-interval-ms", type=int, default=100,
                   help="nvidia-smi sampling interval during the timed region")
    p.add_argument("--atomic", type=int, default=1,
                   help="Schedule.atomic (the reference default is True)")
    p.add_argument("--store-mode", type=int, default=None,
                   help="override the async store mode (0 plain, 1 red, 2 check+plain, "
                        "3 check+red)")
    p.add_argument("--sample-rows", type=int, default=SAMPLE_ROWS,
                   help="rows of the CPU legs' bounded sample (prefix of the edge list)")
    return p.parse_args(argv)


def physical_cores():
    try:
        import psutil
        return psutil.cpu_count(logical=False)
    except Exception:  # noqa: BLE001 -- reporting only
        return None


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            v = float(json.load(fh)["hbm_gbs"])
        return v, "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def store_mode_name(atomic: bool, override) -> str:
    names = {0: "plain stores", 1: "red.global.min", 2: "L2 re-check + plain store",
             3: "L2 re-check of hot cells + red.global.min"}
    mode = override if override is not None else (3 if atomic else 0)
    return names.get(mode, str(mode))


def sizes_of(name):
    """(n, m_input) of a config without generating it."""
    spec = CONFIGS[name]
    if spec["kind"] == "rmat":
        n = 1 << spec["scale"]
        return n, 2 * spec["edgefactor"] * n
    return None, None


def shared_config(name, n, m, atomic):
    """The `config` object -- identical in both arms (the driver compares them)."""
    return {"workload": CONFIGS[name]["label"], "n": int(n), "m_input": int(m),
            "seed": 1, "schedule": f"make_schedule('c2', atomic={bool(atomic)}): C-2, "
                                   f"asynchronous (the reference default)",
            "l2": (f"inputs larger than L2 (edge list {8 * m / 1e9:.1f} GB as uint32 pairs vs "
                   f"126 MB L2); no flush" if 8 * m > 126e6 else
                   f"edge list {8 * m / 1e6:.0f} MB fits L2; no flush (not a bandwidth config)")}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    interval_ms = 100

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(self.interval_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- CPU legs
def sample_edges(name, seed, rows, elem_bytes=8):
    """The CPU legs' bounded sample: rows [0, rows) of the config's edge list
    (all of it when smaller), generated by oracle/ -- never by the product
    library.  Returns (n, edges, m_full)."""
    from oracle import gen as ogen
    from oracle import oracle
    spec = CONFIGS[name]
    if spec["kind"] == "rmat":
        n = 1 << spec["scale"]
        m_full = 2 * spec["edgefactor"] * n
        _, e = oracle.gen_rmat(spec["scale"], spec["edgefactor"], seed, row_lo=0,
                               row_hi=min(rows, m_full), elem_bytes=elem_bytes)
        return n, e, m_full
    if spec["kind"] == "er":
        n, e = ogen.erdos_renyi(spec["n"], spec["pairs"], seed)
    elif spec["kind"] == "grid":
        n, e = ogen.grid(spec["rows"], spec["cols"], spec["p"], seed)
    else:
        n, e = ogen.forest(spec["components"], seed)
    m_full = e.shape[0]
    e = np.ascontiguousarray(e[:rows], dtype=np.int64 if elem_bytes == 8 else np.int32)
    return n, e, m_full


def reference_impl():
    """The unmodified reference package from baseline/_ref (numba), or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "minmapcc")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_minmapcc")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import minmapcc
        from minmapcc import make_schedule, run_contour
        return types.SimpleNamespace(version=getattr(minmapcc, "__version__", "?"),
                                     make_schedule=make_schedule, run_contour=run_contour,
                                     path=os.path.dirname(minmapcc.__file__))
    except Exception as exc:  # noqa: BLE001 -- reported, the port stands in
        return types.SimpleNamespace(error=f"{type(exc).__name__}: {exc}")


def time_reference(ref, n, edges, threads, atomic, runs):
    """The reference's run_contour (engine.py:248-328) through its public API
    on a duck-typed graph (engine.py:268-270 only reads n, m, edges)."""
    g = types.SimpleNamespace(n=n, m=int(edges.shape[0]), edges=edges)
    sched = ref.make_schedule("c2", atomic=atomic)
    times, st, labels = [], None, None
    for _ in range(runs):
        t0 = time.perf_counter()
        labels, st = ref.run_contour(g, sched, threads=threads, seed=0)
        times.append(time.perf_counter() - t0)
    return times, st, labels


def time_port(n, edges, threads, atomic, runs, sync=False):
    from oracle import oracle
    oracle.lib()
    times, st, labels = [], None, None
    for _ in range(runs):
        t0 = time.perf_counter()
        labels, st = oracle.run_contour(n, edges, "C-2", atomic=atomic, sync=sync,
                                        threads=threads, seed=0)
        times.append(time.perf_counter() - t0)
    return times, st, labels


def sample_desc(name, rows, m_full, n):
    whole = rows >= m_full
    return (f"rows [0, {rows}) of the workload's edge list ({'all of it' if whole else f'1/{m_full // rows} of its {m_full} rows'}), "
            f"n = {n} (the full label array), int64 (m, 2) pairs as the reference's Graph, "
            f"generated by oracle/ (not the product library); "
            + ("" if whole else "the sample keeps the full-size O(n) per-sweep label work of "
                                 "the reference (label copy + diff), so its per-edge rate is "
                                 "a lower bound of the full graph's"))


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    atomic = bool(args.atomic)
    n, e, m_full = sample_edges(args.config, args.seed, args.sample_rows)
    rows = int(e.shape[0])
    ref = reference_impl()
    use_ref = ref is not None and not hasattr(ref, "error")
    timer = (lambda runs: time_reference(ref, n, e, threads, atomic, runs)) if use_ref else \
        (lambda runs: time_port(n, e, threads, atomic, runs))
    timer(max(1, args.warmup))  # numba JIT + page-in
    times, st, _ = timer(args.steps)
    ms = 1e3 * sum(times) / len(times)
    value = rows / (ms / 1e3)
    kind = "reference" if use_ref else "port"
    what = (f"minmapcc {ref.version} (unmodified reference, numba) from baseline/_ref: "
            f"run_contour(g, make_schedule('c2'), threads={threads}, seed=0)" if use_ref else
            "oracle/ C port of run_contour (engine.py:248-328), "
            + (f"reference not importable: {ref.error}" if ref is not None else
               "reference not installed in baseline/_ref"))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic", "config": shared_config(args.config, n, m_full, atomic),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "cores_physical": physical_cores(), "what": what,
                         "sample": sample_desc(args.config, rows, m_full, n)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_sweeps": {"executed": int(st.sweeps_executed),
                             "until_stable": int(st.sweeps_until_stable),
                             "converged_by": st.converged_by, "on": "the sample"},
        "parallelism": f"{threads} host threads (static edge chunks, engine.py:296-308)",
    }
    print(json.dumps(line), flush=True)


def load_traffic():
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except Exception:
        return {}


# ---------------------------------------------------------------- launching
def free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args) -> int:
    """--gpus N without torchrun: start N local ranks of this script under
    torch.distributed.run (one per GPU); rank 0 prints the line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    ClockSampler.interval_ms = max(20, args.clock_interval_ms)
    if args.impl == "reference":
        return run_reference_arm(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch(args))
    rank, world, local = dist_env()
    import torch
    ndev = max(1, torch.cuda.device_count())
    # more ranks than GPUs only as a plumbing check (ranks share a GPU; their
    # kernels never wait on one another, the host flag exchange uses gloo)
    local, backend = (local, "nccl") if world <= ndev else (local % ndev, "gloo")
    torch.cuda.set_device(local)
    if world > 1 or args.sharded:
        import torch.distributed as dist
        if "MASTER_ADDR" not in os.environ:  # --sharded without torchrun: one local rank
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(free_port()), RANK="0",
                              WORLD_SIZE="1")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
        return run_multi(args, rank, world, local)
    return run_single(args, local)


# ---------------------------------------------------------------- 1 GPU
def run_single(args, device):
    import torch

    from paper_2311_02811_b200 import _lib, engine, graphgen
    from paper_2311_02811_b200.engine import make_schedule

    spec = CONFIGS[args.config]
    atomic = bool(args.atomic)
    # one dedicated stream: the library launches on it and the CUDA events
    # that time the step are recorded on it
    stream = torch.cuda.Stream(device)
    torch.cuda.set_stream(stream)
    ctx = _lib.Context(device, stream.cuda_stream)
    if args.store_mode is not None:
        ctx.set_option(_lib.CC_OPT_STORE_MODE_ATOMIC if atomic else
                       _lib.CC_OPT_STORE_MODE_PLAIN, args.store_mode)
    e2e_dtype = np.int64 if args.e2e_dtype == "int64" else np.int32
    host_edges = None
    # ---- inputs: generated on the device (RMAT) or on the host; the e2e leg's
    # host copy is taken in generation (input) order, before any layout
    t_prep = time.perf_counter()
    if spec["kind"] == "rmat":
        n, m = graphgen.rmat_device(ctx, spec["scale"], spec.get("edgefactor", 16), args.seed)
        if not args.no_e2e:
            host_edges = graphgen.read_edges(ctx, np.dtype(e2e_dtype).itemsize)
        layout = engine.resolve_layout(args.layout, m, n, counted=False)  # (timed runs: no exact counts)
        t_lay = time.perf_counter()
        if layout != "input":
            engine.apply_layout(ctx, layout)
    else:
        n, host_edges = graphgen.make(spec, args.seed, elem_bytes=np.dtype(e2e_dtype).itemsize)
        m = host_edges.shape[0]
        layout = engine.resolve_layout(args.layout, m, n, counted=False)  # (timed runs: no exact counts)
        t_lay = time.perf_counter()
        engine.stage_graph(ctx, n, host_edges, layout)
    torch.cuda.synchronize()
    layout_s = time.perf_counter() - t_lay
    prep_s = time.perf_counter() - t_prep

    early = args.early_check == "on" or (args.early_check == "auto" and
                                         layout in ("hybrid", "l2_tiled", "l2_tiled_check",
                                                    "relabel"))
    hybrid = layout == "hybrid"
    two_kernel = layout in ("hybrid", "l2_tiled_check")  # sweep 1 and later sweeps differ
    sched = make_schedule("c2", atomic=atomic)
    kw = dict(count_changes=False, early_check=early, first_scatter=args.first_scatter,
              host_loop=args.host_loop)

    for _ in range(args.warmup):
        engine.run_staged(ctx, sched, sweep_times=False, **kw)
    torch.cuda.synchronize()

    # ---- timed region: K whole runs, CUDA events on the launching stream
    clocks = ClockSampler(device)
    clocks.start()
    t_busy = time.perf_counter()  # untimed runs while the sampler warms up
    while time.perf_counter() - t_busy < 0.3:
        engine.run_staged(ctx, sched, sweep_times=False, **kw)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    stats = []
    for _ in range(args.steps):
        _, st = engine.run_staged(ctx, sched, sweep_times=False, **kw)
        stats.append(st)
    ev1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    value = m / (ms / 1e3)

    shortcut = 1  # CC_OPT_SHORTCUT default: one pointer-jumping pass after every sweep
    check = 2 if early else 0  # edge-agreement + idempotence kernels
    if args.host_loop:  # iota + (sweep + shortcut + check) per sweep + compress
        launches = sum(2 + s.sweeps_executed * (1 + shortcut + check) for s in stats)
    elif layout == "l2_tiled_check":
        # per loop iteration: sweep 1's tiled part + 3 kernels (root pick, bitmap
        # pass, bitmap sweep) per bitmap part + the later sweeps' 3 (all order-
        # guarded) + shortcut + the check's 3 + control; around the loop: init,
        # compress (+ 3 x (gate, compress) after the uniting check), publish
        li = ctx.layout_info()
        per = (1 + 3 * li["split_parts"] if li["split_windows"] else 1) + 3 + shortcut + 3 + 1
        around = 3 + (6 if li["uniting_check"] else 0)
        launches = sum(around + s.sweeps_executed * per for s in stats)
    else:  # loop_init + (guarded sweeps + shortcut + check + control) per sweep + compress + publish
        per = (2 if hybrid else 1) + shortcut + check + 1
        launches = sum(3 + s.sweeps_executed * per for s in stats)
    sweep_ms_graph = engine.run_staged(ctx, sched, sweep_times=True, **kw)[1].sweep_seconds
    verify = engine.verify_staged(ctx)
    run_info = ctx.layout_info()  # (sweep 1's split and the check of the timed runs)
    # ---- the same runs with the plain early check (sweeps until it passes):
    # what the uniting check (DESIGN 5.32) buys, on the same staged graph
    plain = None
    if run_info["uniting_check"]:
        ctx.set_option(_lib.CC_OPT_CHECK_UNITE, 0)
        engine.run_staged(ctx, sched, sweep_times=False, **kw)
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        pst = [engine.run_staged(ctx, sched, sweep_times=False, **kw)[1]
               for _ in range(args.steps)]
        p1.record(stream)
        torch.cuda.synchronize()
        pms = p0.elapsed_time(p1) / args.steps
        plain = {"value": m / (pms / 1e3), "unit": UNIT, "ms_per_step": pms,
                 "sweeps_per_run": [x.sweeps_executed for x in pst],
                 "verified": engine.verify_staged(ctx) == 0,
                 "what": "CC_OPT_CHECK_UNITE=0: the plain early check (a failing check costs "
                         "another sweep and another check); sweep 1 split after a quarter of "
                         "the windows, bitmap rebuilt every 3/16"}
        ctx.set_option(_lib.CC_OPT_CHECK_UNITE, 1)
        engine.run_staged(ctx, sched, sweep_times=False, **kw)
    dev_labels = None
    if not args.no_e2e:
        dev_labels = np.empty(n, dtype=np.int64)
        _lib.check(ctx.lib.cc_read_labels(ctx.handle, dev_labels.ctypes.data, 8))

    # ---- roofline of the sweep kernel: its own launch times, CUDA events on
    # the launching stream around each sweep (+ its shortcut pass) in
    # host-driven runs without the check (the graph loop's per-sweep records
    # include control and check kernels); the check kernel separately
    rt1, rt2, rtc = [], [], []
    # (layout 6: with the check on, as the timed runs -- sweep 1's split follows
    # the check that ends the run)
    for _ in range(max(1, min(args.steps, 3))):
        _, st = engine.run_staged(ctx, sched, sweep_times=True, count_changes=False,
                                  early_check=early and layout == "l2_tiled_check",
                                  host_loop=True)
        if two_kernel:
            rt1.append(st.sweep_seconds[0])
            rt2.extend(st.sweep_seconds[1:])
        else:
            rt1.extend(st.sweep_seconds)
    if early:  # the early-check kernels on converged labels (they pass: a full pass)
        for _ in range(3):
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            engine.loop_check(ctx)
            c1.record(stream)
            torch.cuda.synchronize()
            rtc.append(c0.elapsed_time(c1) / 1e3)
    t_sweep = sum(rt1) / len(rt1)
    b_sweep = 8 * m + 4 * n  # edge stream + one label-array read
    peak, peak_src = peak_hbm()
    traffic = load_traffic().get(args.config) or {}
    kernel_text = traffic.get("kernel", "cck::k_sweep<2, ...> (order-2 async sweep)")
    if layout == "l2_tiled_check" and run_info["split_windows"]:
        k, P, parts = run_info["split_windows"], run_info["windows"], run_info["split_parts"]
        kernel_text = (f"sweep 1 = cck::k_sweep<2, 59, 1, 1> over L2 windows 0-{k - 1} of {P} "
                       f"(tiles, 3 CTAs/SM, L2 cache hints) + {parts} x (k_pick_root, "
                       f"k_bits_idem, k_sweep_bits_dp) over windows {k}-{P - 1} of the "
                       + ("canonical copy (each undirected pair once)"
                          if run_info["split_parts_canonical"] else "check copy")
                       + ", bits published as vertices reach the root label")
    roofline = {"bound": "hbm", "achieved": b_sweep / t_sweep / 1e9, "peak": peak, "unit": "GB/s",
                "frac": b_sweep / t_sweep / 1e9 / peak,
                "traffic": traffic.get("dram_bytes_per_launch"),
                "kernel": kernel_text + " + one shortcut pass",
                "launch_ms": [round(t * 1e3, 4) for t in rt1],
                "bytes_per_launch": b_sweep, "avg_launch_s": t_sweep,
                "bytes_definition": "B_sweep = 8 m (src+dst uint32 stream) + 4 n (one label "
                                    "read), SURVEY 8(d); gathers and write-backs excluded",
                "peak_source": peak_src}
    if rtc:
        t_chk = sum(rtc) / len(rtc)
        roofline["check_kernel"] = {
            "what": "early convergence check (edge agreement + idempotence), passing",
            "avg_launch_s": t_chk, "bytes_per_launch": b_sweep,
            "achieved": b_sweep / t_chk / 1e9, "frac": b_sweep / t_chk / 1e9 / peak,
            "traffic": traffic.get("check_dram_bytes_per_launch")}
        info = ctx.layout_info()
        if info.get("canon_rows"):
            # layout 6: the check walks the canonical copy (each undirected pair once)
            # + the label array (idempotence, bitmap) + the bitmap
            bc = info["canon_bytes"] + 4 * n + n // 8
            roofline["check_kernel"].update({
                "kernel": "k_pick_root + k_bits_idem + k_check_bits_dp over the canonical check "
                          "copy (each undirected pair once, delta-packed)"
                          + ("; the timed runs end on its uniting form k_unite_bits_dp (same "
                             "stream; rows whose labels differ are united, then pointer "
                             "jumping) -- run minus sweep 1: "
                             f"{ms - t_sweep * 1e3:.2f} ms" if run_info["uniting_check"] else ""),
                "canonical_copy": {"rows": info["canon_rows"], "bytes": info["canon_bytes"],
                                   "side_groups": info["canon_side_groups"]},
                "streamed_bytes_per_launch": bc, "frac_streamed": bc / t_chk / 1e9 / peak})
    if rt2 and hybrid:  # hybrid layout: later sweeps run the shared-memory slice kernel
        t2 = sum(rt2) / len(rt2)
        b2 = 6 * m + 4 * n  # compact bucketed copy: 4 B src + 2 B dst offset per row
        roofline["slice_kernel"] = {
            "kernel": "cck::k_sweep_slice (dst-bucketed copy, dst labels in shared memory)",
            "avg_launch_s": t2, "frac_of_B_sweep": b_sweep / t2 / 1e9 / peak,
            "streamed_bytes_per_launch": b2, "frac_streamed": b2 / t2 / 1e9 / peak}
    elif rt2:  # layout 6: later sweeps are the bitmap sweep over a row copy
        t2 = sum(rt2) / len(rt2)
        # the copy it walks as staged (cc_layout_info): the canonical copy (each
        # undirected pair once, CC_OPT_CANON_SWEEP default) when it was built,
        # else the dst-bucketed check copy (delta-packed groups, 4.03 B per
        # row; or 6 / 8 B rows) + the bitmap + the vertex pass's label read
        info = ctx.layout_info()
        canon = bool(info.get("canon_rows"))
        cb = info["canon_bytes"] if canon else info["check_bytes"]
        b2 = cb + n // 8 + 4 * n
        roofline["bitmap_sweep_kernel"] = {
            "kernel": "k_pick_root + k_bits_idem + k_sweep_bits_dp over the "
                      + ("canonical copy (each undirected pair once; the operator is symmetric "
                         "in u, v)" if canon else "dst-bucketed check copy")
                      + ", component bitmap; rows both of whose ends carry the root label are "
                        "decided without label gathers",
            "check_copy": {"format": {2: "delta-packed 128-row groups", 1: "6-byte rows",
                                      0: "8-byte rows"}.get(info["check_format"]),
                           "bytes": info["check_bytes"],
                           "bytes_per_row": round(info["check_bytes"] / max(m, 1), 3)},
            "walks": "canonical copy" if canon else "check copy",
            "avg_launch_s": t2, "frac_of_B_sweep": b_sweep / t2 / 1e9 / peak,
            "streamed_bytes_per_launch": b2, "frac_streamed": b2 / t2 / 1e9 / peak,
            "launch_ms": [round(t * 1e3, 4) for t in rt2]}

    # ---- the paper's comparison baseline on the same device and staged edges
    fsv = None
    if args.fastsv > 0:
        from paper_2311_02811_b200.baselines import fastsv_staged
        fastsv_staged(ctx, sweep_times=False)  # untimed: scratch allocation, module load
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        fst = None
        for _ in range(args.fastsv):
            _, fst = fastsv_staged(ctx, sweep_times=False)
        f1.record(stream)
        torch.cuda.synchronize()
        fms = f0.elapsed_time(f1) / args.fastsv
        fsv = {"value": m / (fms / 1e3), "unit": UNIT, "ms_per_step": fms,
               "iterations": fst.sweeps_executed, "contour_speedup": fms / ms,
               "what": "GPU FastSV (synchronous hooking + shortcutting, baselines.py:81-131) "
                       "on the same staged edges; the paper's comparison baseline"}
    ctx.close()  # frees the resident graph before the e2e leg stages its own
    del ctx

    # ---- e2e: the drop-in call on the reference's input type, host clock
    e2e = None
    if not args.no_e2e:
        from paper_2311_02811_b200 import run_contour
        walls, st_e = [], None
        ok = True
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            labels, st_e = run_contour((n, host_edges), sched, layout=args.e2e_layout)
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                walls.append(dt)
            if i == 0:
                ok = bool(np.array_equal(labels, dev_labels))
            del labels
        e2e_s = sum(walls) / len(walls)
        e2e = {"value": m / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(host_edges.nbytes), "d2h_bytes_per_step": int(n * 8),
               "seconds_per_step": e2e_s, "seconds_min": min(walls),
               "seconds_median": statistics.median(walls),
               "step_seconds": [round(w, 3) for w in walls],
               "path": f"run_contour((n, edges), make_schedule('c2', atomic={atomic}), "
                       f"layout={args.e2e_layout!r}) -- the drop-in with the reference's defaults "
                       f"(exact change counts, early check), pageable {host_edges.dtype} (m, 2) "
                       f"numpy edges (writeable: restaged every call), labels -> a fresh int64 "
                       f"numpy array; host wall clock around the call",
               "sweeps_executed": st_e.sweeps_executed, "converged_by": st_e.converged_by,
               "labels_equal_device_resident_run": ok}

    # ---- CPU baseline: the reference on a bounded sample of the workload
    cpu, ref_sweeps = None, None
    if not args.no_cpu_baseline:
        cpu, ref_sweeps = cpu_baseline_leg(args, device)
    del host_edges

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": shared_config(args.config, n, m, atomic),
        "impl_detail": {"layout": layout, "store_mode": store_mode_name(atomic, args.store_mode),
                        "early_check": early,
                        "termination": ("a no-write sweep, or the early check after a changing "
                                        "sweep (engine.py:318-320) in its uniting form: rows "
                                        "whose labels differ are united (larger root lowered "
                                        "to the smaller), pointer jumping finishes the labels "
                                        "-- DESIGN 5.32; `plain_check` = the same runs with "
                                        "the plain check") if run_info["uniting_check"] else
                                       "ballot/OR no-write flag or the early check "
                                       "(engine.py:318-320)",
                        "layout_build_s": round(layout_s, 3), "prep_s": round(prep_s, 2),
                        "value_excludes": "input generation and the staging-time layout "
                                          "(layout_build_s); e2e includes staging + layout",
                        "parallelism": "single GPU"},
        "sweeps_per_run": [s.sweeps_executed for s in stats],
        "sweep_ms": [round(t * 1e3, 4) for t in sweep_ms_graph],
        "verified": verify == 0,
        "plain_check": plain,
        "reference_sweeps": ref_sweeps,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "fastsv_baseline": fsv,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_leg(args, device):
    """The reference (baseline/_ref, else the port) on the bounded sample,
    all host threads, one timed run; plus the port's time, and the sweep
    counts of the device next to the reference's on the same sample (async,
    and sync where the device must reproduce them exactly)."""
    from paper_2311_02811_b200 import run_contour
    from paper_2311_02811_b200.engine import make_schedule
    threads = os.cpu_count() or 1
    atomic = bool(args.atomic)
    n, e, m_full = sample_edges(args.config, args.seed, args.sample_rows)
    rows = int(e.shape[0])
    ref = reference_impl()
    use_ref = ref is not None and not hasattr(ref, "error")
    port_t, port_st, port_lab = time_port(n, e, threads, atomic, 1)
    if use_ref:
        time_reference(ref, n, e, threads, atomic, 1)  # numba JIT
        rt, rst, rlab = time_reference(ref, n, e, threads, atomic, 1)
    else:
        rt, rst, rlab = port_t, port_st, port_lab
    cpu = {"value": rows / rt[0], "unit": UNIT, "cores": threads,
           "kind": "reference" if use_ref else "port", "cores_physical": physical_cores(),
           "what": (f"minmapcc {ref.version} (unmodified, numba) from baseline/_ref"
                    if use_ref else "oracle/ C port of run_contour"),
           "sample": sample_desc(args.config, rows, m_full, n) + f"; 1 timed run, {rt[0]:.2f} s",
           "port": {"value": rows / port_t[0], "seconds": port_t[0]}}
    # the device on the same sample, through the drop-in (labels must match)
    labels, dst = run_contour((n, e), make_schedule("c2", atomic=atomic), device=device)
    _, sync_ref = time_port(n, e, threads, atomic, 1, sync=True)[:2]
    _, sync_dev = run_contour((n, e), make_schedule("c2", sync=True), device=device)
    ref_sweeps = {"on": "the CPU legs' sample",
                  "reference_async": {"executed": int(rst.sweeps_executed),
                                      "until_stable": int(rst.sweeps_until_stable),
                                      "converged_by": rst.converged_by},
                  "device_async": {"executed": dst.sweeps_executed,
                                   "until_stable": dst.sweeps_until_stable,
                                   "converged_by": dst.converged_by},
                  "labels_equal": bool(np.array_equal(labels, rlab)),
                  "sync_c2_reference": list(sync_ref.changed_per_sweep),
                  "sync_c2_device": list(sync_dev.changed_per_sweep),
                  "sync_equal": list(sync_ref.changed_per_sweep) == sync_dev.changed_per_sweep}
    return cpu, ref_sweeps


# ---------------------------------------------------------------- N GPUs
def run_multi(args, rank, world, device):
    import torch
    import torch.distributed as dist

    from paper_2311_02811_b200 import _lib, distributed, engine

    spec = CONFIGS[args.config]
    if spec["kind"] != "rmat":
        raise SystemExit("multi-GPU bench supports the RMAT configs")
    atomic = bool(args.atomic)
    stream = torch.cuda.Stream(device)
    torch.cuda.set_stream(stream)
    exchange = args.exchange
    keep_host = not args.no_e2e
    runner = None
    if exchange == "checked":
        runner = distributed.CheckedShardedContour.from_rmat(
            spec["scale"], spec.get("edgefactor", 16), args.seed, rank, world, device,
            layout=args.layout, atomic=atomic, keep_host=keep_host)
        if dist.get_backend() == "gloo":
            def gloo_min_checked(t):  # plumbing-check runs (ranks sharing a GPU)
                c = t.cpu()
                dist.all_reduce(c, op=dist.ReduceOp.MIN)
                t.copy_(c)
            runner.allreduce = gloo_min_checked
    if exchange in ("peer", "hybrid"):
        try:  # fused sweep + red.min into the peers' replicas (CUDA IPC over NVLink)
            cls = (distributed.HybridShardedContour if exchange == "hybrid"
                   else distributed.FusedShardedContour)
            runner = cls.from_rmat(spec["scale"], spec.get("edgefactor", 16), args.seed, rank,
                                   world, device, layout=args.layout, atomic=atomic,
                                   keep_host=keep_host)
            if exchange == "hybrid" and dist.get_backend() == "gloo":
                def gloo_min(t):  # plumbing-check runs (ranks sharing a GPU)
                    c = t.cpu()
                    dist.all_reduce(c, op=dist.ReduceOp.MIN)
                    t.copy_(c)
                runner.allreduce = gloo_min
        except RuntimeError as exc:  # no IPC peer mapping on this node: use NCCL, say so
            exchange = f"nccl (peer IPC unavailable: {str(exc)[:80]})"
    if runner is None:
        runner = distributed.ShardedContour.from_rmat(spec["scale"], spec.get("edgefactor", 16),
                                                      args.seed, rank, world, device,
                                                      layout=args.layout, cadence=args.cadence,
                                                      atomic=atomic, keep_host=keep_host)
    n, m_total = runner.n, runner.m_total
    for _ in range(args.warmup):
        runner.run()
    dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(device) if rank == 0 else None
    if clocks:
        clocks.start()
    for _ in range(4):  # untimed runs under the sampler; a fixed count (collectives inside)
        runner.run()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    rounds = []
    for _ in range(args.steps):
        rounds.append(runner.run())
    ev1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    tdev = "cuda" if dist.get_backend() == "nccl" else "cpu"

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device=tdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    clk = clocks.stop() if clocks else None

    # ---- roofline of the per-rank sweep kernel: one order-2 sweep of this
    # rank's shard on the converged replica (no lowerings, so no peer
    # traffic), CUDA events on the launching stream, max over ranks
    sctx = runner.shard.ctx
    fused_now = isinstance(runner, distributed.FusedShardedContour)
    sweep_ts = []
    for _ in range(3):
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        _lib.check(sctx.lib.cc_sweep(sctx.handle, 2, 0, int(atomic), 0, None))
        s1.record(stream)
        torch.cuda.synchronize()
        sweep_ts.append(s0.elapsed_time(s1) / 1e3)
    t_sw = max_over_ranks(sum(sweep_ts) / len(sweep_ts))
    m_g = max(hi_ - lo_ for lo_, hi_ in (distributed.shard_rows(m_total, r, world)
                                          for r in range(world)))
    b_sw = 8 * m_g + 4 * n
    peak, peak_src = peak_hbm()
    roofline = {"bound": "hbm", "achieved": b_sw / t_sw / 1e9, "peak": peak, "unit": "GB/s",
                "frac": b_sw / t_sw / 1e9 / peak, "traffic": None,
                "kernel": ("cck::k_sweep_o2_peers (fused sweep + peer red.min)" if fused_now
                           else "cck::k_sweep<2, ...>") + ", one rank's shard",
                "bytes_per_launch": b_sw, "avg_launch_s": t_sw,
                "note": "per GPU: 8 B x the largest shard's rows + 4 B x n, over the slowest "
                        "rank's confirming-sweep time",
                "peak_source": peak_src}
    # certificate over all shards: every rank checks its edges on its replica
    bad = max_over_ranks(engine.verify_staged(runner.shard.ctx))

    # ---- e2e at N GPUs: every rank stages ITS host shard (pageable, its own
    # PCIe link, laid out on arrival) and the ranks run to convergence; rank 0
    # reads the int64 labels back.  Time = max over ranks of the host clock.
    e2e = None
    if keep_host:
        host = runner.host_edges
        labels_out = np.empty(n if rank == 0 else 1, dtype=np.int64)
        times = []
        for i in range(args.warmup + args.steps):
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            runner.stage_host(host, args.layout)
            runner.run()
            if rank == 0:
                runner.read_labels(labels_out)
            torch.cuda.synchronize()
            if i >= args.warmup:
                times.append(time.perf_counter() - t0)
        e2e_s = max_over_ranks(sum(times) / len(times))
        e2e = {"value": m_total / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(m_total * 2 * host.dtype.itemsize),
               "d2h_bytes_per_step": int(n * 8), "seconds_per_step": e2e_s,
               "path": f"per rank: cc_stage_edges(pageable {host.dtype} shard) + layout + the "
                       f"sharded run; rank 0: labels -> int64 numpy; host clock, max over ranks"}
    fused = isinstance(runner, (distributed.FusedShardedContour,
                                distributed.HybridShardedContour))
    if isinstance(runner, distributed.CheckedShardedContour):
        sched = ("per sweep: the local sweep (sweep 1 split, later bitmap sweeps) + shortcut, "
                 "all-reduce-MIN of the labels, the early check on each shard (canonical check "
                 "copy) AND-ed by a 1-word MIN all-reduce")
        launches = sum(2 + r * 20 for r in rounds)  # init + ~20 kernels per round + compress
    elif isinstance(runner, distributed.HybridShardedContour):
        sched = ("round 1: local sweep + shortcut, all-reduce-MIN of the n+1 labels; later "
                 "rounds: fused sweep + red.min into the peer replicas (CUDA IPC / NVLink), "
                 "1-word MAX all-reduce")
        launches = sum(5 + r for r in rounds)  # init, sweep, fold, shortcut, +1/round, compress
    elif fused:
        sched = ("fused sweep + red.min into the peer replicas (CUDA IPC / NVLink), 1-word MAX "
                 "all-reduce per round")
        launches = sum(2 + r for r in rounds)  # init + fused sweep per round + compress
    else:
        sched = f"NCCL all-reduce-MIN every {args.cadence} local sweep(s)"
        launches = sum(2 + r * args.cadence * 3 for r in rounds)
    if rank == 0:
        line = {
            "metric": METRIC, "value": m_total / (ms / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic", "config": shared_config(args.config, n, m_total, atomic),
            "impl_detail": {"exchange": exchange, "exchange_schedule": sched,
                            "layout": runner.layout,
                            "store_mode": store_mode_name(atomic, args.store_mode),
                            "parallelism": f"edge-sharded x{world}, labels replicated"},
            "exchanges_per_run": rounds,
            "verified": int(bad) == 0,
            "roofline": roofline,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if fused:
        dist.barrier()
        runner.shard.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
