"""Benchmark: Contour CC throughput (input edges/s to converged labels) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config rmat22]
                    [--impl b200|reference] [--no-cpu-baseline]

Workload (BASELINE.json configs[1]): RMAT scale 22, edgefactor 16,
symmetrised -> n = 4,194,304 vertices, m = 134,217,728 input edge rows,
seeded synthetic.  One step = one whole run of the
hot path: labels = arange(n) -> order-2 asynchronous sweeps until a sweep
lowers nothing -> pointer-jumping compress, with the edges already resident
in HBM (the edge list, 1.07 GB, is larger than the 126 MB L2, so no extra
flush is needed between steps).

N > 1 (torchrun, one rank per GPU): the same graph's edges are split into N
contiguous shards, labels replicated, and after every local sweep an
in-place NCCL all-reduce(MIN) over n+1 int32 (slot n folds "any rank
lowered a label").  Strong scaling (total work fixed).

--impl reference: the reference's CPU implementation (the oracle port of
run_contour, oracle/, all host threads) on the same workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CC throughput: input edges/s to converged labels; per-sweep HBM GB/s vs peak"
UNIT = "edges/s"
HBM_FALLBACK_GBS = 6650.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="rmat22")
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--early-check", default="auto", choices=["auto", "on", "off"],
                   help="the reference's early convergence check after each changing sweep "
                        "(engine.py:318-320), inside the device loop.  auto: on for the hybrid "
                        "layout, whose shared-memory check (0.18 ms on RMAT-22) is cheaper "
                        "than the confirming sweep it saves, and for L2-window tiles (RMAT-28 "
                        "78 vs 82 ms, forest 693 vs 701 ms); off on flat chunk-sorted rows, "
                        "where the check costs what that sweep costs (RMAT-22 1.19 vs 1.15 ms)")
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--layout", default="auto",
                   choices=["auto", "input", "src_sorted", "chunk_sorted", "dst_bucketed",
                            "l2_tiled", "hybrid"],
                   help="staging-time edge layout (auto: chunk_sorted -- each 2^23-row chunk "
                        "radix-sorted by src on device while the next chunk is copied in -- "
                        "when the labels fit L2, l2_tiled windows otherwise)")
    p.add_argument("--first-scatter", action="store_true",
                   help="run sweep 1 as the load-free identity scatter")
    p.add_argument("--host-loop", action="store_true",
                   help="drive sweeps from the host instead of the CUDA-graph WHILE loop "
                        "(same kernels; ncu cannot see kernels inside conditional nodes)")
    p.add_argument("--no-e2e", action="store_true", help="skip the end-to-end leg")
    p.add_argument("--no-fastsv", action="store_true", help="skip the GPU FastSV comparison")
    p.add_argument("--sharded", action="store_true",
                   help="use the edge-sharded NCCL driver even with one rank (plumbing check)")
    p.add_argument("--cadence", type=int, default=1,
                   help="local sweeps per MIN exchange in the sharded driver")
    p.add_argument("--exchange", default="hybrid", choices=["hybrid", "peer", "nccl"],
                   help="multi-GPU label exchange: hybrid (default: one all-reduce-MIN "
                        "after the local sweep 1, then fused red.min into the peer replicas), "
                        "peer (fused from the start, CUDA IPC) or nccl (all-reduce-MIN every "
                        "--cadence local sweeps)")
    p.add_argument("--clock-interval-ms", type=int, default=100,
                   help="nvidia-smi sampling interval during the timed region")
    p.add_argument("--atomic", type=int, default=1,
                   help="Schedule.atomic (the reference default is True)")
    p.add_argument("--store-mode", type=int, default=None,
                   help="override the async store mode (0 plain, 1 red, 2 check+plain, "
                        "3 check+red)")
    return p.parse_args()


def physical_cores():
    """Physical core count of the host (SURVEY 8(d) asks for it beside the
    logical count the CPU legs use), or None when psutil cannot tell."""
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


def config_spec(name):
    from paper_2311_02811_b200.graphgen import CONFIGS
    if name not in CONFIGS:
        raise SystemExit(f"unknown config {name}")
    return CONFIGS[name]


def workload_name(name, n, m):
    labels = {"rmat22": "configs[1] RMAT scale 22 ef 16 (a,b,c,d)=(.57,.19,.19,.05), permuted, "
                        "symmetrised",
              "er": "configs[0] Erdos-Renyi n=65536 pairs=524288",
              "grid4096": "configs[2] 4096x4096 grid p=0.55 permuted",
              "forest": "configs[3] forest 200k components + 20% isolated",
              "rmat28": "configs[4] RMAT scale 28 ef 16 symmetrised"}
    return f"{labels.get(name, name)} (n={n}, m_input={m})"


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


def cpu_baseline(n, edges, threads, runs=1, atomic=True):
    """The oracle port of run_contour (engine.py:248-328) on the host cores:
    C-2, async, the same Schedule.atomic as the GPU arm, seed=0, early check
    as the reference does."""
    from oracle import oracle
    oracle.lib()
    times, st = [], None
    for _ in range(runs):
        t0 = time.perf_counter()
        _, st = oracle.run_contour(n, edges, "C-2", atomic=atomic, threads=threads, seed=0)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    return t, st


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2311_02811_b200 import graphgen
    spec = config_spec(args.config)
    n, edges = graphgen.make(spec, args.seed, elem_bytes=4)
    m = edges.shape[0]
    threads = os.cpu_count() or 1
    atomic = bool(args.atomic)
    for _ in range(args.warmup):
        cpu_baseline(n, edges, threads, atomic=atomic)
    times, st = [], None
    for _ in range(args.steps):
        t, st = cpu_baseline(n, edges, threads, atomic=atomic)
        times.append(t)
    ms = 1e3 * sum(times) / len(times)
    value = m / (ms / 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": workload_name(args.config, n, m),
                   "schedule": f"C-2 async atomic={atomic}",
                   "parallelism": f"{threads} host threads (static edge chunks, engine.py:296-308)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "cores_physical": physical_cores(),
                         "sample": f"full workload, {args.steps} timed runs after {args.warmup} "
                                   f"warm-up; sweeps_executed={st.sweeps_executed}, "
                                   f"converged_by={st.converged_by}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_sweeps": {"executed": st.sweeps_executed, "until_stable": st.sweeps_until_stable},
    }
    print(json.dumps(line), flush=True)


def load_traffic():
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except Exception:
        return {}


def main():
    args = parse()
    ClockSampler.interval_ms = max(20, args.clock_interval_ms)
    if args.impl == "reference":
        return run_reference_arm(args)
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
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", RANK="0",
                              WORLD_SIZE="1")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
        return run_multi(args, rank, world, local)
    return run_single(args, local)


def run_single(args, device):
    import torch

    from paper_2311_02811_b200 import _lib, engine, graphgen
    from paper_2311_02811_b200.engine import make_schedule

    spec = config_spec(args.config)
    # one dedicated stream: the library launches on it and the CUDA events
    # that time the step are recorded on it
    stream = torch.cuda.Stream(device)
    torch.cuda.set_stream(stream)
    ctx = _lib.Context(device, stream.cuda_stream)
    if args.store_mode is not None:
        ctx.set_option(_lib.CC_OPT_STORE_MODE_ATOMIC if args.atomic else
                       _lib.CC_OPT_STORE_MODE_PLAIN, args.store_mode)
    # ---- inputs resident in HBM in the staged layout (not timed)
    layout_arg = args.layout
    if spec["kind"] == "rmat":
        n, m = graphgen.rmat_device(ctx, spec["scale"], spec.get("edgefactor", 16), args.seed)
        args.layout = engine.resolve_layout(args.layout, m, n)
        if args.layout != "input":
            engine.apply_layout(ctx, args.layout)
        host_edges = None
    else:
        n, host_edges = graphgen.make(spec, args.seed, elem_bytes=4)
        m = host_edges.shape[0]
        args.layout = engine.resolve_layout(args.layout, m, n)
        engine.stage_graph(ctx, n, host_edges, args.layout)
    # e2e is a one-shot run from host memory: "auto" keeps chunk-sorted rows
    # there so sweep 1 streams behind the copy (engine.resolve_layout)
    e2e_layout = engine.resolve_layout(layout_arg, m, n, resident=False)

    def early_for(layout):
        return args.early_check == "on" or (args.early_check == "auto" and
                                            layout in ("hybrid", "l2_tiled"))

    args.early = early_for(args.layout)
    hybrid = args.layout == "hybrid"
    sched = make_schedule("c2", atomic=bool(args.atomic))
    kw = dict(count_changes=False, early_check=args.early,
              first_scatter=args.first_scatter, host_loop=args.host_loop)

    for _ in range(args.warmup):
        engine.run_staged(ctx, sched, sweep_times=False, **kw)
    torch.cuda.synchronize()

    # ---- timed region: K whole runs, CUDA events on the launching stream
    clocks = ClockSampler(device)
    clocks.start()
    # keep the GPU busy with untimed runs while the sampler warms up, so the
    # sampled clocks are clocks under this load (the timed region itself is
    # a few ms)
    t_busy = time.perf_counter()
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

    sweeps = [s.sweeps_executed for s in stats]
    shortcut = 1  # CC_OPT_SHORTCUT default: one pointer-jumping pass after every sweep
    check = 2 if args.early else 0  # idempotence + edge-agreement kernels
    if args.host_loop:  # iota + (sweep + shortcut + check) per sweep + compress
        launches = sum(2 + s.sweeps_executed * (1 + shortcut + check) for s in stats)
    else:  # iota + loop_init + (guarded sweeps + shortcut + check + control) per sweep + compress
        per = (2 if hybrid else 1) + shortcut + check + 1
        launches = sum(3 + s.sweeps_executed * per for s in stats)

    # ---- roofline of the sweep kernels: their own launch times, CUDA events
    # on the launching stream around each sweep (+ its shortcut pass) in
    # host-driven runs without the check (the graph loop's per-sweep records
    # include control and check kernels).  Hybrid layout: sweep 1 is the
    # chunk-sorted kernel, later sweeps the shared-memory slice kernel.
    rt1, rt2 = [], []
    for _ in range(max(1, min(args.steps, 3))):
        _, st = engine.run_staged(ctx, sched, sweep_times=True, count_changes=False,
                                  early_check=False, host_loop=True)
        if hybrid:
            rt1.append(st.sweep_seconds[0])
            rt2.extend(st.sweep_seconds[1:])
        else:
            rt1.extend(st.sweep_seconds)
    t_sweep = sum(rt1) / len(rt1)
    b_sweep = 8 * m + 4 * n  # edge stream + one label-array read
    achieved = b_sweep / t_sweep / 1e9
    peak, peak_src = peak_hbm()
    traffic = (load_traffic().get(args.config) or {}).get("dram_bytes_per_launch")
    rt = rt1

    # ---- the paper's comparison baseline on the same device and staged edges:
    # GPU FastSV (baselines.py:81-131), not part of `value`
    fsv = None
    if not args.no_fastsv:
        from paper_2311_02811_b200.baselines import fastsv_staged
        fastsv_staged(ctx, sweep_times=False)
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        fst = None
        for _ in range(args.steps):
            _, fst = fastsv_staged(ctx, sweep_times=False)
        f1.record(stream)
        torch.cuda.synchronize()
        fms = f0.elapsed_time(f1) / args.steps
        fsv = {"value": m / (fms / 1e3), "unit": UNIT, "ms_per_step": fms,
               "iterations": fst.sweeps_executed, "contour_speedup": fms / ms,
               "what": "GPU FastSV (synchronous hooking + shortcutting, baselines.py:81-131) "
                       "on the same staged edges; the paper's comparison baseline"}

    # ---- e2e through the C-ABI with HOST buffers (pinned), H2D + D2H timed
    need_host = not (args.no_e2e and args.no_cpu_baseline)
    if need_host and host_edges is None:
        host_edges_t = torch.empty((m, 2), dtype=torch.int32, pin_memory=True)
        graphgen.rmat(spec["scale"], spec.get("edgefactor", 16), args.seed, elem_bytes=4,
                      out=host_edges_t.numpy())
        host_edges = host_edges_t.numpy()
    elif need_host:
        t = torch.empty((m, 2), dtype=torch.int32, pin_memory=True)
        t.numpy()[:] = host_edges
        host_edges = t.numpy()
    e2e = None
    e2e_kw = dict(kw, early_check=early_for(e2e_layout))
    if not args.no_e2e:
        labels_t = torch.empty(n, dtype=torch.int64, pin_memory=True)
        labels_host = labels_t.numpy()
        e2e_times = []
        for i in range(args.warmup + args.steps):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            # run_contour's host-graph path: one cc_run_host call (sweep 1
            # streamed behind the copy where the layout allows it)
            engine.run_host(ctx, n, host_edges, sched, layout=e2e_layout, sweep_times=False,
                            labels_out=labels_host, **e2e_kw)
            b.record(stream)
            torch.cuda.synchronize()
            if i >= args.warmup:
                e2e_times.append(a.elapsed_time(b) / 1e3)
        e2e_s = sum(e2e_times) / len(e2e_times)
        e2e = {"value": m / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(host_edges.nbytes),
               "d2h_bytes_per_step": int(labels_host.nbytes), "seconds_per_step": e2e_s,
               "path": "cc_run_host(pinned int32 (m,2) edges, chunk-sorted and swept while "
                       "copying; labels -> pinned int64), the run_contour host-graph path"}

    # ---- the drop-in call on the reference's own input type: run_contour(g,
    # make_schedule("c2")) with its defaults (exact counts, early check) on a
    # pageable (m, 2) int64 numpy array, labels into a fresh numpy array; host
    # wall clock around the whole call (informational, beside `e2e`)
    dropin = None
    if not args.no_e2e:
        from paper_2311_02811_b200 import run_contour
        e64 = np.ascontiguousarray(host_edges, dtype=np.int64)
        run_contour((n, e64), sched)
        walls = []
        for _ in range(3):
            t0 = time.perf_counter()
            run_contour((n, e64), sched)
            walls.append(time.perf_counter() - t0)
        dropin = {"value": m / min(walls), "unit": UNIT, "seconds": min(walls),
                  "call": "run_contour((n, edges), make_schedule('c2')) -- reference defaults, "
                          "pageable int64 (m, 2) numpy edges, int64 numpy labels; host wall "
                          "clock, best of 3"}
        del e64

    # ---- CPU baseline: the reference path (oracle port) on the host cores
    cpu = None
    if not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        t_cpu, st_cpu = cpu_baseline(n, host_edges, threads, atomic=bool(args.atomic))
        cpu = {"value": m / t_cpu, "unit": UNIT, "cores": threads, "kind": "port",
               "cores_physical": physical_cores(),
               "sample": f"1 full run of the same workload (oracle port of run_contour, C-2 "
                         f"async atomic={bool(args.atomic)}, {threads} threads): {t_cpu:.2f} s, "
                         f"sweeps_executed={st_cpu.sweeps_executed}"}
        ref_sweeps = {"executed": st_cpu.sweeps_executed, "until_stable": st_cpu.sweeps_until_stable}
        # the reference's 1-thread time and its synchronous C-2
        # counts (deterministic: the device's sync run must match them)
        from oracle import oracle
        t1 = time.perf_counter()
        _, st1 = oracle.run_contour(n, host_edges, "C-2", atomic=bool(args.atomic), threads=1,
                                    seed=0)
        t1 = time.perf_counter() - t1
        cpu["threads_1"] = {"value": m / t1, "seconds": t1, "sweeps_executed": st1.sweeps_executed}
        _, sts = oracle.run_contour(n, host_edges, "C-2", sync=True, threads=threads, seed=0)
        ref_sweeps["sync_c2"] = {"executed": sts.sweeps_executed,
                                 "until_stable": sts.sweeps_until_stable,
                                 "changed_per_sweep": list(sts.changed_per_sweep)}
        _, stg = engine.run_staged(ctx, make_schedule("c2", sync=True), count_changes=True,
                                   early_check=True, sweep_times=False)
        ref_sweeps["sync_c2_device"] = {"executed": stg.sweeps_executed,
                                        "until_stable": stg.sweeps_until_stable,
                                        "changed_per_sweep": stg.changed_per_sweep,
                                        "equal": stg.changed_per_sweep == list(sts.changed_per_sweep)}
    else:
        ref_sweeps = None

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": workload_name(args.config, n, m), "n": n, "m_input": m,
                   "schedule": f"C-2 async atomic={bool(args.atomic)}, ballot/OR flag"
                               + (", early check (engine.py:318-320)" if args.early else "")
                               + (", load-free sweep 1" if args.first_scatter else ""),
                   "layout": args.layout,
                   "e2e_layout": e2e_layout,
                   "parallelism": "single GPU",
                   "l2": "inputs larger than L2 (edge stream 8m B > 126 MB); no flush"},
        "sweeps_per_run": sweeps,
        # per-sweep device times of one untimed run (the timed runs skip the records)
        "sweep_ms": [round(t * 1e3, 4) for t in
                     engine.run_staged(ctx, sched, sweep_times=True, **kw)[1].sweep_seconds],
        "reference_sweeps": ref_sweeps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "cck::k_sweep<2, 3, 1, 1> (order-2 async sweep, check+red stores, "
                               "4 rows/thread) + one shortcut pass",
                     "launch_ms": [round(t * 1e3, 4) for t in rt],
                     "bytes_per_launch": b_sweep, "avg_launch_s": t_sweep,
                     "peak_source": peak_src},
        # hybrid layout: the later sweeps' kernel (shared-memory dst slices)
        "roofline_slice_kernel": None if not rt2 else {
            "bound": "hbm", "kernel": "cck::k_sweep_slice<3, true> (dst-bucketed copy, dst labels "
                                      "in shared memory) + one shortcut pass",
            "achieved": b_sweep / (sum(rt2) / len(rt2)) / 1e9, "peak": peak, "unit": "GB/s",
            "frac": b_sweep / (sum(rt2) / len(rt2)) / 1e9 / peak,
            "launch_ms": [round(t * 1e3, 4) for t in rt2]},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "e2e_dropin_pageable_int64": dropin,
        "gpu_launches": launches,
        "fastsv_baseline": fsv,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    ctx.close()


def run_multi(args, rank, world, device):
    import torch
    import torch.distributed as dist

    from paper_2311_02811_b200 import distributed, engine, graphgen

    spec = config_spec(args.config)
    if spec["kind"] != "rmat":
        raise SystemExit("multi-GPU bench supports the RMAT configs")
    stream = torch.cuda.Stream(device)
    torch.cuda.set_stream(stream)
    exchange = args.exchange
    runner = None
    if exchange in ("peer", "hybrid"):
        try:  # fused sweep + red.min into the peers' replicas (CUDA IPC over NVLink)
            cls = (distributed.HybridShardedContour if exchange == "hybrid"
                   else distributed.FusedShardedContour)
            runner = cls.from_rmat(spec["scale"], spec.get("edgefactor", 16), args.seed, rank,
                                   world, device, layout=args.layout, atomic=bool(args.atomic))
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
                                                      atomic=bool(args.atomic))
    n, m_total = runner.n, runner.m_total
    for _ in range(args.warmup):
        runner.run()
    dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(device) if rank == 0 else None
    if clocks:
        clocks.start()
    for _ in range(16):  # untimed runs under the sampler; a fixed count (collectives inside)
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
    from paper_2311_02811_b200 import _lib
    sctx = runner.shard.ctx
    fused_now = isinstance(runner, distributed.FusedShardedContour)
    sweep_ts = []
    for _ in range(3):
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        _lib.check(sctx.lib.cc_sweep(sctx.handle, 2, 0, int(bool(args.atomic)), 0, None))
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
                           else "cck::k_sweep<2, 3, 1, 1>") + ", one rank's shard",
                "bytes_per_launch": b_sw, "avg_launch_s": t_sw,
                "note": "per GPU: 8 B x the largest shard's rows + 4 B x n, over the slowest "
                        "rank's confirming-sweep time",
                "peak_source": peak_src}
    # certificate over all shards: every rank checks its edges on its replica
    bad = max_over_ranks(engine.verify_staged(runner.shard.ctx))

    # ---- e2e at N GPUs: every rank stages ITS host shard (pinned int32, its
    # own PCIe link) and the ranks run to convergence; rank 0 reads the int64
    # labels back.  Time = max over ranks of the per-rank CUDA-event time.
    e2e = None
    if not args.no_e2e:
        lo, hi = distributed.shard_rows(m_total, rank, world)
        host_t = torch.empty((hi - lo, 2), dtype=torch.int32, pin_memory=True)
        graphgen.rmat(spec["scale"], spec.get("edgefactor", 16), args.seed, elem_bytes=4,
                      row_lo=lo, row_hi=hi, out=host_t.numpy())
        labels_t = torch.empty(n if rank == 0 else 1, dtype=torch.int64, pin_memory=True)
        times = []
        for i in range(args.warmup + args.steps):
            dist.barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            runner.stage_host(host_t.numpy(), args.layout)
            runner.run()
            if rank == 0:
                runner.read_labels(labels_t.numpy())
            b.record(stream)
            torch.cuda.synchronize()
            if i >= args.warmup:
                times.append(a.elapsed_time(b) / 1e3)
        e2e_s = max_over_ranks(sum(times) / len(times))
        e2e = {"value": m_total / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(m_total * 8), "d2h_bytes_per_step": int(n * 8),
               "seconds_per_step": e2e_s,
               "path": "per rank: cc_stage_edges(pinned int32 shard, chunk-sorted while "
                       "copying) + the sharded run; rank 0: labels -> pinned int64"}
    fused = isinstance(runner, (distributed.FusedShardedContour,
                                distributed.HybridShardedContour))
    if isinstance(runner, distributed.HybridShardedContour):
        sched = (f"C-2 async atomic={bool(args.atomic)}; round 1: local sweep + shortcut, "
                 f"all-reduce-MIN of the n+1 labels; later rounds: fused sweep + red.min into "
                 f"the peer replicas (CUDA IPC / NVLink), 1-word MAX all-reduce")
        launches = sum(5 + r for r in rounds)  # init, sweep, fold, shortcut, +1/round, compress
    elif fused:
        sched = (f"C-2 async atomic={bool(args.atomic)}, fused sweep + red.min into the peer "
                 f"replicas (CUDA IPC / NVLink), 1-word MAX all-reduce per round")
        launches = sum(2 + r for r in rounds)  # init + fused sweep per round + compress
    else:
        sched = (f"C-2 async atomic={bool(args.atomic)}, NCCL allreduce-min every "
                 f"{args.cadence} local sweep(s)")
        # init + per sweep (sweep + fold + shortcut) + compress
        launches = sum(2 + r * args.cadence * 3 for r in rounds)
    if rank == 0:
        line = {
            "metric": METRIC, "value": m_total / (ms / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic",
            "config": {"workload": workload_name(args.config, n, m_total), "n": n,
                       "m_input": m_total, "schedule": sched, "exchange": exchange,
                       "layout": runner.layout,
                       "parallelism": f"edge-sharded x{world}, labels replicated",
                       "l2": "inputs larger than L2"},
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
