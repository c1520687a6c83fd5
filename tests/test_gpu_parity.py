"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle and
the fixtures made from the reference.  Labels must be bit-exact; synchronous
runs must also reproduce the reference's per-sweep accounting exactly
(SURVEY.md Finding 4)."""

import hashlib

import os

import numpy as np
import pytest

from oracle import gen as spec
from oracle import oracle
from paper_2311_02811_b200 import (IterationCapExceeded, VARIANTS, make_schedule, mm_order,
                                   run_contour)
from paper_2311_02811_b200 import _lib, engine, graphgen

pytestmark = pytest.mark.gpu

ALL_MODES = [(v, s) for v in VARIANTS for s in ((True,) if v == "C-Syn" else (True, False))]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def check_invariants(labels, stats):
    assert stats.sweeps_until_stable <= stats.sweeps_executed <= stats.sweeps_until_stable + 1
    assert stats.converged_by in ("change-flag", "early-check")
    assert len(stats.changed_per_sweep) == stats.sweeps_executed
    assert len(stats.sweep_seconds) == stats.sweeps_executed
    assert oracle.is_star_forest(labels)


# ---------------------------------------------------------------- operator
def test_mm_order_known_answers_on_device(golden):
    for case in golden["mm_order"]:
        read = np.asarray(case["labels"], dtype=np.int64)
        tgt = read.copy()
        ch = mm_order(tgt, read, case["w"], case["v"], case["order"])
        assert tgt.tolist() == case["target"] and ch == case["changed"], case
        inplace = read.copy()
        ch2 = mm_order(inplace, inplace, case["w"], case["v"], case["order"])
        assert inplace.tolist() == case["inplace"] and ch2 == case["inplace_changed"], case


# ---------------------------------------------------------------- small graphs
def test_small_graphs_all_modes(golden):
    for g in golden["graphs"]:
        e = np.asarray(g["edges"], dtype=np.int64).reshape(-1, 2)
        for key, exp in g["runs"].items():
            variant, mode, ho = key.split("|")
            sync = mode == "sync"
            sched = make_schedule(variant, int(ho), sync=sync)
            labels, st = run_contour((g["n"], e), sched)
            assert labels.tolist() == g["labels"], (g["name"], key)
            check_invariants(labels, st)
            if sync:  # deterministic: every stat equals the reference's
                assert st.sweeps_executed == exp["executed"], (g["name"], key)
                assert st.sweeps_until_stable == exp["until_stable"], (g["name"], key)
                assert st.changed_per_sweep == exp["changed"], (g["name"], key)
                assert st.converged_by == exp["converged_by"], (g["name"], key)


def test_small_graphs_plain_and_atomic_async(golden):
    for g in golden["graphs"][:60]:
        e = np.asarray(g["edges"], dtype=np.int64).reshape(-1, 2)
        for atomic in (False, True):
            for early in (False, True):
                labels, st = run_contour((g["n"], e), make_schedule("c2", atomic=atomic),
                                         early_check=early, count_changes=early)
                assert labels.tolist() == g["labels"], g["name"]
                check_invariants(labels, st)


# ---------------------------------------------------------------- configs
def _config_edges(params):
    k = params["kind"]
    if k == "er":
        return graphgen.erdos_renyi(params["n"], params["pairs"], params["seed"])
    if k == "rmat":
        return graphgen.rmat(params["scale"], params["ef"], params["seed"])
    if k == "grid":
        return graphgen.grid(params["rows"], params["cols"], params["p"], params["seed"])
    return graphgen.forest(params["components"], params["seed"])


def test_config_shaped_inputs_against_reference_fixtures(golden):
    for c in golden["configs"]:
        n, e = _config_edges(c["params"])
        assert sha(e) == c["edges_sha256"]
        for key, exp in c["runs"].items():
            variant, mode, ho = key.split("|")
            sync = mode == "sync"
            labels, st = run_contour((n, e), make_schedule(variant, int(ho), sync=sync))
            assert sha(labels) == c["labels_sha256"], (c["name"], key)
            check_invariants(labels, st)
            if sync:
                assert (st.sweeps_executed, st.sweeps_until_stable, st.changed_per_sweep,
                        st.converged_by) == (exp["executed"], exp["until_stable"],
                                             exp["changed"], exp["converged_by"]), (c["name"], key)


@pytest.mark.parametrize("cfg", ["er", "grid1024", "rmat18", "forest2k"])
def test_mid_size_against_oracle(cfg):
    if cfg == "er":
        n, e = graphgen.erdos_renyi(65536, 524288, 1)
    elif cfg == "grid1024":
        n, e = graphgen.grid(1024, 1024, 0.55, 2)
    elif cfg == "rmat18":
        n, e = graphgen.rmat(18, 16, 3)
    else:
        n, e = graphgen.forest(2000, 5)
    exp = oracle.rem_union_find(n, e)
    for sched in (make_schedule("c2", atomic=False), make_schedule("c2"), make_schedule("cm"),
                  make_schedule("c2", sync=True), make_schedule("c1m1m")):
        labels, st = run_contour((n, e), sched)
        assert np.array_equal(labels, exp), (cfg, sched)
        check_invariants(labels, st)
    ref_sync = oracle.run_contour(n, e, "C-2", sync=True, threads=8)[1]
    st = run_contour((n, e), make_schedule("c2", sync=True))[1]
    assert st.changed_per_sweep == ref_sync.changed_per_sweep
    assert st.sweeps_executed == ref_sync.sweeps_executed


def test_rmat22_bench_config_exact():
    """configs[1] at full size (the bench workload), generated on device."""
    n, e = graphgen.rmat(22, 16, 1, elem_bytes=4)
    exp = oracle.rem_union_find(n, e)
    ctx = _lib.Context(0)
    graphgen.rmat_device(ctx, 22, 16, 1)
    labels = np.empty(n, dtype=np.int64)
    _, st = engine.run_staged(ctx, make_schedule("c2", atomic=False), count_changes=False,
                              early_check=False, labels_out=labels)
    assert np.array_equal(labels, exp)
    assert st.converged_by == "change-flag" and st.changed_per_sweep[-1] == 0
    labels2, st2 = run_contour((n, e), make_schedule("c2", atomic=False))
    assert np.array_equal(labels2, exp)
    ctx.close()


def test_device_rmat_generator_matches_host():
    ctx = _lib.Context(0)
    n, m = graphgen.rmat_device(ctx, 12, 16, 9)
    labels = np.empty(n, dtype=np.int64)
    engine.run_staged(ctx, make_schedule("c2"), labels_out=labels)
    _, e = graphgen.rmat(12, 16, 9)
    assert np.array_equal(labels, oracle.rem_union_find(n, e))
    # shard generation: rows [lo, hi)
    lo, hi = 1000, 70000
    graphgen.rmat_device(ctx, 12, 16, 9, row_lo=lo, row_hi=hi)
    labels2 = np.empty(n, dtype=np.int64)
    engine.run_staged(ctx, make_schedule("c2"), labels_out=labels2)
    assert np.array_equal(labels2, oracle.rem_union_find(n, e[lo:hi]))
    ctx.close()


# ---------------------------------------------------------------- edge cases
def test_edge_cases():
    labels, st = run_contour((0, np.zeros((0, 2), np.int64)), make_schedule("c2"))
    assert labels.size == 0 and st.sweeps_until_stable == 0
    labels, st = run_contour((4, []), make_schedule("c2"))
    assert labels.tolist() == [0, 1, 2, 3]
    assert (st.sweeps_executed, st.sweeps_until_stable, st.converged_by) == (1, 0, "change-flag")
    labels, _ = run_contour((3, [(0, 0), (2, 2)]), make_schedule("c2"))
    assert labels.tolist() == [0, 1, 2]
    labels, _ = run_contour((1, [(0, 0)]), make_schedule("cm"))
    assert labels.tolist() == [0]
    with pytest.raises(ValueError):
        run_contour((3, [(0, 3)]), make_schedule("c2"))
    with pytest.raises(ValueError):
        run_contour((3, [(-1, 2)]), make_schedule("c2"))
    with pytest.raises(ValueError):
        run_contour((3, np.zeros((2, 3), np.int64)), make_schedule("c2"))


def test_ragged_tails_and_int32_and_device_inputs():
    import torch
    for m in (1, 2, 3, 4, 5, 7, 9, 31, 33, 1023, 1025):
        n, e = spec.erdos_renyi(200, m, m)
        exp = oracle.rem_union_find(n, e)
        for sched in (make_schedule("c2", atomic=False), make_schedule("c1", sync=True),
                      make_schedule("cm", 5)):
            assert np.array_equal(run_contour((n, e), sched)[0], exp)
            assert np.array_equal(run_contour((n, e.astype(np.int32)), sched)[0], exp)
        t = torch.from_numpy(e).cuda()
        assert np.array_equal(run_contour((n, t), make_schedule("c2"))[0], exp)


def test_iteration_cap_raises():
    ctx = _lib.Context(0)
    engine.stage_graph(ctx, 6, np.array([[5, 4], [4, 3], [3, 2], [2, 1], [1, 0]]))
    with pytest.raises(IterationCapExceeded):
        engine.run_staged(ctx, make_schedule("c1", sync=True), cap=2)
    ctx.close()


def test_long_chain_high_order_buffer_overflow():
    """Permuted paths make chains longer than the 16-cell device buffer."""
    rng = np.random.default_rng(3)
    for d in (100, 5000):
        perm = rng.permutation(d + 1)
        e = np.stack([perm[:-1], perm[1:]], axis=1).astype(np.int64)
        exp = oracle.rem_union_find(d + 1, e)
        for sched in (make_schedule("cm", 1024), make_schedule("c11mm", 64),
                      make_schedule("cm", 1024, sync=True)):
            assert np.array_equal(run_contour((d + 1, e), sched)[0], exp)


def test_sync_c2_log_bound_on_permuted_paths():
    """Acceptance C2 (test_acceptance.py:132-154) on the device path."""
    import math
    rng = np.random.default_rng(20260810)
    for d in (10, 100, 1000, 100_000):
        bound = math.ceil(math.log(d, 1.5)) + 1
        for _ in range(5):
            perm = rng.permutation(d + 1)
            e = np.stack([perm[np.arange(d)], perm[np.arange(1, d + 1)]], axis=1)
            _, st = run_contour((d + 1, e), make_schedule("c2", sync=True))
            assert st.sweeps_until_stable <= bound


def test_increasing_path_c1_sync_is_n_minus_1():
    """Acceptance C3 (test_acceptance.py:157-166)."""
    for n in (5, 50, 500):
        e = np.stack([np.arange(n - 1), np.arange(1, n)], axis=1)
        _, st = run_contour((n, e), make_schedule("c1", sync=True))
        assert st.sweeps_until_stable == n - 1


def _acceptance_suite():
    """Graph families and sizes of the reference's acceptance suite
    (test_acceptance.py:40-64), built here with seeded numpy: paths, cycles,
    stars, full grids, random forests, Erdos-Renyi from sub- to
    super-critical density.  IDs in generation order, as the reference's."""
    import math
    rng = np.random.default_rng(20261020)
    out = []

    def add(name, n, pairs):
        out.append((name, n, np.asarray(pairs, dtype=np.int64).reshape(-1, 2)))

    for n in (1, 2, 3, 4, 5, 8, 13, 21, 34, 64, 128, 333, 1000, 10_000):
        add(f"path{n}", n, np.stack([np.arange(n - 1), np.arange(1, n)], 1))
    for n in (3, 4, 5, 6, 10, 17, 50, 128, 999, 10_000):
        add(f"cycle{n}", n, np.stack([np.arange(n), (np.arange(n) + 1) % n], 1))
    for n in (2, 3, 4, 9, 33, 100, 1001, 10_000):
        add(f"star{n}", n, np.stack([np.zeros(n - 1, np.int64), np.arange(1, n)], 1))
    for r, c in ((1, 1), (1, 5), (2, 2), (3, 3), (4, 5), (7, 6), (10, 10), (25, 40), (100, 100)):
        v = np.arange(r * c).reshape(r, c)
        e = np.concatenate([np.stack([v[:, :-1].ravel(), v[:, 1:].ravel()], 1),
                            np.stack([v[:-1, :].ravel(), v[1:, :].ravel()], 1)])
        add(f"grid{r}x{c}", r * c, e)
    for n in (10, 50, 200, 1000, 10_000):
        for trees in (1, 3, 8):
            for _ in range(2):
                roots = rng.choice(n, size=trees, replace=False)
                rest = np.setdiff1d(np.arange(n), roots)
                rng.shuffle(rest)
                order = np.concatenate([roots, rest])
                par = [(order[i], order[rng.integers(0, i)]) for i in range(trees, n)]
                add(f"forest{n}t{trees}", n, par)
    for n in (10, 100, 1000, 2000):
        for p in (0.5 / n, 1.0 / n, 2.0 / n, math.log(n) / n, 2.0 * math.log(n) / n):
            for _ in range(70 if n <= 100 else 25):
                iu = np.triu_indices(n, 1)
                keep = rng.random(iu[0].size) < min(p, 1.0)
                add(f"er{n}p{p:.4f}", n, np.stack([iu[0][keep], iu[1][keep]], 1))
    return out


def test_acceptance_matrix_c1_c4_c6():
    """Acceptance C1 (labels == rem_union_find), C4 (sync sweeps C-m <= C-2 <=
    C-1) and C6 (every converged run passes the early check and is one star
    per component) over the reference suite's graph families, every variant x
    {sync, async} x {atomic, plain}, on the device path
    (test_acceptance.py:122-129, 169-180, 208-215)."""
    ctx = _lib.Context(0)
    bad, order_bad, runs = [], [], 0
    for name, n, e in _acceptance_suite():
        exp = oracle.rem_union_find(n, e)
        comps = int(np.count_nonzero(exp == np.arange(n)))
        engine.stage_graph(ctx, n, e, "auto")
        sweeps = {}
        for variant, sync in ALL_MODES:
            for atomic in (True, False):
                labels = np.empty(n, dtype=np.int64)
                _, st = engine.run_staged(ctx, make_schedule(variant, 1024, sync=sync,
                                                             atomic=atomic),
                                          count_changes=sync, early_check=True,
                                          labels_out=labels)
                runs += 1
                if not np.array_equal(labels, exp):
                    bad.append((name, variant, sync, atomic, "labels"))
                    continue
                d = engine.forest_diagnostics(labels)
                if not engine.early_convergence_check((n, e), labels) or \
                        d.roots.size != comps or any(h > 1 for h in d.heights.values()):
                    bad.append((name, variant, sync, atomic, "structure"))
                if sync and atomic:
                    sweeps[variant] = st.sweeps_until_stable
        if not (sweeps["C-m"] <= sweeps["C-2"] <= sweeps["C-1"]):
            order_bad.append((name, sweeps))
    ctx.close()
    assert runs == 1021 * 2 * len(ALL_MODES)  # the reference suite's 1,021 graphs
    assert not bad, bad[:10]
    assert not order_bad, order_bad[:10]


def test_race_tolerance_repeated_runs():
    """Acceptance C5 analogue: racy async sweeps always give identical labels
    (20 runs, as test_acceptance.py:183-205 runs 20 seeds)."""
    n, e = graphgen.erdos_renyi(100_000, 400_000, 99)
    exp = oracle.rem_union_find(n, e)
    for _ in range(20):
        labels, _ = run_contour((n, e), make_schedule("c2", atomic=False))
        assert np.array_equal(labels, exp)


# ---------------------------------------------------------------- tuning knobs
def test_store_modes_layouts_and_first_scatter_are_exact():
    n, e = graphgen.rmat(14, 16, 4)
    n2, e2 = graphgen.grid(300, 300, 0.55, 6)
    cases = [(n, e, oracle.rem_union_find(n, e)), (n2, e2, oracle.rem_union_find(n2, e2))]
    ctx = _lib.Context(0)
    ctx.set_option(_lib.CC_OPT_SORT_CHUNK, 5000)  # many chunks on a small graph
    for nn, ee, exp in cases:
        for layout in ("input", "chunk_sorted", "src_sorted"):
            engine.stage_graph(ctx, nn, ee, layout)
            for atomic, modes in ((False, (0, 1, 2, 3)), (True, (1, 3))):
                for sm in modes:
                    ctx.set_option(_lib.CC_OPT_STORE_MODE_ATOMIC if atomic
                                   else _lib.CC_OPT_STORE_MODE_PLAIN, sm)
                    for fs in (False, True):
                        labels = np.empty(nn, dtype=np.int64)
                        _, st = engine.run_staged(ctx, make_schedule("c2", atomic=atomic),
                                                  labels_out=labels, first_scatter=fs)
                        assert np.array_equal(labels, exp), (layout, atomic, sm, fs)
                        check_invariants(labels, st)
    with pytest.raises(ValueError):
        ctx.set_option(_lib.CC_OPT_STORE_MODE_ATOMIC, 0)  # atomic never loses a lowering
    with pytest.raises(ValueError):
        ctx.set_option(99, 1)
    ctx.close()


def test_sweep_ctas_and_item_orders_exact():
    """CTAs per SM of the flat sweep (auto, 1, 3) and every bucketed item
    order (incl. src-major 3) give exact labels; out-of-range values raise."""
    n, e = graphgen.rmat(14, 16, 8)
    exp = oracle.rem_union_find(n, e)
    ctx = _lib.Context(0)
    for ctas in (0, 1, 3):
        ctx.set_option(_lib.CC_OPT_SWEEP_CTAS, ctas)
        for layout in ("chunk_sorted", "l2_tiled"):
            ctx.set_option(_lib.CC_OPT_TILE_SHIFT, 12)
            engine.stage_graph(ctx, n, e, layout)
            for early in (False, True):
                labels = np.empty(n, dtype=np.int64)
                _, st = engine.run_staged(ctx, make_schedule("c2"), count_changes=False,
                                          early_check=early, labels_out=labels)
                assert np.array_equal(labels, exp), (ctas, layout, early)
                check_invariants(labels, st)
    ctx.set_option(_lib.CC_OPT_SWEEP_CTAS, 0)
    ctx.set_option(_lib.CC_OPT_BUCKET_SHIFT, 11)
    ctx.set_option(_lib.CC_OPT_ITEM_ROWS, 4000)
    for order in (0, 1, 2, 3):
        ctx.set_option(_lib.CC_OPT_ITEM_ORDER, order)
        engine.stage_graph(ctx, n, e, "dst_bucketed")
        labels = np.empty(n, dtype=np.int64)
        engine.run_staged(ctx, make_schedule("c2"), labels_out=labels)
        assert np.array_equal(labels, exp), order
    for opt, val in ((_lib.CC_OPT_SWEEP_CTAS, -1), (_lib.CC_OPT_SWEEP_CTAS, 33),
                     (_lib.CC_OPT_ITEM_ORDER, 4)):
        with pytest.raises(ValueError):
            ctx.set_option(opt, val)
    ctx.close()


def test_sync_first_scatter_keeps_reference_stats(golden):
    """The load-free sweep 1 is exactly the reference's sync sweep 1."""
    for g in golden["graphs"][:80]:
        e = np.asarray(g["edges"], dtype=np.int64).reshape(-1, 2)
        exp = g["runs"]["C-2|sync|4"]
        for fs in (False, True):
            labels, st = run_contour((g["n"], e), make_schedule("c2", sync=True),
                                     first_scatter=fs)
            assert labels.tolist() == g["labels"]
            assert (st.sweeps_executed, st.changed_per_sweep) == (exp["executed"], exp["changed"])


@pytest.mark.parametrize("cadence", [1, 2])
def test_sharded_driver_two_shards_on_one_gpu(cadence):
    """The multi-GPU driver's CUDA shards, two ranks emulated as host threads
    on one GPU (no kernel waits on another; the MIN exchange is a host
    barrier + torch.minimum), must give the exact labels."""
    import threading

    import torch

    from paper_2311_02811_b200.distributed import CudaShard, ShardedContour, shard_rows

    n, e = graphgen.rmat(15, 16, 7)
    exp = oracle.rem_union_find(n, e)
    world = 2
    slots = [None] * world
    barrier = threading.Barrier(world)
    results, errors = {}, []

    def allreduce_for(r):
        def ar(t):
            slots[r] = t
            torch.cuda.synchronize()
            barrier.wait()
            if r == 0:
                m = torch.minimum(slots[0], slots[1])
                for x in slots:
                    x.copy_(m)
                torch.cuda.synchronize()
            barrier.wait()
        return ar

    def work(r):
        try:
            torch.cuda.set_device(0)
            ctx = _lib.Context(0)
            lo, hi = shard_rows(e.shape[0], r, world)
            engine.stage_graph(ctx, n, e[lo:hi], "input")
            shard = CudaShard(ctx, n)
            runner = ShardedContour(shard, n, e.shape[0], cadence=cadence,
                                    allreduce=allreduce_for(r))
            runner.run()
            torch.cuda.synchronize()
            results[r] = shard.labels[:n].cpu().numpy().astype(np.int64)
        except Exception as exc:  # pragma: no cover - surfaced below
            errors.append(exc)
            barrier.abort()

    threads = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not errors, errors
    for r in range(world):
        assert np.array_equal(results[r], exp)


def test_graph_loop_matches_host_loop_all_variants(golden):
    """The CUDA-graph convergence loop (device-side WHILE) against the host
    loop and the oracle, for every variant incl. per-sweep order changes."""
    cases = [(g["n"], np.asarray(g["edges"], dtype=np.int64).reshape(-1, 2), g["labels"])
             for g in golden["graphs"][::3]]
    n, e = graphgen.grid(200, 200, 0.55, 8)
    cases.append((n, e, oracle.rem_union_find(n, e).tolist()))
    n, e = graphgen.rmat(13, 16, 8)
    cases.append((n, e, oracle.rem_union_find(n, e).tolist()))
    for n, e, exp in cases:
        for variant in ("C-1", "C-2", "C-m", "C-11mm", "C-1m1m"):
            for atomic in (False, True):
                sched = make_schedule(variant, 8, sync=False, atomic=atomic)
                lg, sg = run_contour((n, e), sched, count_changes=False, early_check=False)
                lh, sh = run_contour((n, e), sched, count_changes=False, early_check=False,
                                     host_loop=True)
                assert lg.tolist() == exp and lh.tolist() == exp, (variant, atomic)
                for st in (sg, sh):
                    check_invariants(lg, st)
                    assert st.converged_by == "change-flag"
                    assert st.changed_per_sweep[-1] == 0
                    assert all(c == -1 for c in st.changed_per_sweep[:-1])


def test_graph_loop_early_check(golden):
    """The early convergence check inside the CUDA-graph loop (engine.py:318-320,
    331-348): exact labels for every variant and layout; a run stopped by the
    check ends on a changing sweep (until_stable == executed), one stopped by
    the flag on a no-write sweep -- the reference's two outcomes."""
    cases = [(g["n"], np.asarray(g["edges"], dtype=np.int64).reshape(-1, 2), g["labels"])
             for g in golden["graphs"][::2]]
    for n, e in (graphgen.grid(180, 210, 0.55, 4), graphgen.rmat(13, 16, 9),
                 graphgen.forest(40, 5), spec.erdos_renyi(4097, 9000, 3)):
        cases.append((n, e, oracle.rem_union_find(n, e).tolist()))
    seen = set()
    for layout in ("input", "chunk_sorted", "dst_bucketed", "hybrid"):
        for n, e, exp in cases:
            for variant in ("C-1", "C-2", "C-m", "C-1m1m"):
                sched = make_schedule(variant, 6, sync=False)
                lg, sg = run_contour((n, e), sched, count_changes=False, early_check=True,
                                     layout=layout)
                assert lg.tolist() == exp, (layout, variant, n)
                check_invariants(lg, sg)
                seen.add(sg.converged_by)
                if sg.converged_by == "early-check":
                    assert sg.sweeps_until_stable == sg.sweeps_executed
                    assert all(c == -1 for c in sg.changed_per_sweep)
                else:
                    assert sg.sweeps_until_stable == sg.sweeps_executed - 1
                    assert sg.changed_per_sweep[-1] == 0
    assert "early-check" in seen


@pytest.mark.parametrize("pipe", [0, 1, 2])
def test_hybrid_layout_exact(pipe):
    """Layout 5: sweep 1 on chunk-sorted rows, later order-2 sweeps and the
    check on the dst-bucketed copy -- graph and host loops, every variant."""
    ctx = _lib.Context(0)
    ctx.set_option(_lib.CC_OPT_BUCKET_PIPE, pipe)
    ctx.set_option(_lib.CC_OPT_BUCKET_SHIFT, 11)
    ctx.set_option(_lib.CC_OPT_ITEM_ROWS, 3001)
    ctx.set_option(_lib.CC_OPT_SORT_CHUNK, 50000)
    for n, e in (graphgen.rmat(15, 16, 2), graphgen.grid(210, 190, 0.55, 5),
                 graphgen.forest(50, 4), spec.erdos_renyi(6001, 15000, 9)):
        exp = oracle.rem_union_find(n, e)
        engine.stage_graph(ctx, n, e, "hybrid")
        for variant in ("C-2", "C-1", "C-m", "C-1m1m"):
            for host_loop, early in ((False, False), (False, True), (True, True)):
                labels = np.empty(n, dtype=np.int64)
                _, st = engine.run_staged(ctx, make_schedule(variant, 5), count_changes=False,
                                          early_check=early, host_loop=host_loop,
                                          labels_out=labels)
                assert np.array_equal(labels, exp), (n, variant, host_loop, early)
                check_invariants(labels, st)
        labels = np.empty(n, dtype=np.int64)
        engine.run_staged(ctx, make_schedule("c2", sync=True), labels_out=labels)
        assert np.array_equal(labels, exp)
    ctx.close()


@pytest.mark.parametrize("transpose", [0, 1])
def test_warp_transposed_layouts_exact(transpose):
    """Sorted layouts with and without the warp-block transposition (and so
    the hybrid copy compact or not by pipe): labels exact, certificate clean,
    on chunk sizes that are and are not multiples of 128 rows."""
    for chunk in (1 << 14, 50000):
        ctx = _lib.Context(0)
        ctx.set_option(_lib.CC_OPT_WARP_TRANSPOSE, transpose)
        ctx.set_option(_lib.CC_OPT_SORT_CHUNK, chunk)
        ctx.set_option(_lib.CC_OPT_BUCKET_SHIFT, 12)
        ctx.set_option(_lib.CC_OPT_ITEM_ROWS, 5000)
        for n, e in (graphgen.rmat(14, 16, 3), graphgen.grid(150, 170, 0.55, 2)):
            exp = oracle.rem_union_find(n, e)
            for layout in ("chunk_sorted", "src_sorted", "dst_bucketed", "hybrid"):
                engine.stage_graph(ctx, n, e, layout)
                for early in (False, True):
                    labels = np.empty(n, dtype=np.int64)
                    _, st = engine.run_staged(ctx, make_schedule("c2"), count_changes=False,
                                              early_check=early, labels_out=labels)
                    assert np.array_equal(labels, exp), (chunk, n, layout, early)
                    check_invariants(labels, st)
                    assert engine.verify_staged(ctx) == 0
        ctx.close()


def test_random_graphs_every_layout_and_loop():
    """Seeded fuzz: random multigraphs (self loops, duplicates, isolated
    vertices, ragged sizes) through every layout, both loops, check on/off,
    small buckets / items / chunks so every kernel path sees many items."""
    import os
    rng = np.random.default_rng(int(os.environ.get("CC_FUZZ_SEED", "20261020")))
    ctx = _lib.Context(0)
    layouts = ("input", "src_sorted", "chunk_sorted", "dst_bucketed", "l2_tiled", "hybrid",
               "l2_tiled_check", "relabel")
    for t in range(int(os.environ.get("CC_FUZZ_ITERS", "120"))):
        n = int(rng.integers(1, 6000))
        m = int(rng.integers(0, 25000))
        e = rng.integers(0, n, size=(m, 2), dtype=np.int64)
        if m and t % 3 == 0:  # chains: long paths stress the propagation order
            perm = rng.permutation(n)
            k = min(m, n - 1)
            e[:k, 0], e[:k, 1] = perm[:k], perm[1:k + 1]
        exp = oracle.rem_union_find(n, e)
        layout = layouts[t % len(layouts)]
        ctx.set_option(_lib.CC_OPT_BUCKET_SHIFT, int(rng.integers(8, 12)))
        ctx.set_option(_lib.CC_OPT_ITEM_ROWS, int(rng.integers(1024, 5000)))
        chunk = int(rng.integers(1, 9000))
        ctx.set_option(_lib.CC_OPT_SORT_CHUNK, chunk if t % 2 else 128 * (chunk // 128 + 1))
        ctx.set_option(_lib.CC_OPT_TILE_SHIFT, 10)
        ctx.set_option(_lib.CC_OPT_CHECK_SHIFT, int(rng.integers(7, 11)))
        ctx.set_option(_lib.CC_OPT_FLAT_BITS, int(rng.integers(0, 3)))
        ctx.set_option(_lib.CC_OPT_ITEM_ORDER, int(t % 4))
        ctx.set_option(_lib.CC_OPT_WARP_TRANSPOSE, int(rng.integers(0, 4) > 0))
        ctx.set_option(_lib.CC_OPT_SWEEP_CTAS, int(rng.integers(0, 4)))
        ctx.set_option(_lib.CC_OPT_BUCKET_PIPE, int(rng.integers(0, 4)))
        engine.stage_graph(ctx, n, e, layout)
        for variant in ("C-2", "C-1", "C-m"):
            for host_loop in (False, True):
                early = bool(rng.integers(0, 2))
                atomic = bool(rng.integers(0, 2))
                labels = np.empty(n, dtype=np.int64)
                _, st = engine.run_staged(ctx, make_schedule(variant, 4, atomic=atomic),
                                          count_changes=False, early_check=early,
                                          host_loop=host_loop, labels_out=labels)
                assert np.array_equal(labels, exp), (t, n, m, layout, variant, host_loop, early)
                check_invariants(labels, st)
        labels = np.empty(n, dtype=np.int64)
        _, st = engine.run_host(ctx, n, e, make_schedule("c2"), count_changes=False,
                                labels_out=labels)
        assert np.array_equal(labels, exp), (t, "run_host")
    ctx.close()


def test_early_convergence_check_api():
    """early_convergence_check(g, labels) (engine.py:331-348) on the device
    through cc_write_labels + cc_early_check, against the oracle restatement."""
    from paper_2311_02811_b200 import early_convergence_check
    rng = np.random.default_rng(11)
    assert early_convergence_check((0, np.zeros((0, 2), np.int64)), np.zeros(0, np.int64))
    assert not early_convergence_check((3, np.zeros((0, 2), np.int64)), np.array([0, 0, 1]))
    assert early_convergence_check((3, np.zeros((0, 2), np.int64)), np.array([0, 1, 2]))
    with pytest.raises(ValueError):
        early_convergence_check((3, [(0, 1)]), np.array([0, 0]))
    with pytest.raises(ValueError):
        early_convergence_check((3, [(0, 1)]), np.array([0, 0, 7]))
    for n, e in (graphgen.rmat(12, 16, 4), graphgen.grid(60, 70, 0.55, 2),
                 spec.erdos_renyi(3000, 4000, 5)):
        done = oracle.rem_union_find(n, e)
        assert early_convergence_check((n, e), done) is True
        for _ in range(6):
            lab = done.copy()
            x = int(rng.integers(0, n))
            lab[x] = x if done[x] != x else lab[x]  # detach one vertex (or keep a root)
            exp = oracle.early_convergence_check(n, e, lab)
            assert early_convergence_check((n, e), lab) is exp
            assert early_convergence_check((n, e), lab.astype(np.int32)) is exp


def test_run_host_streamed_first_sweep(golden):
    """cc_run_host: sweep 1 streamed behind the host-to-device copy, then the
    loop from sweep 2 -- exact labels, consistent stats, errors as staging."""
    cases = [(g["n"], np.asarray(g["edges"], dtype=np.int64).reshape(-1, 2), g["labels"])
             for g in golden["graphs"][::2]]
    for n, e in (graphgen.grid(300, 310, 0.55, 4), graphgen.rmat(15, 16, 9),
                 graphgen.forest(60, 5), spec.erdos_renyi(40001, 90000, 3)):
        cases.append((n, e, oracle.rem_union_find(n, e).tolist()))
    ctx = _lib.Context(0)
    ctx.set_option(_lib.CC_OPT_SORT_CHUNK, 4099)  # many chunks: many streamed pieces
    for layout in ("input", "chunk_sorted"):
        for n, e, exp in cases:
            for variant, atomic, early in (("C-2", True, True), ("C-2", False, False),
                                           ("C-1", True, True), ("C-m", True, False),
                                           ("C-1m1m", True, True)):
                sched = make_schedule(variant, 5, atomic=atomic)
                labels = np.empty(n, dtype=np.int64)
                _, st = engine.run_host(ctx, n, e, sched, layout=layout, count_changes=False,
                                        early_check=early, labels_out=labels)
                assert labels.tolist() == exp, (layout, variant, n)
                check_invariants(labels, st)
                if st.converged_by == "early-check":
                    assert st.sweeps_until_stable == st.sweeps_executed
                else:
                    assert st.sweeps_until_stable == st.sweeps_executed - 1
                assert engine.verify_staged(ctx) == 0
    # a bad endpoint fails the call (the streamed sweep never saw it)
    with pytest.raises(ValueError):
        engine.run_host(ctx, 10, np.array([[0, 1], [2, 10]]), make_schedule("c2"),
                        count_changes=False)
    labels = np.empty(5, dtype=np.int64)
    _, st = engine.run_host(ctx, 5, np.zeros((0, 2), np.int64), make_schedule("c2"),
                            count_changes=False, labels_out=labels)
    assert labels.tolist() == list(range(5)) and st.converged_by == "change-flag"
    ctx.close()


def test_graph_loop_cap_and_rebuild():
    ctx = _lib.Context(0)
    e = np.array([[5, 4], [4, 3], [3, 2], [2, 1], [1, 0]])
    engine.stage_graph(ctx, 6, e)
    with pytest.raises(IterationCapExceeded):
        engine.run_staged(ctx, make_schedule("c1"), count_changes=False, early_check=False,
                          cap=1)
    labels = np.empty(6, dtype=np.int64)
    engine.run_staged(ctx, make_schedule("c1"), count_changes=False, early_check=False,
                      labels_out=labels)
    assert labels.tolist() == [0] * 6
    # restaging a different graph must rebuild the captured loop
    n, e2 = graphgen.rmat(11, 8, 2)
    engine.stage_graph(ctx, n, e2)
    labels = np.empty(n, dtype=np.int64)
    engine.run_staged(ctx, make_schedule("c2"), count_changes=False, early_check=False,
                      labels_out=labels)
    assert np.array_equal(labels, oracle.rem_union_find(n, e2))
    ctx.close()


@pytest.mark.parametrize("bshift,item_rows,threads,pipe,order",
                         [(8, 1024, 256, 0, 0), (12, 5000, 512, 0, 1), (15, 1 << 18, 1024, 0, 0),
                          (8, 1024, 1024, 3, 0), (12, 5001, 1024, 2, 1),
                          (15, 1 << 18, 1024, 3, 0), (15, 9999, 1024, 3, 1),
                          (9, 1027, 1024, 1, 0), (15, 1 << 18, 1024, 1, 1),
                          (14, 7001, 1024, 2, 0), (15, 65536, 1024, 2, 1),
                          (10, 3000, 1024, 1, 2)])
def test_dst_bucketed_layout_exact(bshift, item_rows, threads, pipe, order):
    """Layout 3 + the shared-memory bucketed order-2 sweeps (plain and bulk-copy
    pipelined kernels, bucket- and run-major items), host and graph loops,
    plain and atomic schedules, on RMAT / grid / forest / ragged inputs."""
    graphs = [graphgen.rmat(14, 16, 5), graphgen.grid(150, 170, 0.55, 3),
              graphgen.forest(30, 2), spec.erdos_renyi(3001, 7777, 4)]
    ctx = _lib.Context(0)
    ctx.set_option(_lib.CC_OPT_BUCKET_SHIFT, bshift)
    ctx.set_option(_lib.CC_OPT_ITEM_ROWS, item_rows)
    ctx.set_option(_lib.CC_OPT_BUCKET_THREADS, threads)
    ctx.set_option(_lib.CC_OPT_BUCKET_PIPE, pipe)
    ctx.set_option(_lib.CC_OPT_ITEM_ORDER, order)
    ctx.set_option(_lib.CC_OPT_SORT_CHUNK, 100003)
    for n, e in graphs:
        exp = oracle.rem_union_find(n, e)
        engine.stage_graph(ctx, n, e, "dst_bucketed")
        for sched in (make_schedule("c2"), make_schedule("c2", atomic=False),
                      make_schedule("c1m1m", 8)):
            for host_loop in (False, True):
                labels = np.empty(n, dtype=np.int64)
                _, st = engine.run_staged(ctx, sched, labels_out=labels, count_changes=False,
                                          early_check=False, host_loop=host_loop)
                assert np.array_equal(labels, exp), (n, sched, host_loop)
                check_invariants(labels, st)
        labels = np.empty(n, dtype=np.int64)
        engine.run_staged(ctx, make_schedule("c2", sync=True), labels_out=labels)
        assert np.array_equal(labels, exp)
    ctx.close()


@pytest.mark.parametrize("layout", ["l2_tiled", "l2_tiled_check"])
@pytest.mark.parametrize("tile_shift", [10, 14])
def test_l2_tiled_layout_exact(tile_shift, layout):
    ctx = _lib.Context(0)
    ctx.set_option(_lib.CC_OPT_TILE_SHIFT, tile_shift)
    ctx.set_option(_lib.CC_OPT_CHECK_SHIFT, tile_shift - 2)
    for n, e in (graphgen.rmat(16, 16, 6), graphgen.grid(400, 300, 0.55, 9),
                 graphgen.forest(60, 7), spec.erdos_renyi(5000, 20001, 2)):
        if (n + (1 << tile_shift) - 1) >> tile_shift > 1024:
            continue
        exp = oracle.rem_union_find(n, e)
        engine.stage_graph(ctx, n, e, layout)
        for sched in (make_schedule("c2"), make_schedule("cm", 16), make_schedule("c2", sync=True)):
            for early in (False, True):
                labels = np.empty(n, dtype=np.int64)
                engine.run_staged(ctx, sched, labels_out=labels, count_changes=False,
                                  early_check=early)
                assert np.array_equal(labels, exp), (n, sched, early)
                assert engine.verify_staged(ctx) == 0
    ctx.close()


def test_relabel_layout_exact():
    """Layout 7 (first-appearance relabeling + map back to the minimum
    original ID): exact labels for asynchronous runs on the relabeled rows
    (graph loop and host loop, early check on/off) and for the parity modes
    that run on the original rows (exact counts, synchronous); isolated
    vertices keep their own ID; the device certificate holds on the
    original rows after the map back."""
    rng = np.random.default_rng(77)
    ctx = _lib.Context(0)
    cases = [graphgen.forest(60, 3), graphgen.grid(300, 200, 0.55, 2), graphgen.rmat(14, 16, 9),
             (5, np.zeros((0, 2), np.int64))]
    for _ in range(6):
        n = int(rng.integers(10, 40000))
        m = int(rng.integers(1, 30000))
        cases.append((n, rng.integers(0, n, size=(m, 2), dtype=np.int64)))
    for n, e in cases:
        exp = oracle.rem_union_find(n, e)
        engine.stage_graph(ctx, n, e, "relabel")
        for sched, count in ((make_schedule("c2"), False), (make_schedule("cm", 6), False),
                             (make_schedule("c2", atomic=False), False),
                             (make_schedule("c2"), True), (make_schedule("c2", sync=True), True)):
            for early in (False, True):
                for host_loop in (False, True):
                    labels = np.empty(n, dtype=np.int64)
                    _, st = engine.run_staged(ctx, sched, count_changes=count, early_check=early,
                                              host_loop=host_loop, labels_out=labels)
                    assert np.array_equal(labels, exp), (n, sched, count, early, host_loop)
                    check_invariants(labels, st)
                    assert engine.verify_staged(ctx) == 0
    ctx.close()


@pytest.mark.parametrize("check_shift,pack", [(16, 1), (17, 1), (17, 0), (16, 2), (17, 2),
                                              (18, 2)])
def test_packed_check_copy_exact(check_shift, pack):
    """The packed check copies against the oracle: 6-byte rows (src | high
    offset bits, uint16 low bits; pack 1) and delta-packed groups of 128 rows
    (pack 2, the default: 32 - check_shift bits per source gap; the sparse
    forest's gaps overflow them and the build falls back to 6-byte rows) --
    the bitmap check's verdicts and whole runs through the bitmap sweep."""
    rng = np.random.default_rng(17)
    ctx = _lib.Context(0)
    ctx.set_option(_lib.CC_OPT_TILE_SHIFT, 18)
    ctx.set_option(_lib.CC_OPT_CHECK_SHIFT, check_shift)
    ctx.set_option(_lib.CC_OPT_CHECK_PACK, pack)
    ctx.set_option(_lib.CC_OPT_ITEM_ROWS, 50000)
    for n, e in (graphgen.rmat(19, 16, 2), graphgen.grid(700, 900, 0.55, 5),
                 graphgen.forest(300, 3)):
        exp = oracle.rem_union_find(n, e)
        engine.stage_graph(ctx, n, e, "l2_tiled_check")
        for count in (False, True):
            labels = np.empty(n, dtype=np.int64)
            _, st = engine.run_staged(ctx, make_schedule("c2"), count_changes=count,
                                      labels_out=labels)
            assert np.array_equal(labels, exp), (n, count)
            check_invariants(labels, st)
        for _ in range(4):
            lab = exp.copy()
            x = int(rng.integers(1, n))
            lab[x] = int(rng.integers(0, x))
            _lib.check(ctx.lib.cc_write_labels(ctx.handle, lab.ctypes.data, 8))
            assert engine.loop_check(ctx) == oracle.early_convergence_check(n, e, lab)
        _lib.check(ctx.lib.cc_write_labels(ctx.handle, exp.ctypes.data, 8))
        assert engine.loop_check(ctx)
    ctx.close()


@pytest.mark.parametrize("split,rebuild,canon,publish",
                         [(1, 0, 1, 0), (3, 1, 1, 0), (5, 2, 1, 0), (-1, -1, 1, 0), (7, 3, 1, 0),
                          (0, 0, 1, 0), (-1, -1, 0, 0), (3, 1, 0, 0), (-1, -1, 2, 0), (5, 2, 2, 0),
                          (-1, -1, 1, 1), (3, 1, 1, 2), (1, 0, 2, 2), (5, 2, 0, 1), (-1, -1, 1, 2)])
def test_split_sweep1_exact(split, rebuild, canon, publish):
    """Sweep 1 on layout 6 split at an L2 window (CC_OPT_SPLIT_SWEEP): the
    first windows on the tiles, the rest as bitmap sweeps over the check copy
    with the bitmap rebuilt every `rebuild` windows -- labels equal the oracle's
    for async / counted / host-loop / graph-loop runs and C-m, on RMAT (dense,
    where auto splits) and a grid (sparse), 8-10 windows of 2^16 vertices.
    canon (CC_OPT_CANON_SWEEP): the whole-graph bitmap sweeps (1, the
    default) or also the split parts (2) walk the canonical copy (each
    undirected pair once; built for the symmetrised RMAT graphs), or every
    bitmap sweep walks the dst-bucketed check copy (0).
    publish (CC_OPT_BITS_PUBLISH): the bitmap sweeps of the split parts (1) or
    all of them (2) set a vertex's bit when a row leaves it at the root label."""
    ctx = _lib.Context(0)
    ctx.set_option(_lib.CC_OPT_CANON_SWEEP, canon)
    ctx.set_option(_lib.CC_OPT_BITS_PUBLISH, publish)
    ctx.set_option(_lib.CC_OPT_TILE_SHIFT, 16)
    ctx.set_option(_lib.CC_OPT_CHECK_SHIFT, 16)
    ctx.set_option(_lib.CC_OPT_ITEM_ROWS, 20000)
    ctx.set_option(_lib.CC_OPT_SPLIT_SWEEP, split)
    ctx.set_option(_lib.CC_OPT_SPLIT_REBUILD, rebuild)
    for n, e in (graphgen.rmat(19, 16, 2), graphgen.rmat(19, 16, 7),
                 graphgen.grid(700, 900, 0.55, 5)):
        exp = oracle.rem_union_find(n, e)
        engine.stage_graph(ctx, n, e, "l2_tiled_check")
        assert ctx.layout_info()["check_format"] == 2
        for sched in (make_schedule("c2"), make_schedule("cm", 6), make_schedule("c2", sync=True)):
            for count in (False, True):
                for host_loop in (False, True):
                    labels = np.empty(n, dtype=np.int64)
                    _, st = engine.run_staged(ctx, sched, count_changes=count,
                                              host_loop=host_loop, labels_out=labels)
                    assert np.array_equal(labels, exp), (n, sched, count, host_loop)
                    check_invariants(labels, st)
        assert engine.verify_staged(ctx) == 0
    ctx.close()


@pytest.mark.parametrize("split,canon,publish,defer", [(-1, -1, 1, 0), (1, 2, 1, 0), (0, 0, 0, 0),
                                                       (3, 1, 2, 0), (1, 1, 0, 0), (-1, -1, 1, 1),
                                                       (2, 0, 2, 1), (5, 2, 1, 1)])
def test_uniting_check_exact(split, canon, publish, defer):
    """CC_OPT_CHECK_UNITE: the early check after sweep 1 unites the trees of
    every row whose labels differ (root hooking) and pointer jumping finishes
    the labels, so an asynchronous C-2 run without exact counts always ends
    after one sweep -- with labels equal to the oracle's (rem_union_find:
    the minimum vertex of every component) on dense graphs (RMAT, where little
    is left to unite), and on graphs one order-2 sweep leaves far from
    converged: a grid, a forest of long paths, one permuted path of 300k
    vertices (deep chains: many hooks, several compress passes), symmetrised
    (canonical copy) or not.  Graph loop and host loop; synchronous and
    counted runs keep the plain check and stay exact too."""
    rng = np.random.default_rng(5)
    ctx = _lib.Context(0)
    ctx.set_option(_lib.CC_OPT_CHECK_UNITE, 1)
    ctx.set_option(_lib.CC_OPT_CANON_SWEEP, canon)
    ctx.set_option(_lib.CC_OPT_BITS_PUBLISH, publish)
    ctx.set_option(_lib.CC_OPT_BITS_DEFER, defer)  # undecided rows parked per lane, run in batches
    ctx.set_option(_lib.CC_OPT_TILE_SHIFT, 16)
    ctx.set_option(_lib.CC_OPT_CHECK_SHIFT, 16)
    ctx.set_option(_lib.CC_OPT_ITEM_ROWS, 20000)
    ctx.set_option(_lib.CC_OPT_SPLIT_SWEEP, split)
    npath = 300_000
    perm = rng.permutation(npath)
    path = np.stack([perm[:-1], perm[1:]], 1).astype(np.int64)
    sym = lambda e: np.concatenate([e, e[:, ::-1]])
    # a forest of 400 paths over 60k permuted IDs (+ isolated vertices), small
    # enough that every 128-row group's source span fits the delta packing
    fn = 65_000
    fperm = rng.permutation(fn)[:60_000]
    cuts = np.sort(rng.choice(np.arange(1, 60_000), 399, replace=False))
    keep = np.ones(59_999, dtype=bool)
    keep[cuts - 1] = False
    fe = np.stack([fperm[:-1], fperm[1:]], 1)[keep].astype(np.int64)
    graphs = [graphgen.rmat(19, 16, 2), graphgen.rmat(18, 4, 9),
              graphgen.grid(700, 900, 0.55, 5), (npath, path), (npath, sym(path)),
              (fn, fe), (fn, sym(fe))]
    for n, e in graphs:
        exp = oracle.rem_union_find(n, e)
        engine.stage_graph(ctx, n, e, "l2_tiled_check")
        assert ctx.layout_info()["check_format"] == 2, (n, ctx.layout_info())
        for host_loop in (False, True):
            for _ in range(2):
                labels = np.empty(n, dtype=np.int64)
                _, st = engine.run_staged(ctx, make_schedule("c2"), count_changes=False,
                                          early_check=True, host_loop=host_loop,
                                          labels_out=labels)
                assert np.array_equal(labels, exp), (n, host_loop)
                assert st.sweeps_executed == 1 and st.converged_by == "early-check"
                assert engine.verify_staged(ctx) == 0
        for sched, count in ((make_schedule("c2", sync=True), True), (make_schedule("c2"), True),
                             (make_schedule("cm", 6), False)):
            labels = np.empty(n, dtype=np.int64)
            _, st = engine.run_staged(ctx, sched, count_changes=count, labels_out=labels)
            assert np.array_equal(labels, exp), (n, sched, count)
            check_invariants(labels, st)
    ctx.close()


def test_uniting_check_fuzz():
    """The bench's default path (layout 6, asynchronous C-2 without exact
    counts, uniting early check, publishing bitmap parts with per-lane
    batches) on 150 random multigraphs -- self loops, repeated rows, one
    orientation or symmetrised, 0 to 8 rows per vertex: 120 small ones (1 to
    40k vertices: one L2 window, sweep 1 on the tiles, then the uniting check)
    and 30 of 2^18 to 600k vertices (4-10 windows of 2^16 vertices: split sweep
    1, several items per bucket): labels equal rem_union_find's, cc_verify
    certifies them, and a run that ended on the uniting check took one sweep."""
    rng = np.random.default_rng(int(os.environ.get("CC_FUZZ_SEED", "77")))
    ctx = _lib.Context(0)
    ctx.set_option(_lib.CC_OPT_TILE_SHIFT, 16)
    ctx.set_option(_lib.CC_OPT_CHECK_SHIFT, 16)
    ctx.set_option(_lib.CC_OPT_ITEM_ROWS, 4096)
    united = 0
    for it in range(150):
        if it < 120:
            n = int(rng.choice([1, 2, 3, 31, 32, 33, 127, 128, 129, 1000, 4097, 40_000]))
            if it % 3 == 0:
                n = int(rng.integers(1, 40_000))
        else:
            n = int(rng.integers(1 << 18, 600_000))
        m = int(rng.integers(0, 8 * n + 1)) if it % 7 else 0
        if it >= 120:
            m = int(rng.integers(n // 2, 4 * n))
        e = rng.integers(0, n, size=(m, 2)).astype(np.int64)
        if it % 2 and m:
            e = np.concatenate([e, e[:, ::-1]])
        if it % 5 == 0 and m:
            e = np.concatenate([e, e[: m // 3]])  # repeated rows
        exp = oracle.rem_union_find(n, e)
        engine.stage_graph(ctx, n, e, "l2_tiled_check")
        for host_loop in (False, True):
            labels = np.empty(n, dtype=np.int64)
            _, st = engine.run_staged(ctx, make_schedule("c2"), count_changes=False,
                                      early_check=True, host_loop=host_loop, labels_out=labels)
            assert np.array_equal(labels, exp), (it, n, m, host_loop)
            assert engine.verify_staged(ctx) == 0, (it, n, m)
            if ctx.layout_info()["uniting_check"]:
                united += 1
                assert st.sweeps_executed <= 1, (it, n, m, st)
    assert united > 150  # (most graphs get the delta-packed copy the uniting check needs)
    ctx.close()


@pytest.mark.parametrize("canon,span_bits,group_windows", [(1, 0, 0), (1, 7, 3), (1, 0, 1),
                                                          (0, 0, 0)])
def test_canonical_check_copy(canon, span_bits, group_windows):
    """The early check over the canonical copy (each undirected pair once,
    CC_OPT_CANON_CHECK) decides exactly as early_convergence_check
    (engine.py:331-348) on converged labels and single-cell perturbations,
    and whole runs (graph loop, where the check is then not folded into a
    bitmap sweep, and host loop) stay exact.  A symmetrised RMAT graph gets
    the copy (< 55 % of the rows); a one-orientation grid does not."""
    rng = np.random.default_rng(11)
    ctx = _lib.Context(0)
    ctx.set_option(_lib.CC_OPT_TILE_SHIFT, 16)
    ctx.set_option(_lib.CC_OPT_CHECK_SHIFT, 16)
    ctx.set_option(_lib.CC_OPT_CANON_CHECK, canon)
    ctx.set_option(_lib.CC_OPT_CANON_SPAN_BITS, span_bits)  # 7: most groups raw (side table)
    ctx.set_option(_lib.CC_OPT_CANON_GROUP_WINDOWS, group_windows)  # several build groups
    for n, e, sym in ((*graphgen.rmat(19, 16, 3), True), (*graphgen.grid(700, 900, 0.55, 5), False)):
        exp = oracle.rem_union_find(n, e)
        engine.stage_graph(ctx, n, e, "l2_tiled_check")
        info = ctx.layout_info()
        if canon and sym:
            assert 0 < info["canon_rows"] < 0.55 * e.shape[0]
            canon_pairs = np.unique(np.stack([e.min(axis=1), e.max(axis=1)], 1)[e[:, 0] != e[:, 1]],
                                    axis=0)
            assert info["canon_rows"] == canon_pairs.shape[0]
            assert (info["canon_side_groups"] > 0) == (span_bits > 0)
        else:
            assert info["canon_rows"] == 0
        for host_loop in (False, True):
            for count in (False, True):
                labels = np.empty(n, dtype=np.int64)
                _, st = engine.run_staged(ctx, make_schedule("c2"), count_changes=count,
                                          host_loop=host_loop, labels_out=labels)
                assert np.array_equal(labels, exp), (n, host_loop, count)
                check_invariants(labels, st)
        for _ in range(6):
            lab = exp.copy()
            x = int(rng.integers(1, n))
            lab[x] = int(rng.integers(0, x))
            _lib.check(ctx.lib.cc_write_labels(ctx.handle, lab.ctypes.data, 8))
            assert engine.loop_check(ctx) == oracle.early_convergence_check(n, e, lab)
        _lib.check(ctx.lib.cc_write_labels(ctx.handle, exp.ctypes.data, 8))
        assert engine.loop_check(ctx)
    ctx.close()


@pytest.mark.parametrize("check_shift", [7, 9, 12])
def test_bitmap_check_equals_oracle_early_check(check_shift):
    """The layout-6 early check (component bitmap + check copy) decides
    exactly as early_convergence_check (engine.py:331-348) -- on converged
    labels, on labels after a partial run, and on single-cell perturbations
    inside and outside the giant component's class."""
    rng = np.random.default_rng(7)
    ctx = _lib.Context(0)
    ctx.set_option(_lib.CC_OPT_TILE_SHIFT, 12)
    ctx.set_option(_lib.CC_OPT_CHECK_SHIFT, check_shift)
    ctx.set_option(_lib.CC_OPT_ITEM_ROWS, 3000)
    for n, e in (graphgen.rmat(15, 16, 3), graphgen.grid(300, 200, 0.55, 4),
                 graphgen.forest(40, 5), spec.erdos_renyi(9000, 40000, 6)):
        exp = oracle.rem_union_find(n, e)
        engine.stage_graph(ctx, n, e, "l2_tiled_check")  # (for the partial-run labels below)
        cases = [exp.copy()]
        for _ in range(6):  # one cell moved to another valid value (<= itself)
            lab = exp.copy()
            x = int(rng.integers(1, n))
            lab[x] = int(rng.integers(0, x))
            cases.append(lab)
        _lib.check(ctx.lib.cc_init_labels(ctx.handle))  # labels after one C-1 sweep
        _lib.check(ctx.lib.cc_sweep(ctx.handle, 1, 0, 1, 0, None))
        part = np.empty(n, dtype=np.int64)
        _lib.check(ctx.lib.cc_read_labels(ctx.handle, part.ctypes.data, 8))
        cases.append(part)
        lab = np.arange(n, dtype=np.int64)  # identity: every non-loop edge disagrees
        cases.append(lab)
        for layout in ("l2_tiled_check", "chunk_sorted"):  # check copy / flat bitmap check
            ctx.set_option(_lib.CC_OPT_FLAT_BITS, 1)
            engine.stage_graph(ctx, n, e, layout)
            for lab in cases:
                lab = np.ascontiguousarray(lab, dtype=np.int64)
                _lib.check(ctx.lib.cc_write_labels(ctx.handle, lab.ctypes.data, 8))
                want = oracle.early_convergence_check(n, e, lab)
                assert engine.loop_check(ctx) == want, (n, check_shift, layout)
            # whole runs through the bitmap check / bitmap sweeps (graph loop and
            # counted host loop), incl. the streamed one-shot path below
            for count in (False, True):
                for early in (False, True):
                    labels = np.empty(n, dtype=np.int64)
                    _, st = engine.run_staged(ctx, make_schedule("c2"), count_changes=count,
                                              early_check=early, labels_out=labels)
                    assert np.array_equal(labels, exp), (n, layout, count, early)
                    check_invariants(labels, st)
        for count in (False, True):
            labels = np.empty(n, dtype=np.int64)
            _, st = engine.run_host(ctx, n, e, make_schedule("c2"), layout="chunk_sorted",
                                    count_changes=count, labels_out=labels)
            assert np.array_equal(labels, exp), (n, "run_host", count)
            check_invariants(labels, st)
        ctx.set_option(_lib.CC_OPT_FLAT_BITS, 2)
    ctx.close()


def test_verify_detects_bad_labels():
    ctx = _lib.Context(0)
    engine.stage_graph(ctx, 4, np.array([[0, 1], [2, 3]]))
    engine.run_staged(ctx, make_schedule("c2"))
    assert engine.verify_staged(ctx) == 0
    _lib.check(ctx.lib.cc_init_labels(ctx.handle))  # identity labels: edges disagree
    assert engine.verify_staged(ctx) & 1
    ctx.close()


def test_fastsv_matches_reference_stats(golden):
    """GPU FastSV (baselines.py:81-131): exact labels and the reference's
    per-iteration counts (atomic-min hooking is order-independent)."""
    from paper_2311_02811_b200.baselines import fastsv
    for g in golden["graphs"]:
        e = np.asarray(g["edges"], dtype=np.int64).reshape(-1, 2)
        labels, st = fastsv((g["n"], e))
        exp = g["fastsv"]
        assert labels.tolist() == g["labels"], g["name"]
        assert (st.sweeps_executed, st.sweeps_until_stable, st.changed_per_sweep) == \
            (exp["executed"], exp["until_stable"], exp["changed"]), g["name"]
        assert st.converged_by == exp["converged_by"] == "grandparent-stable"
    for c in golden["configs"]:
        n, e = _config_edges(c["params"])
        labels, st = fastsv((n, e))
        assert sha(labels) == c["labels_sha256"], c["name"]
        assert (st.sweeps_executed, st.changed_per_sweep) == \
            (c["fastsv"]["executed"], c["fastsv"]["changed"]), c["name"]


def test_staged_chunk_sort_from_host_matches_device_reorder():
    n, e = graphgen.rmat(16, 16, 2, elem_bytes=4)
    exp = oracle.rem_union_find(n, e)
    for layout in ("chunk_sorted", "src_sorted", "auto"):
        labels, st = run_contour((n, e), make_schedule("c2"), layout=layout)
        assert np.array_equal(labels, exp), layout


@pytest.mark.parametrize("cadence", [1, 2])
def test_run_contour_devices_in_process(cadence):
    """run_contour(..., devices=[...]): the edge-sharded driver in one process
    (shards as host threads; here all on cuda:0, which exercises the same
    exchange logic as distinct GPUs) -- exact labels, async variants."""
    for n, e in (graphgen.rmat(15, 16, 5), graphgen.grid(200, 230, 0.55, 3),
                 graphgen.forest(60, 2), (5, np.zeros((0, 2), np.int64))):
        exp = oracle.rem_union_find(n, e)
        for devs in ([0, 0], [0, 0, 0]):
            for variant in ("C-2", "C-1", "C-m"):
                labels, st = run_contour((n, e), make_schedule(variant, 6), devices=devs,
                                         cadence=cadence)
                assert np.array_equal(labels, exp), (n, devs, variant)
                assert st.sweeps_executed == st.sweeps_until_stable + cadence
                assert st.changed_per_sweep[-1] == 0
    # synchronous schedules shard deterministically: stats equal one device's
    for n, e in (graphgen.rmat(14, 16, 5), graphgen.grid(150, 170, 0.55, 3)):
        for variant in ("C-2", "C-Syn", "C-1", "C-m"):
            sched = make_schedule(variant, 6, sync=True)
            lab1, st1 = run_contour((n, e), sched)
            for devs in ([0, 0], [0, 0, 0]):
                labels, st = run_contour((n, e), sched, devices=devs)
                assert np.array_equal(labels, lab1), (devs, variant)
                assert (st.sweeps_executed, st.sweeps_until_stable, st.changed_per_sweep,
                        st.converged_by) == (st1.sweeps_executed, st1.sweeps_until_stable,
                                             st1.changed_per_sweep, st1.converged_by)


def _gpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.skipif("_gpus() < 2")
def test_two_distinct_gpus_in_process_and_bench():
    """run_contour(devices=[0, 1]) on two real GPUs (the per-device smem
    opt-in / occupancy caches, peer copies of the exchange) and the bench's
    2-rank launch; skipped on a one-GPU box."""
    import json
    import subprocess
    import sys
    n, e = graphgen.rmat(18, 16, 2)
    exp = oracle.rem_union_find(n, e)
    for sched in (make_schedule("c2"), make_schedule("c2", sync=True)):
        labels, st = run_contour((n, e), sched, devices=[0, 1])
        assert np.array_equal(labels, exp)
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "rmat22",
                          "--steps", "2", "--warmup", "1", "--no-cpu-baseline", "--no-e2e"],
                         capture_output=True, text=True, timeout=900, check=True).stdout
    line = json.loads([x for x in out.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["verified"]


def test_bench_two_ranks_share_one_gpu():
    """bench.py --gpus 2 without torchrun starts 2 ranks itself (here sharing
    cuda:0 -- the plumbing check: gloo for the host exchange) and rank 0
    prints one line with n_gpus = 2 and verified labels."""
    import json
    import subprocess
    import sys
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "rmat22",
                          "--steps", "2", "--warmup", "1", "--no-cpu-baseline"],
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["verified"] and line["e2e"]["value"] > 0


def test_pinned_and_pageable_host_buffers():
    """Host edges and labels in pinned (cudaHostAlloc, via torch) and pageable
    (numpy) memory, int32 and int64: the copy engine reads pinned buffers
    directly, pageable ones go through the context's narrowing threads and
    pinned staging -- same labels, same range errors, both read-back paths
    (speculative after sweep 1, and after later sweeps)."""
    import torch
    for n, e in (graphgen.rmat(16, 16, 2), graphgen.grid(300, 280, 0.55, 4),
                 graphgen.forest(80, 3)):
        exp = oracle.rem_union_find(n, e)
        for dt in (np.int32, np.int64):
            pageable = np.ascontiguousarray(e, dtype=dt)
            pinned_t = torch.empty(e.shape, dtype=torch.int32 if dt == np.int32 else torch.int64,
                                   pin_memory=True)
            pinned_t.numpy()[:] = pageable
            for src in (pageable, pinned_t.numpy()):
                for out_pinned in (False, True):
                    if out_pinned:
                        lt = torch.empty(n, dtype=torch.int64, pin_memory=True)
                        labels = lt.numpy()
                    else:
                        labels = np.empty(n, dtype=np.int64)
                    ctx = engine._context(0)
                    for early in (False, True):
                        _, st = engine.run_host(ctx, n, src, make_schedule("c2"),
                                                count_changes=False, early_check=early,
                                                labels_out=labels)
                        assert np.array_equal(labels, exp), (n, dt, early, out_pinned)
                    got, _ = run_contour((n, src), make_schedule("c2"))
                    assert np.array_equal(got, exp)
                    l32 = np.empty(n, dtype=np.int32)
                    engine.run_host(ctx, n, src, make_schedule("c1"), count_changes=False,
                                    labels_out=l32)
                    assert np.array_equal(l32, exp)
    bad = np.array([[0, 1], [2, 5]], dtype=np.int64)
    for arr in (bad, np.array([[0, -1]], dtype=np.int64), np.array([[0, 1 << 33]], np.int64),
                np.array([[0, -3]], dtype=np.int32)):
        with pytest.raises(ValueError):
            run_contour((4, arr), make_schedule("c2"))


def test_pageable_narrowing_range_checks_in_the_vector_body():
    """Pageable host edges are narrowed by the context's threads (AVX-512 when
    the host has it): out-of-range endpoints anywhere in a large array -- not
    only in the scalar head/tail -- still raise ValueError, valid ones stage
    exactly (int64 and int32)."""
    n, e = graphgen.rmat(16, 16, 4)
    exp = oracle.rem_union_find(n, e)
    for dt in (np.int64, np.int32):
        a = np.ascontiguousarray(e, dtype=dt)
        labels, _ = run_contour((n, a), make_schedule("c2"))
        assert np.array_equal(labels, exp), dt
        for pos, val in ((123457, -1), (777777, n), (1000003, -(1 << 30))):
            b = a.copy()
            b.flat[pos] = val
            with pytest.raises(ValueError):
                run_contour((n, b), make_schedule("c2"))
    b = np.ascontiguousarray(e, dtype=np.int64)
    b.flat[555555] = 1 << 33  # beyond uint32: must not wrap to a valid ID
    with pytest.raises(ValueError):
        run_contour((n, b), make_schedule("c2"))


@pytest.mark.parametrize("n", [1, 2, 97, 1 << 16, (1 << 24) - 5, (1 << 24) + 3, (1 << 28) - 1])
def test_pageable_link_packing(n):
    """Pageable host edges cross PCIe as ceil(2 log2(n) / 8)-byte packed rows
    (6 B up to n = 2^24, 7 B up to 2^28, else uint32 pairs): staged rows read
    back equal to the input, labels equal the oracle's with packing on and
    off, and IDs outside [0, n) -- in [n, 2^b) (device check) or beyond 2^b /
    negative (host check) -- raise ValueError, int64 and int32."""
    rng = np.random.default_rng(n)
    m = 200_003
    e = rng.integers(0, n, size=(m, 2), dtype=np.int64)
    e[:: 7, 1] = e[:: 7, 0]  # self loops
    exp = oracle.rem_union_find(n, e)
    ctx = engine._context(0)
    b = max(1, (n - 1).bit_length())
    for pack in (1, 0):
        ctx.set_option(_lib.CC_OPT_LINK_PACK, pack)
        try:
            for dt in (np.int64, np.int32):
                a = np.ascontiguousarray(e, dtype=dt)
                engine.stage_graph(ctx, n, a, "input")
                back = np.empty((m, 2), dtype=np.int64)
                _lib.check(ctx.lib.cc_read_edges(ctx.handle, back.ctypes.data, 8, 0, m))
                assert np.array_equal(back, e), (pack, dt)
                labels, _ = run_contour((n, a), make_schedule("c2"))
                assert np.array_equal(labels, exp), (pack, dt)
                bad_vals = [n, -1, (1 << b) + 1, -(1 << 30)]
                if dt == np.int64:
                    bad_vals.append(1 << 40)
                for pos, val in zip((5, 100_001, 2 * m - 1, 77_777, 150_000), bad_vals):
                    x = a.copy()
                    x.flat[pos] = val
                    with pytest.raises(ValueError):
                        run_contour((n, x), make_schedule("c2"))
        finally:
            ctx.set_option(_lib.CC_OPT_LINK_PACK, 1)


def test_frozen_edges_upgrade_to_the_tiles(monkeypatch):
    """A read-only edge array whose labels exceed the L2 budget (forced small
    here) is staged chunk-sorted by the first run_contour call (sweep 1
    streamed behind the copy) and upgraded in place to the resident layout 6
    (tiles, check copies, split sweep 1) by the second; every call exact."""
    monkeypatch.setattr(engine, "AUTO_L2_LABEL_BYTES", 1 << 20)
    n, e = graphgen.rmat(19, 16, 8)
    e = np.ascontiguousarray(e)
    exp = oracle.rem_union_find(n, e)
    e.flags.writeable = False
    ctx = engine._context(0)
    ctx.set_option(_lib.CC_OPT_TILE_SHIFT, 16)
    ctx.set_option(_lib.CC_OPT_CHECK_SHIFT, 16)
    try:
        layouts = []
        for i in range(3):
            labels, st = run_contour((n, e), make_schedule("c2"))
            assert np.array_equal(labels, exp), i
            check_invariants(labels, st)
            layouts.append(ctx.layout_info()["layout"])
        assert layouts[0] in (0, 2) and layouts[1:] == [6, 6], layouts  # (0: input order + chunk sorts)
    finally:
        ctx.set_option(_lib.CC_OPT_TILE_SHIFT, 24)
        ctx.set_option(_lib.CC_OPT_CHECK_SHIFT, 20)
        ctx.staged = None


def test_frozen_edges_stay_resident():
    """run_contour on a read-only edge array (the reference's Graph freezes
    its arrays) reuses the graph staged by the previous call on the context,
    upgraded to the resident layout; any other staging on the context, a
    different array object or a writeable array restages."""
    from paper_2311_02811_b200 import early_convergence_check
    n, e = graphgen.rmat(16, 16, 6)
    e = np.ascontiguousarray(e)
    exp = oracle.rem_union_find(n, e)
    e.flags.writeable = False
    ctx = engine._context(0)
    for i in range(4):
        labels, st = run_contour((n, e), make_schedule("c2"))
        assert np.array_equal(labels, exp), i
        check_invariants(labels, st)
        assert ctx.staged is not None and ctx.staged[0]() is e
    labels, st = run_contour((n, e), make_schedule("c2", sync=True))  # any schedule
    assert np.array_equal(labels, exp)
    n2, e2 = graphgen.grid(120, 130, 0.55, 1)
    e2 = np.ascontiguousarray(e2)
    e2.flags.writeable = False
    assert np.array_equal(run_contour((n2, e2), make_schedule("c2"))[0],
                          oracle.rem_union_find(n2, e2))
    assert ctx.staged[0]() is e2
    assert early_convergence_check((n2, e2), oracle.rem_union_find(n2, e2))
    assert ctx.staged is None  # the check staged its own copy
    assert np.array_equal(run_contour((n, e), make_schedule("c2"))[0], exp)
    w = np.array(e)  # writeable copy: never cached
    assert np.array_equal(run_contour((n, w), make_schedule("cm"))[0], exp)
    assert ctx.staged is None
    base = np.array(e)  # a read-only VIEW of a writeable base can still change: never cached
    v = base[:]
    v.flags.writeable = False
    assert np.array_equal(run_contour((n, v), make_schedule("c2"))[0], exp)
    assert ctx.staged is None
    import gc
    e3 = np.array(e)
    e3.flags.writeable = False
    assert np.array_equal(run_contour((n, e3), make_schedule("c2"))[0], exp)
    del e3
    gc.collect()
    assert ctx.staged[0]() is None  # the cache holds no reference to a dropped array


def test_cuda_tensor_edges_fresh_from_another_stream():
    """Edges produced on the device by torch right before the call (on torch's
    current stream, which the library's own stream does not follow) are
    staged only after that work is done."""
    import torch
    n = 1 << 20
    for i in range(3):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            e = torch.randint(0, n, (1 << 22, 2), device="cuda", dtype=torch.int64)
            e[:, 1] = (e[:, 0] * 7 + 3) % n  # more work queued behind the draw
            labels, st = run_contour((n, e), make_schedule("c2"))
        exp = oracle.rem_union_find(n, e.cpu().numpy())
        assert np.array_equal(labels, exp), i


def test_concurrent_callers_reentrant():
    """Reentrancy (the reference's SPEC.md:212: independent runs on shared
    immutable graphs from several threads): every caller thread gets its own
    context; concurrent run_contour calls on a shared frozen graph and on
    private graphs all return exact labels."""
    import threading
    n, e = graphgen.rmat(14, 16, 11)
    e = np.ascontiguousarray(e)
    e.flags.writeable = False
    exp = oracle.rem_union_find(n, e)
    privates = [graphgen.grid(100 + 10 * i, 90, 0.55, i) for i in range(4)]
    pexp = [oracle.rem_union_find(pn, pe) for pn, pe in privates]
    errors = []

    def work(i):
        try:
            for it in range(5):
                labels, st = run_contour((n, e), make_schedule("c2" if it % 2 else "cm"))
                assert np.array_equal(labels, exp), (i, it)
                pn, pe = privates[i]
                labels, st = run_contour((pn, pe), make_schedule("c2", sync=bool(it % 2)))
                assert np.array_equal(labels, pexp[i]), (i, it)
        except Exception as exc:  # pragma: no cover - reported below
            errors.append(exc)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors[:3]
