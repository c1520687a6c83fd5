"""Pin the CPU oracle (oracle/) against fixtures made by running the
reference itself (tests/golden/make_golden.py).  CPU only."""

import hashlib

import numpy as np
import pytest

from oracle import gen, oracle


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def test_mm_order_known_answers(golden):
    # test_engine.py:53-75 states are the first three cases
    first = golden["mm_order"][:3]
    assert first[0]["target"] == [0, 1, 1, 3]
    assert first[1]["target"] == [0, 0, 0, 0]
    assert first[2]["changed"] is False
    for case in golden["mm_order"]:
        tgt = list(case["labels"])
        ch = oracle.mm_step(tgt, list(case["labels"]), case["w"], case["v"], case["order"])
        assert tgt == case["target"] and ch == case["changed"]
        inplace = list(case["labels"])
        ch2 = oracle.mm_step(inplace, inplace, case["w"], case["v"], case["order"])
        assert inplace == case["inplace"] and ch2 == case["inplace_changed"]


def test_mm_order_rejects_order_zero():
    with pytest.raises(ValueError):
        oracle.mm_step([0, 1], [0, 1], 0, 1, 0)


def test_union_find_matches_reference(golden):
    for g in golden["graphs"]:
        e = np.asarray(g["edges"], dtype=np.int64).reshape(-1, 2)
        assert oracle.rem_union_find(g["n"], e).tolist() == g["labels"], g["name"]


def test_sequential_runs_match_reference_stats(golden):
    """threads=1 runs are deterministic: labels AND every IterationStats
    field except wall time must equal the reference's."""
    for g in golden["graphs"]:
        e = np.asarray(g["edges"], dtype=np.int64).reshape(-1, 2)
        for key, exp in g["runs"].items():
            variant, mode, ho = key.split("|")
            labels, st = oracle.run_contour(g["n"], e, variant, high_order=int(ho),
                                            sync=(mode == "sync"), threads=1)
            assert labels.tolist() == g["labels"], (g["name"], key)
            assert st.sweeps_executed == exp["executed"], (g["name"], key)
            assert st.sweeps_until_stable == exp["until_stable"], (g["name"], key)
            assert st.changed_per_sweep == exp["changed"], (g["name"], key)
            assert st.converged_by == exp["converged_by"], (g["name"], key)


def _config_edges(params):
    k = params["kind"]
    if k == "er":
        return gen.erdos_renyi(params["n"], params["pairs"], params["seed"])
    if k == "rmat":
        return gen.rmat(params["scale"], params["ef"], params["seed"])
    if k == "grid":
        return gen.grid(params["rows"], params["cols"], params["p"], params["seed"])
    if k == "forest":
        return gen.forest(params["components"], params["seed"])
    raise ValueError(k)


def test_config_generators_and_oracle_pinned(golden):
    for c in golden["configs"]:
        n, e = _config_edges(c["params"])
        assert n == c["n"] and e.shape[0] == c["m"], c["name"]
        assert sha(e) == c["edges_sha256"], c["name"]
        labels = oracle.rem_union_find(n, e)
        assert sha(labels) == c["labels_sha256"], c["name"]
        for key, exp in c["runs"].items():
            if exp["executed"] > 1000:  # C-1 on the forest: 32k sweeps, GPU-tested only
                continue
            variant, mode, ho = key.split("|")
            lab, st = oracle.run_contour(n, e, variant, high_order=int(ho),
                                         sync=(mode == "sync"), threads=1)
            assert sha(lab) == c["labels_sha256"], (c["name"], key)
            assert (st.sweeps_executed, st.sweeps_until_stable, st.changed_per_sweep,
                    st.converged_by) == (exp["executed"], exp["until_stable"],
                                         exp["changed"], exp["converged_by"]), (c["name"], key)


def test_threaded_async_oracle_labels_exact():
    n, e = gen.rmat(12, 16, 7)
    exp = oracle.rem_union_find(n, e)
    for seed in range(4):
        lab, st = oracle.run_contour(n, e, "C-2", atomic=False, threads=4, seed=seed)
        assert np.array_equal(lab, exp)
        assert st.sweeps_until_stable <= st.sweeps_executed <= st.sweeps_until_stable + 1


def test_threaded_sync_atomic_is_order_independent():
    """SURVEY Finding 4: sync + CAS gives the same per-sweep counts for any
    thread count -- the anchor the GPU sync mode is held to."""
    n, e = gen.grid(48, 48, 0.55, 3)
    ref = oracle.run_contour(n, e, "C-2", sync=True, threads=1)[1]
    for t in (2, 5):
        st = oracle.run_contour(n, e, "C-2", sync=True, threads=t, seed=t)[1]
        assert st.changed_per_sweep == ref.changed_per_sweep
        assert st.sweeps_executed == ref.sweeps_executed


def test_parallel_checker_matches_sequential_oracle(golden):
    for g in golden["graphs"][::4]:
        e = np.asarray(g["edges"], dtype=np.int64).reshape(-1, 2)
        assert oracle.parallel_components(g["n"], e, threads=3).tolist() == g["labels"]
    for n, e in (gen.rmat(14, 16, 2), gen.grid(200, 200, 0.55, 1), gen.forest(25, 3)):
        exp = oracle.rem_union_find(n, e)
        for t in (1, 8):
            assert np.array_equal(oracle.parallel_components(n, e, threads=t), exp)
        assert np.array_equal(oracle.parallel_components(n, e.astype(np.int32), 4), exp)


def test_normalize_and_stars():
    assert oracle.normalize_labels(np.array([0, 0, 1, 2])).tolist() == [0, 0, 0, 0]
    with pytest.raises(ValueError):
        oracle.normalize_labels(np.array([0, 5]))
    assert oracle.is_star_forest(np.array([0, 0, 2, 0]))
    assert not oracle.is_star_forest(np.array([0, 0, 1]))


def test_forest_diagnostics_equal_reference():
    """engine.forest_diagnostics (pointer doubling) equals the reference's
    forest_diagnostics (engine.py:373-405) on the committed fixture, errors
    included (cycle -> IterationCapExceeded, out of range -> ValueError)."""
    import json
    import os

    import numpy as np

    from paper_2311_02811_b200 import IterationCapExceeded
    from paper_2311_02811_b200.engine import forest_diagnostics
    with open(os.path.join(os.path.dirname(__file__), "golden", "forest_diag.json")) as fh:
        cases = json.load(fh)["cases"]
    errors = {"IterationCapExceeded": IterationCapExceeded, "ValueError": ValueError}
    for case in cases:
        lab = np.asarray(case["labels"], dtype=np.int64)
        want = case["result"]
        if "error" in want:
            try:
                forest_diagnostics(lab)
            except errors[want["error"]]:
                continue
            raise AssertionError(f"expected {want['error']} for {case['labels'][:10]}")
        d = forest_diagnostics(lab)
        assert d.roots.tolist() == want["roots"]
        assert sorted(d.heights.items()) == [tuple(x) for x in want["heights"]]
        assert sorted(d.class_sizes.items()) == [tuple(x) for x in want["class_sizes"]]
        assert d.merged_min_count == want["merged_min_count"]
