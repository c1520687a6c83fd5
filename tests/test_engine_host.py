"""Host-side logic of the drop-in engine (schedules, validation) -- the same
known answers as the reference's test_engine.py:99-132, 181-183.  CPU only."""

import pytest

from oracle import oracle
from paper_2311_02811_b200 import VARIANTS, make_schedule, run_contour
from paper_2311_02811_b200.engine import Schedule, canonical_variant


def test_alternating_variant():
    s = make_schedule("c1m1m", 1024)
    assert [s.order_for(k) for k in range(1, 7)] == [1, 1024, 1, 1024, 1, 1024]


def test_constant_high_order():
    assert {make_schedule("cm", 1024).order_for(k) for k in range(1, 9)} == {1024}


def test_warmup_then_high():
    s = make_schedule("c11mm", 8, warmup=2)
    assert [s.order_for(k) for k in range(1, 7)] == [1, 1, 8, 8, 8, 8]


def test_csyn_is_sync_order_two():
    s = make_schedule("csyn")
    assert s.sync is True and s.order_for(3) == 2
    with pytest.raises(ValueError):
        make_schedule("csyn", sync=False)


def test_validation():
    with pytest.raises(ValueError):
        make_schedule("c3")
    with pytest.raises(ValueError):
        make_schedule("cm", high_order=1)
    with pytest.raises(ValueError):
        make_schedule("c2", warmup=0)
    make_schedule("c1", high_order=1)
    assert make_schedule("C-2").variant == "C-2"
    assert canonical_variant(" c-11MM ") == "C-11mm"


def test_order_for_matches_oracle_restatement():
    for v in VARIANTS:
        s = make_schedule(v, 16, warmup=3)
        assert [s.order_for(k) for k in range(1, 12)] == \
            [oracle.order_for(v, k, 16, 3) for k in range(1, 12)]


def test_defaults_match_reference():
    s = Schedule("C-2")
    assert (s.high_order, s.warmup, s.sync, s.atomic) == (1024, 2, False, True)


def test_threads_validated_before_any_device_work():
    with pytest.raises(ValueError):
        run_contour((3, [(0, 1), (1, 2)]), make_schedule("c2"), threads=0)


def test_auto_layout_policy():
    """engine.resolve_layout: input order for small inputs, L2 windows for label
    arrays beyond L2, the hybrid layout only for dense graphs staged once and
    run from HBM (m >= 8n, m < 2^31), chunk_sorted otherwise and for one-shot
    host runs (sweep 1 streams behind the copy)."""
    from paper_2311_02811_b200.engine import resolve_layout
    assert resolve_layout("auto", (1 << 16) - 1, 1000) == "input"
    assert resolve_layout("auto", 524282, 65536) == "chunk_sorted"                 # ER config
    assert resolve_layout("auto", 134217728, 4194304) == "hybrid"               # RMAT-22
    assert resolve_layout("auto", 134217728, 4194304, resident=False) == "chunk_sorted"
    assert resolve_layout("auto", 18446634, 16777216) == "chunk_sorted"          # grid 4096^2
    assert resolve_layout("auto", 8589934592, 268435456) == "l2_tiled_check"     # RMAT-28
    assert resolve_layout("auto", 8589934592, 268435456, resident=False) == "chunk_sorted"
    assert resolve_layout("auto", 8589934592 // 8, 268435456, copies=False) == "l2_tiled"
    assert resolve_layout("auto", 1845476017, 2307095021, resident=False) == "l2_tiled"
    assert resolve_layout("auto", 1845476017, 2307095021) == "relabel"           # forest
    assert resolve_layout("auto", 1845476017, 2307095021, copies=False) == "l2_tiled"
    assert resolve_layout("auto", 1 << 31, 1 << 24) == "chunk_sorted"            # m >= 2^31
    for lay in ("input", "src_sorted", "chunk_sorted", "dst_bucketed", "l2_tiled", "hybrid",
                "l2_tiled_check", "relabel"):
        assert resolve_layout(lay, 10, 10) == lay
    with pytest.raises(ValueError):
        resolve_layout("bogus", 10, 10)


def test_conditional_min_assign_semantics():
    """engine.py:158-189: only cells strictly above the value are lowered;
    atomic and plain modes agree."""
    import numpy as np
    from paper_2311_02811_b200 import conditional_min_assign
    a = np.array([5, 2, 8, 3], dtype=np.int64)
    assert conditional_min_assign(a, [0, 2, 3], 3) is True
    assert a.tolist() == [3, 2, 3, 3]
    assert conditional_min_assign(a, [1, 3], 3) is False  # equal or below: untouched
    b = np.array([6, 1, 9], dtype=np.int64)
    c = b.copy()
    assert conditional_min_assign(b, [0, 2], 4) == conditional_min_assign(c, [0, 2], 4, True)
    assert b.tolist() == c.tolist() == [4, 1, 4]


def test_forest_diagnostics_matches_a_chain_walk():
    """engine.py:373-405 restated by pointer doubling: roots, heights, class
    sizes against a direct per-vertex chain walk, plus the error cases."""
    import numpy as np
    from paper_2311_02811_b200 import IterationCapExceeded, forest_diagnostics
    rng = np.random.default_rng(7)
    for n in (0, 1, 2, 9, 200, 1500):
        lab = np.array([int(rng.integers(0, i + 1)) for i in range(n)], dtype=np.int64)
        d = forest_diagnostics(lab)
        roots = [x for x in range(n) if lab[x] == x]
        heights = {r: 0 for r in roots}
        for x in range(n):
            y, depth = x, 0
            while lab[y] != y:
                y, depth = int(lab[y]), depth + 1
            heights[y] = max(heights[y], depth)
        sizes = {}
        for v in lab.tolist():
            sizes[v] = sizes.get(v, 0) + 1
        assert d.roots.tolist() == roots
        assert d.heights == heights
        assert d.class_sizes == sizes and d.merged_min_count == len(sizes)
    d = forest_diagnostics(np.array([0, 0, 1, 2, 3]))
    assert d.heights == {0: 4} and d.class_sizes == {0: 2, 1: 1, 2: 1, 3: 1}
    with pytest.raises(ValueError):
        forest_diagnostics(np.array([0, 3]))
    with pytest.raises(IterationCapExceeded):
        forest_diagnostics(np.array([1, 0, 2]))  # 0 <-> 1 cycle
