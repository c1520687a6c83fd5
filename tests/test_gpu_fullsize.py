"""Full-size parity for BASELINE.json configs[2..4] on the device (SURVEY.md
8(c); the reference's acceptance C1, test_acceptance.py:122-129: labels equal
to the union-find oracle's).

* configs[2] grid 4096^2: labels against the sequential oracle restatement.
* configs[3] forest (n = 2,307,095,021 > INT32_MAX, uint32 vertex IDs): labels
  against the multi-threaded union-find checker (rem_union_find's output
  contract) on the full graph; plus a cheap graph whose edges use only IDs
  above 2^31 on n = 2^31 + 2^20, checked on the compacted ID set and, for
  every untouched vertex, L[x] == x.
* configs[4] RMAT-28 (8,589,934,592 rows): generated on the device, run in
  the bench's layout, certified by cc_verify, and equal to the checker's
  labels computed from the same rows read back to the host.

These need up to ~75 GB of host RAM and ~140 GB of HBM (a B200 box)."""

import numpy as np
import pytest

from oracle import oracle
from paper_2311_02811_b200 import _lib, engine, graphgen, make_schedule

pytestmark = pytest.mark.gpu


def _read_labels(ctx, n, eb=8):
    out = np.empty(n, dtype=np.int64 if eb == 8 else np.uint32)
    _lib.check(ctx.lib.cc_read_labels(ctx.handle, out.ctypes.data, eb))
    return out


def test_grid4096_full_size_exact():
    n, e = graphgen.grid(4096, 4096, 0.55, 1, elem_bytes=8)
    exp = oracle.rem_union_find(n, e)
    ctx = _lib.Context(0)
    for layout in ("auto", "l2_tiled"):
        engine.stage_graph(ctx, n, e, layout)
        for early in (False, True):
            labels = np.empty(n, dtype=np.int64)
            _, st = engine.run_staged(ctx, make_schedule("c2"), count_changes=False,
                                      early_check=early, labels_out=labels)
            assert np.array_equal(labels, exp), (layout, early)
            assert engine.verify_staged(ctx) == 0
    # synchronous C-2 on the full grid: the device's per-sweep counts equal the
    # reference restatement's (SURVEY Finding 4)
    labels = np.empty(n, dtype=np.int64)
    _, st = engine.run_staged(ctx, make_schedule("c2", sync=True), labels_out=labels)
    _, ref = oracle.run_contour(n, e, "C-2", sync=True, threads=8)
    assert np.array_equal(labels, exp)
    assert st.changed_per_sweep == list(ref.changed_per_sweep)
    assert st.sweeps_executed == ref.sweeps_executed
    ctx.close()


def test_ids_above_int32_max_compacted_check():
    """uint32 vertex IDs beyond 2^31 on the device (k_stage range check,
    lab_t arithmetic, widening to int64 on the way out)."""
    rng = np.random.default_rng(31)
    n = (1 << 31) + (1 << 20)
    hi = rng.integers(1 << 31, n, size=(300_000, 2), dtype=np.int64)
    lo = rng.integers(0, 1 << 20, size=(2_000, 2), dtype=np.int64)  # a few mixed edges too
    lo[:, 1] = rng.integers(1 << 31, n, size=2_000)
    e = np.concatenate([hi, lo])
    ids, inv = np.unique(e.ravel(), return_inverse=True)
    comp = oracle.rem_union_find(ids.size, inv.reshape(-1, 2))
    exp_touched = ids[comp]  # the component minimum, mapped back to the original IDs
    ctx = _lib.Context(0)
    engine.stage_graph(ctx, n, e, "input")
    engine.run_staged(ctx, make_schedule("c2"), count_changes=False, early_check=False)
    assert engine.verify_staged(ctx) == 0
    lab = _read_labels(ctx, n, 4)
    ctx.close()
    expected = np.arange(n, dtype=np.uint32)  # untouched vertices keep their own ID
    expected[ids] = exp_touched.astype(np.uint32)
    assert np.array_equal(lab, expected)
    del lab, expected
    # the same through the drop-in entry point, labels as int64
    from paper_2311_02811_b200 import run_contour
    labels, st = run_contour((n, e), make_schedule("c2"))
    assert np.array_equal(labels[ids], exp_touched)
    assert labels[(1 << 31) - 1] == (1 << 31) - 1 or ((1 << 31) - 1) in ids


def test_forest_config_full_size_exact():
    """configs[3] at full size: 200,000 paths / random trees + 20 % isolated
    vertices, n = 2,307,095,021 (uint32 IDs), 1,845,476,017 rows."""
    n, e = graphgen.forest(200_000, 1, elem_bytes=8)
    assert n > 2 ** 31
    ctx = _lib.Context(0)
    layout = engine.resolve_layout("auto", e.shape[0], n)
    engine.stage_graph(ctx, n, e, layout)
    _, st = engine.run_staged(ctx, make_schedule("c2"), count_changes=False, early_check=True)
    assert engine.verify_staged(ctx) == 0
    labels = _read_labels(ctx, n, 8)
    ctx.close()
    exp = oracle.parallel_components(n, e)
    assert np.array_equal(labels, exp)
    assert st.sweeps_until_stable <= st.sweeps_executed <= st.sweeps_until_stable + 1


def test_rmat28_north_star_config_exact():
    """configs[4] at full size on one B200, in the bench's layout (L2-window
    tiles + the bitmap check copy), against the union-find checker."""
    ctx = _lib.Context(0)
    n, m = graphgen.rmat_device(ctx, 28, 16, 1)
    assert (n, m) == (1 << 28, 8_589_934_592)
    host = graphgen.read_edges(ctx, 4)  # input order, before any layout
    layout = engine.resolve_layout("auto", m, n)
    assert layout == "l2_tiled_check"
    engine.apply_layout(ctx, layout)
    for _ in range(2):
        _, st = engine.run_staged(ctx, make_schedule("c2"), count_changes=False,
                                  early_check=True)
        assert engine.verify_staged(ctx) == 0
        assert st.sweeps_until_stable <= st.sweeps_executed <= st.sweeps_until_stable + 1
    labels = _read_labels(ctx, n, 8)
    ctx.close()
    exp = oracle.parallel_components(n, host)
    del host
    assert np.array_equal(labels, exp)
    assert int(np.count_nonzero(exp == np.arange(n))) == 147_230_794  # components (DESIGN 8)
