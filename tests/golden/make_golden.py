"""Generate the golden fixtures by running the REFERENCE implementation.

Run (in the build container, where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

It imports the unmodified reference package ``minmapcc`` from
/root/reference/pkg/src and records, for seeded inputs:

* single-edge operator results (engine.py:209-231 ``mm_order``), including
  the known-answer states of the reference's own tests
  (test_engine.py:53-75);
* for a suite of small graphs: ``rem_union_find`` labels (baselines.py:41)
  and the full ``IterationStats`` of ``run_contour`` with threads=1 for
  every variant x {sync, async} (sequential runs are deterministic);
* for config-shaped inputs from oracle/gen.py: edge-array and label
  checksums plus the reference's sweep counts.

The output ``golden.json`` is committed; nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import minmapcc as ref  # noqa: E402
from types import SimpleNamespace  # noqa: E402

from oracle import gen  # noqa: E402

MODES = [(v, s) for v in ref.VARIANTS for s in ((True,) if v == "C-Syn" else (True, False))]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def stats_dict(st):
    return {"executed": st.sweeps_executed, "until_stable": st.sweeps_until_stable,
            "changed": list(map(int, st.changed_per_sweep)), "converged_by": st.converged_by}


def mm_cases(rng):
    cases = []
    # known-answer states from the reference's tests (test_engine.py:53-75)
    fixed = [([0, 1, 2, 3], 1, 2, 1), ([0, 0, 1, 2], 2, 3, 2), ([0, 0, 1, 2], 3, 3, 4)]
    for labels, w, v, order in fixed:
        cases.append((labels, w, v, order))
    for _ in range(150):
        n = int(rng.integers(2, 14))
        labels = [int(rng.integers(0, x + 1)) for x in range(n)]
        cases.append((labels, int(rng.integers(0, n)), int(rng.integers(0, n)),
                      int(rng.integers(1, 6))))
    out = []
    for labels, w, v, order in cases:
        read = np.asarray(labels, dtype=np.int64)
        tgt = read.copy()
        ch = ref.mm_order(tgt, read, w, v, order)
        inplace = read.copy()
        ch2 = ref.mm_order(inplace, inplace, w, v, order)
        out.append({"labels": labels, "w": w, "v": v, "order": order,
                    "target": tgt.tolist(), "changed": bool(ch),
                    "inplace": inplace.tolist(), "inplace_changed": bool(ch2)})
    return out


def small_graphs(rng):
    gs = []
    for n in (1, 2, 3, 5, 8, 13):
        g = ref.generate("path", n=n)
        gs.append((f"path{n}", g.n, g.edges))
    for n in (3, 9):
        g = ref.generate("cycle", n=n)
        gs.append((f"cycle{n}", g.n, g.edges))
    g = ref.generate("star", n=6)
    gs.append(("star6", g.n, g.edges))
    g = ref.generate("grid2d", rows=3, cols=4)
    gs.append(("grid3x4", g.n, g.edges))
    gs.append(("two_components", 4, np.array([[0, 1], [2, 3]])))
    gs.append(("empty", 0, np.zeros((0, 2), np.int64)))
    gs.append(("no_edges", 4, np.zeros((0, 2), np.int64)))
    gs.append(("self_loops_only", 3, np.array([[0, 0], [2, 2]])))
    gs.append(("decreasing_path", 6, np.array([[5, 4], [4, 3], [3, 2], [2, 1], [1, 0]])))
    g = ref.permute_vertices(ref.generate("path", n=40), rng.permutation(40))
    gs.append(("permuted_path40", g.n, g.edges))
    g = ref.generate("erdos_renyi", n=60, p=0.04, seed=3)
    gs.append(("er60", g.n, g.edges))
    g = ref.generate("forest", n=50, trees=4, seed=1)
    gs.append(("forest50", g.n, g.edges))
    for i in range(120):
        n = int(rng.integers(1, 41))
        m = int(rng.integers(0, 81))
        e = rng.integers(0, n, size=(m, 2))
        gs.append((f"rand{i}", n, e))
    out = []
    for name, n, e in gs:
        e = np.asarray(e, dtype=np.int64).reshape(-1, 2)
        ns = SimpleNamespace(n=n, m=e.shape[0], edges=e)
        oracle = ref.rem_union_find(ns)
        runs = {}
        for v, s in MODES:
            for ho in (4, 1024):
                if ho == 1024 and v not in ("C-m", "C-11mm", "C-1m1m"):
                    continue
                lab, st = ref.run_contour(ns, ref.make_schedule(v, ho, sync=s), threads=1)
                assert np.array_equal(lab, oracle)
                runs[f"{v}|{'sync' if s else 'async'}|{ho}"] = stats_dict(st)
        flab, fst = ref.fastsv(ns)
        assert np.array_equal(flab, oracle)
        out.append({"name": name, "n": n, "edges": e.tolist(), "labels": oracle.tolist(),
                    "runs": runs, "fastsv": stats_dict(fst)})
    return out


def configs():
    specs = [
        ("er_config1", lambda: gen.erdos_renyi(65536, 524288, 1),
         {"kind": "er", "n": 65536, "pairs": 524288, "seed": 1}),
        ("rmat10", lambda: gen.rmat(10, 16, 1), {"kind": "rmat", "scale": 10, "ef": 16, "seed": 1}),
        ("rmat14", lambda: gen.rmat(14, 16, 1), {"kind": "rmat", "scale": 14, "ef": 16, "seed": 1}),
        ("grid64", lambda: gen.grid(64, 64, 0.55, 1), {"kind": "grid", "rows": 64, "cols": 64, "p": 0.55, "seed": 1}),
        ("grid512", lambda: gen.grid(512, 512, 0.55, 1), {"kind": "grid", "rows": 512, "cols": 512, "p": 0.55, "seed": 1}),
        ("forest40", lambda: gen.forest(40, 1), {"kind": "forest", "components": 40, "seed": 1}),
    ]
    out = []
    for name, fn, params in specs:
        n, e = fn()
        ns = SimpleNamespace(n=n, m=e.shape[0], edges=e)
        oracle = ref.rem_union_find(ns)
        runs = {}
        for v, s in (("C-2", True), ("C-2", False), ("C-1", True), ("C-m", True), ("C-Syn", True),
                     ("C-11mm", True), ("C-1m1m", True)):
            lab, st = ref.run_contour(ns, ref.make_schedule(v, 1024, sync=s), threads=1)
            assert np.array_equal(lab, oracle)
            runs[f"{v}|{'sync' if s else 'async'}|1024"] = stats_dict(st)
        flab, fst = ref.fastsv(ns)
        assert np.array_equal(flab, oracle)
        out.append({"name": name, "params": params, "n": n, "m": int(e.shape[0]),
                    "edges_sha256": sha(e), "labels_sha256": sha(oracle),
                    "components": int(np.unique(oracle).size),
                    "checksum": ref.label_checksum(oracle), "runs": runs,
                    "fastsv": stats_dict(fst)})
        print(name, n, e.shape[0], out[-1]["components"], runs["C-2|sync|1024"]["executed"],
              flush=True)
    return out


EDGE_LIST_CASES = [
    ("0 1\n1 2\n", {}),
    ("# comment\n% also\n\n3 1\n1 3\n5 5\n", {}),
    ("# comment\n% also\n\n3 1\n1 3\n5 5\n", {"remap": False}),
    ("# comment\n% also\n\n3 1\n1 3\n5 5\n", {"dedupe": False}),
    ("4 2\n2 4\n0 9\n", {"dedupe": False, "remap": False}),
    ("0 1 2\n", {}),
    ("a b\n", {}),
    ("-1 2\n", {}),
    ("#c\n0 1\n\n1\n", {}),
    ("0 1\n2 x\n3\n", {}),
    ("1_0 2\n", {}),
    ("+3 4\n", {}),
    ("", {}),
    ("# only comments\n\n% x\n", {}),
    ("  7\t8  \r\n9 7\r\n", {}),
    ("10 20\n20 30\n40 50\n", {}),
]

MTX_CASES = [
    "%%MatrixMarket matrix coordinate pattern general\n% c\n4 4 3\n1 2\n2 3\n4 4\n",
    "%%MatrixMarket matrix coordinate real symmetric\n3 3 3\n2 1 0.5\n3 1 1.5\n3 3 2\n",
    "%%MatrixMarket matrix coordinate integer general\n3 3 4\n1 2 7\n2 1 7\n% mid\n\n3 2 1\n2 3 1\n",
    "",
    "%%MatrixMarket matrix coordinate pattern\n2 2 1\n1 2\n",
    "%%MatrixMarket matrix array real general\n2 2 1\n1 2\n",
    "%%MatrixMarket matrix coordinate complex general\n2 2 1\n1 2\n",
    "%%MatrixMarket matrix coordinate real hermitian\n2 2 1\n1 2\n",
    "%%MatrixMarket matrix coordinate pattern general\n2 3 1\n1 2\n",
    "%%MatrixMarket matrix coordinate pattern general\n2 2\n1 2\n",
    "%%MatrixMarket matrix coordinate pattern general\n2 2 x\n1 2\n",
    "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1\n",
    "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 y\n",
    "%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 2\n0 1\n",
    "%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 2\n",
    "%%MatrixMarket matrix coordinate pattern general\n% only comments\n",
    "%%MatrixMarket matrix coordinate pattern general\n3 3 2\n1 3\n3 4\n",
    "%%MatrixMarket matrix coordinate pattern general\n0 0 0\n",
]


def ingest_cases():
    import io
    out = []

    def record(kind, text, kwargs, fn):
        try:
            g = fn()
            res = {"n": g.n, "edges": g.edges.tolist(),
                   "id_map": None if g.id_map is None else g.id_map.tolist()}
        except Exception as exc:  # noqa: BLE001 - recording the reference's error
            res = {"error": type(exc).__name__, "message": str(exc)}
        out.append({"kind": kind, "text": text, "kwargs": kwargs, "result": res})

    for text, kw in EDGE_LIST_CASES:
        record("edgelist", text, kw, lambda: ref.load_edge_list(io.StringIO(text), **kw))
    for text in MTX_CASES:
        record("mtx", text, {}, lambda: ref.load_matrix_market(io.StringIO(text)))
    return out


def ingest_large_cases():
    """The reference loaders on seeded texts (oracle/gen.py ingest_text) of
    ~60k lines: outputs as SHA-256 of the int64 edges / id_map, or the error."""
    import io
    out = []
    for case in gen.INGEST_TEXT_CASES:
        text = gen.ingest_text(case)
        kwargs = ([{}, {"remap": False}, {"dedupe": False}, {"remap": False, "dedupe": False}]
                  if case.startswith("edgelist") else [{}])
        for kw in kwargs:
            try:
                if case.startswith("edgelist"):
                    g = ref.load_edge_list(io.StringIO(text), **kw)
                else:
                    g = ref.load_matrix_market(io.StringIO(text))
                res = {"n": int(g.n), "m": int(g.m), "edges": sha(g.edges),
                       "id_map": None if g.id_map is None else sha(g.id_map),
                       "head": g.edges[:3].tolist()}
            except Exception as exc:  # noqa: BLE001 - recording the reference's error
                res = {"error": type(exc).__name__, "message": str(exc)}
            out.append({"case": case, "kwargs": kw, "result": res})
    return out


def forest_diag_cases(rng):
    """forest_diagnostics (engine.py:373-405) on pointer graphs: the
    reference's own examples (test_engine.py:281-309), converged run labels,
    random parent forests (labels[x] <= x), deep chains, and the two error
    cases (a cycle -> IterationCapExceeded, out of range -> ValueError)."""
    arrays = [[0, 0, 1, 2], [0, 1, 2], [0, 0, 0, 1], [0, 0, 1, 0, 3], [], [0],
              list(range(0, 1)) + list(range(0, 29)), [1, 0], [0, 5], [0, -1]]
    for n in (5, 17, 60, 200, 1000):
        for _ in range(4):
            arrays.append([int(rng.integers(0, x + 1)) for x in range(n)])
    for n, e in (gen.rmat(9, 8, 2), gen.grid(12, 12, 0.55, 3), gen.forest(5, 2)):
        ns = SimpleNamespace(n=n, m=e.shape[0], edges=e)
        lab, _ = ref.run_contour(ns, ref.make_schedule("C-2", sync=True), threads=1)
        arrays.append(lab.tolist())
    out = []
    for arr in arrays:
        try:
            d = ref.forest_diagnostics(np.asarray(arr, dtype=np.int64))
            res = {"roots": d.roots.tolist(),
                   "heights": [[k, v] for k, v in sorted(d.heights.items())],
                   "class_sizes": [[k, v] for k, v in sorted(d.class_sizes.items())],
                   "merged_min_count": d.merged_min_count}
        except Exception as exc:  # noqa: BLE001 - recording the reference's error
            res = {"error": type(exc).__name__}
        out.append({"labels": arr, "result": res})
    return out


def main():
    if "--ingest-large" in sys.argv:  # only the large ingestion fixture (ingest_large.json)
        with open(os.path.join(HERE, "ingest_large.json"), "w") as fh:
            json.dump({"generator": "tests/golden/make_golden.py --ingest-large",
                       "reference": "minmapcc " + ref.__version__,
                       "cases": ingest_large_cases()}, fh, indent=0)
        return
    if "--forest-diag" in sys.argv:  # only the forest_diagnostics fixture (forest_diag.json)
        with open(os.path.join(HERE, "forest_diag.json"), "w") as fh:
            json.dump({"generator": "tests/golden/make_golden.py --forest-diag",
                       "reference": "minmapcc " + ref.__version__,
                       "cases": forest_diag_cases(np.random.default_rng(405))}, fh,
                      separators=(",", ":"))
        return
    rng = np.random.default_rng(20261020)
    data = {"generator": "tests/golden/make_golden.py", "reference": "minmapcc " + ref.__version__,
            "mm_order": mm_cases(rng), "graphs": small_graphs(rng), "configs": configs(),
            "ingest": ingest_cases()}
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(data, fh, separators=(",", ":"))


if __name__ == "__main__":
    main()
