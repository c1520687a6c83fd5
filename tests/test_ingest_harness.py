"""Ingestion (edge list / Matrix Market) and harness helpers against the
reference's own loaders and checksum, via fixtures made from the reference
(tests/golden/make_golden.py).  CPU unless marked."""

import io

import numpy as np
import pytest

from oracle import gen, oracle
from paper_2311_02811_b200 import build, harness, ingest
from paper_2311_02811_b200.errors import EdgeListParseError, MatrixMarketFormatError


@pytest.fixture(scope="module", autouse=True)
def _built():
    build.build()


def _load(case):
    if case["kind"] == "edgelist":
        return ingest.load_edge_list(io.StringIO(case["text"]), **case["kwargs"])
    return ingest.load_matrix_market(io.StringIO(case["text"]))


def test_loaders_match_reference(golden):
    errors = {"EdgeListParseError": EdgeListParseError,
              "MatrixMarketFormatError": MatrixMarketFormatError}
    for case in golden["ingest"]:
        res = case["result"]
        if "error" in res:
            with pytest.raises(errors[res["error"]]) as ei:
                _load(case)
            assert str(ei.value) == res["message"], case["text"]
        else:
            g = _load(case)
            assert g.n == res["n"], case["text"]
            assert g.edges.reshape(-1, 2).tolist() == res["edges"], case["text"]
            got_map = None if g.id_map is None else g.id_map.tolist()
            assert got_map == res["id_map"], case["text"]


def test_large_edge_list_multithreaded_parse(tmp_path):
    """> 1 MiB inputs are tokenised by several threads; rows stay in file
    order and the first error keeps its global line number."""
    n, e = gen.rmat(15, 8, 3)
    lines = [f"{u} {v}" for u, v in e.tolist()]
    text = "# header\n" + "\n".join(lines) + "\n"
    assert len(text) > (1 << 20)
    p = tmp_path / "g.txt"
    p.write_text(text)
    g = ingest.load_edge_list(p, dedupe=False, remap=False)
    canon = np.column_stack([e.min(axis=1), e.max(axis=1)])
    assert np.array_equal(g.edges, canon)
    bad = text.split("\n")
    bad[len(bad) * 3 // 4] = "12 oops"
    p.write_text("\n".join(bad))
    with pytest.raises(EdgeListParseError) as ei:
        ingest.load_edge_list(p)
    assert str(ei.value) == f"line {len(bad) * 3 // 4 + 1}: non-integer token"


def test_binary_edges(tmp_path):
    e = np.array([[0, 1], [2, 3], [3, 3]], dtype=np.int32)
    p = tmp_path / "e.bin"
    e.tofile(p)
    g = ingest.load_binary_edges(p, 4)
    assert g.n == 4 and np.array_equal(g.edges, e)


def test_label_checksum_matches_reference(golden):
    for c in golden["configs"]:
        k = c["params"]["kind"]
        if k == "er":
            n, e = gen.erdos_renyi(c["params"]["n"], c["params"]["pairs"], c["params"]["seed"])
        elif k == "rmat":
            n, e = gen.rmat(c["params"]["scale"], c["params"]["ef"], c["params"]["seed"])
        elif k == "grid":
            n, e = gen.grid(c["params"]["rows"], c["params"]["cols"], c["params"]["p"],
                            c["params"]["seed"])
        else:
            n, e = gen.forest(c["params"]["components"], c["params"]["seed"])
        assert harness.label_checksum(oracle.rem_union_find(n, e)) == c["checksum"], c["name"]


def test_csv_schema_extends_reference():
    assert harness.CSV_COLUMNS == (
        "graph", "n", "m", "algorithm", "variant", "sync", "atomic", "threads",
        "sweeps_until_stable", "sweeps_executed", "wall_time_ms", "components",
        "label_checksum", "oracle_match")
    rec = harness.ExperimentRecord("g", 3, 2, "contour", "C-2", False, True, 1, 1, 2, 0.5, 1,
                                   "abc", True)
    buf = io.StringIO()
    harness.write_csv([rec], buf)
    head, row = buf.getvalue().splitlines()
    assert head.split(",")[:14] == list(harness.CSV_COLUMNS)
    assert row.startswith("g,3,2,contour,C-2,false,true,1,1,2,0.500,1,abc,true")


@pytest.mark.gpu
def test_gpu_harness_records(tmp_path):
    n, e = gen.rmat(12, 16, 4)
    p = tmp_path / "g.txt"
    p.write_text("\n".join(f"{u} {v}" for u, v in e.tolist()) + "\n")
    plan = [harness.PlanItem(graph=(n, e), name="rmat12", variant=v) for v in ("c1", "c2", "cm")]
    plan += [harness.PlanItem(graph=(n, e), name="rmat12", mode="sync"),
             harness.PlanItem(graph=str(p), fmt="edgelist", name="file"),
             harness.PlanItem(graph=(n, e), name="bad", variant="c3")]
    recs = harness.run_experiment(plan, repeats=2,
                                  oracle=lambda nn, ee: oracle.rem_union_find(nn, ee))
    exp = harness.label_checksum(oracle.rem_union_find(n, e))
    for r in recs[:4]:
        assert r.oracle_match and r.verified and r.label_checksum == exp
        assert r.edges_per_s > 0 and r.device_ms > 0
    assert recs[4].oracle_match  # file input: densified IDs, its own oracle
    assert recs[5].error and not recs[5].oracle_match
    harness.write_csv(recs, tmp_path / "out.csv")
    assert (tmp_path / "out.csv").read_text().count("\n") == len(recs) + 1


def _sha(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def _ingest_large():
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "ingest_large.json")) as fh:
        return json.load(fh)["cases"]


def check_ingest_large(load, to_numpy):
    """Run every ~60k-line fixture (oracle/gen.py ingest_text) through
    ``load(case, text, kwargs)`` and compare with the reference's recorded
    output (tests/golden/ingest_large.json)."""
    errors = {"EdgeListParseError": EdgeListParseError,
              "MatrixMarketFormatError": MatrixMarketFormatError}
    for c in _ingest_large():
        text = gen.ingest_text(c["case"])
        res = c["result"]
        if res.get("error") == "MemoryError":
            continue  # the reference's CSR of n = max ID + 1 ~ 1e12 (graph.py:80); see below
        if "error" in res:
            with pytest.raises(errors[res["error"]]) as ei:
                load(c["case"], text, c["kwargs"])
            assert str(ei.value) == res["message"], (c["case"], c["kwargs"])
            continue
        g = load(c["case"], text, c["kwargs"])
        edges = to_numpy(g.edges)
        assert (g.n, edges.shape[0]) == (res["n"], res["m"]), (c["case"], c["kwargs"])
        assert edges[:3].tolist() == res["head"]
        assert _sha(edges) == res["edges"], (c["case"], c["kwargs"])
        got_map = None if g.id_map is None else _sha(to_numpy(g.id_map))
        assert got_map == res["id_map"], (c["case"], c["kwargs"])


def _load_host(case, text, kwargs):
    if case.startswith("edgelist"):
        return ingest.load_edge_list(io.StringIO(text), **kwargs)
    return ingest.load_matrix_market(io.StringIO(text))


def test_loaders_match_reference_large():
    check_ingest_large(_load_host, np.asarray)
