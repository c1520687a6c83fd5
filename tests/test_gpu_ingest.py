"""Device ingestion (csrc/ingest.inc) against the
reference loaders' recorded outputs (graph.py:149-274; fixtures made by
tests/golden/make_golden.py from the unmodified reference) and against the
host path on inputs the reference cannot load (IDs ~1e12 without remap)."""

import io

import numpy as np
import pytest

from oracle import gen, oracle
from paper_2311_02811_b200 import build, ingest, make_schedule, run_contour
from paper_2311_02811_b200.errors import EdgeListParseError, MatrixMarketFormatError

from test_ingest_harness import _load, check_ingest_large

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    build.build()


def _np(t):
    return t.cpu().numpy()


def _load_dev(case, text, kwargs):
    if case.startswith("edgelist"):
        return ingest.load_edge_list(io.StringIO(text), device=0, **kwargs)
    return ingest.load_matrix_market(io.StringIO(text), device=0)


def test_device_loaders_match_reference_small(golden):
    errors = {"EdgeListParseError": EdgeListParseError,
              "MatrixMarketFormatError": MatrixMarketFormatError}
    for case in golden["ingest"]:
        res = case["result"]
        if case["kind"] == "edgelist":
            fn = lambda: ingest.load_edge_list(io.StringIO(case["text"]), device=0,  # noqa: E731
                                               **case["kwargs"])
        else:
            fn = lambda: ingest.load_matrix_market(io.StringIO(case["text"]), device=0)  # noqa
        if "error" in res:
            with pytest.raises(errors[res["error"]]) as ei:
                fn()
            assert str(ei.value) == res["message"], case["text"]
            continue
        g = fn()
        assert g.edges.is_cuda
        assert g.n == res["n"], case["text"]
        assert _np(g.edges).reshape(-1, 2).tolist() == res["edges"], case["text"]
        got = None if g.id_map is None else _np(g.id_map).tolist()
        assert got == res["id_map"], case["text"]


def test_device_loaders_match_reference_large():
    check_ingest_large(_load_dev, _np)


def test_device_ids_beyond_32_bits_equal_host():
    """remap=False with IDs up to 1e12: the two-pass (v, then u) stable sort
    path; the reference itself cannot build this graph (its CSR has n entries)."""
    text = gen.ingest_text("edgelist_sparse")
    for dedupe in (True, False):
        h = ingest.load_edge_list(io.StringIO(text), remap=False, dedupe=dedupe)
        d = ingest.load_edge_list(io.StringIO(text), remap=False, dedupe=dedupe, device=0)
        assert d.n == h.n and d.id_map is None
        assert np.array_equal(_np(d.edges), h.edges)


def test_device_text_tensor_and_file(tmp_path):
    import torch
    text = gen.ingest_text("edgelist_dense", seed=3)
    p = tmp_path / "g.txt"
    p.write_text(text)
    h = ingest.load_edge_list(p)
    d1 = ingest.load_edge_list(p, device=0)
    t = torch.frombuffer(bytearray(text.encode()), dtype=torch.uint8).cuda()
    d2 = ingest.load_edge_list(t, device="cuda:0")
    for d in (d1, d2):
        assert d.n == h.n and np.array_equal(_np(d.edges), h.edges)
        assert (d.id_map is None) == (h.id_map is None)
        if h.id_map is not None:
            assert np.array_equal(_np(d.id_map), h.id_map)


def test_device_edge_cases():
    for text in ("", "\n\n", "# only\n% comments", "0 1", "3 3\n3 3\n", "5\t7\r\n7 5\r\n",
                 "1 2\n" * 5000, "  +1_0   0012  \n"):
        for kw in ({}, {"remap": False}, {"dedupe": False}):
            h = ingest.load_edge_list(io.StringIO(text), **kw)
            d = ingest.load_edge_list(io.StringIO(text), device=0, **kw)
            assert d.n == h.n, (text, kw)
            assert _np(d.edges).reshape(-1, 2).tolist() == h.edges.reshape(-1, 2).tolist()
    with pytest.raises(EdgeListParseError, match="line 3: non-integer token"):
        ingest.load_edge_list(io.StringIO("1 2\n\n1 a\n"), device=0)
    # the handle survives an error and parses the next input
    g = ingest.load_edge_list(io.StringIO("4 2\n"), device=0)
    assert g.n == 2 and _np(g.edges).tolist() == [[0, 1]]


def test_device_large_multimegabyte_parse_and_run(tmp_path):
    """A few-MiB RMAT edge list (several pinned chunks when pageable): the
    loaded CUDA tensor goes straight into run_contour (device-to-device
    staging) and the labels equal the oracle's on the host-loaded graph."""
    n, e = gen.rmat(16, 8, 5)
    text = "# rmat 16\n" + "\n".join(f"{u} {v}" for u, v in e.tolist()) + "\n"
    g = ingest.load_edge_list(io.StringIO(text), device=0)
    h = ingest.load_edge_list(io.StringIO(text))
    assert g.n == h.n and np.array_equal(_np(g.edges), h.edges)
    labels, _ = run_contour(g, make_schedule("c2"))
    assert np.array_equal(labels, oracle.rem_union_find(h.n, h.edges))


def test_device_golden_kinds_through_helper(golden):
    # the host helper used by the CPU test keeps working next to the device path
    for case in golden["ingest"][:3]:
        if "error" not in case["result"]:
            assert _load(case).n == case["result"]["n"]
