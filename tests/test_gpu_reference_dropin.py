"""The drop-in boundary exercised from the reference's side (INTEGRATION.md
Option B): the unmodified reference package (installed in baseline/_ref),
copied with the maintainer's two additions -- minmapcc/_cuda.py binding
libcontour.so and the MINMAPCC_DEVICE=cuda dispatch in engine.run_contour --
runs its OWN harness (bench.run_experiment, bench.py:149-201, with its oracle
gate, and verify_labels, bench.py:85-92) on RMAT, grid and forest plans.
Every record must match the oracle, with the same label_checksum as the
reference's CPU run of the same plan; synchronous plans must also report the
same sweep counts.  Skipped when the reference is not installed."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PKG = os.path.join(ROOT, "baseline", "_ref", "minmapcc")
LIB = os.path.join(ROOT, "paper_2311_02811_b200", "lib", "libcontour.so")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.isdir(REF_PKG),
                                 reason="reference not installed in baseline/_ref")]

_SCRIPT = r"""
import json, sys
sys.path.insert(0, {root!r})
import numpy as np
from oracle import gen
from minmapcc import Graph, bench, run_contour, make_schedule
graphs = {{
    "rmat12": gen.rmat(12, 16, 3),
    "grid120": gen.grid(120, 120, 0.55, 2),
    "forest": gen.forest(12, 5),
}}
plan = []
for name, (n, e) in graphs.items():
    g = Graph.from_edges(n, e, name=name)
    for variant, mode in (("c2", "async"), ("c2", "sync"), ("c1", "sync"), ("cm", "async"),
                          ("c11mm", "sync")):
        plan.append(bench.PlanItem(graph=g, name=name, variant=variant, mode=mode,
                                   high_order=8))
recs = bench.run_experiment(plan, repeats=1)
out = [dict(graph=r.graph, variant=r.variant, sync=r.sync, match=r.oracle_match,
            checksum=r.label_checksum, executed=r.sweeps_executed,
            until=r.sweeps_until_stable, components=r.components, error=r.error)
       for r in recs]
n, e = graphs["rmat12"]
g = Graph.from_edges(n, e)
labels, st = run_contour(g, make_schedule("c2"))
rep = bench.verify_labels(g, labels)
print("RESULT " + json.dumps(dict(records=out, verify=rep.match,
                                  sweeps=st.sweeps_executed, by=st.converged_by)))
"""


def _run(tmp, cuda):
    env = dict(os.environ, PYTHONPATH=str(tmp), NUMBA_CACHE_DIR=str(tmp / "numba"),
               PYTHONDONTWRITEBYTECODE="1", MINMAPCC_CONTOUR_LIB=LIB)
    env.pop("MINMAPCC_DEVICE", None)
    if cuda:
        env["MINMAPCC_DEVICE"] = "cuda"
    out = subprocess.run([sys.executable, "-c", _SCRIPT.format(root=ROOT)], env=env, cwd=tmp,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads([x for x in out.stdout.splitlines() if x.startswith("RESULT ")][-1][7:])


def test_reference_harness_through_option_b(tmp_path):
    sys.path.insert(0, os.path.join(ROOT, "integration"))
    import apply_option_b
    pkg = apply_option_b.apply(REF_PKG, str(tmp_path))
    assert os.path.exists(os.path.join(pkg, "_cuda.py"))
    gpu = _run(tmp_path, cuda=True)
    cpu = _run(tmp_path, cuda=False)
    assert gpu["verify"] and cpu["verify"]
    assert len(gpu["records"]) == len(cpu["records"]) == 15
    for a, b in zip(gpu["records"], cpu["records"]):
        assert a["error"] is None and a["match"], a
        assert a["checksum"] == b["checksum"] and a["components"] == b["components"], (a, b)
        if a["sync"]:  # deterministic: the same per-sweep accounting as the reference
            assert (a["executed"], a["until"]) == (b["executed"], b["until"]), (a, b)
