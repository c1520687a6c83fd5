"""INTEGRATION.md Option B on CPU: the maintainer-side patch applies cleanly
to a copy of the installed reference (baseline/_ref), the patched package
imports, keeps its CPU path when MINMAPCC_DEVICE is unset, and the
_cuda.py binding declares exactly the C-ABI symbols it uses (all exported by
libcontour.so).  The GPU run of the reference's harness through it is
tests/test_gpu_reference_dropin.py."""

import ctypes
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PKG = os.path.join(ROOT, "baseline", "_ref", "minmapcc")

pytestmark = pytest.mark.skipif(not os.path.isdir(REF_PKG),
                                reason="reference not installed in baseline/_ref")


def test_patch_applies_and_cpu_path_unchanged(tmp_path):
    sys.path.insert(0, os.path.join(ROOT, "integration"))
    import apply_option_b
    pkg = apply_option_b.apply(REF_PKG, str(tmp_path))
    src = open(os.path.join(pkg, "engine.py")).read()
    assert src.count('os.environ.get("MINMAPCC_DEVICE") == "cuda"') == 1
    script = ("import inspect, numpy as np\n"
              "from minmapcc import engine, run_contour, make_schedule, rem_union_find, Graph\n"
              "assert 'run_contour_cuda' in inspect.getsource(engine.run_contour)\n"
              "g = Graph.from_edges(6, np.array([[0, 1], [2, 3], [3, 4]]))\n"
              "labels, st = run_contour(g, make_schedule('c2'))\n"
              "assert labels.tolist() == [0, 0, 2, 2, 2, 5], labels\n"
              "print('ok')\n")
    env = dict(os.environ, PYTHONPATH=str(tmp_path), NUMBA_CACHE_DIR=str(tmp_path / "nb"),
               PYTHONDONTWRITEBYTECODE="1")
    env.pop("MINMAPCC_DEVICE", None)
    out = subprocess.run([sys.executable, "-c", script], env=env, cwd=tmp_path,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_binding_symbols_exported():
    from paper_2311_02811_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    src = open(os.path.join(ROOT, "integration", "minmapcc_cuda.py")).read()
    for sym in ("cc_create", "cc_run_host", "cc_last_error"):
        assert sym in src
        assert hasattr(lib, sym)
