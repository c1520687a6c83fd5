"""Product generators (C++ host, in libcontour.so) == the numpy
specification in oracle/gen.py, bit for bit.  CPU only."""

import numpy as np
import pytest

from oracle import gen as spec
from paper_2311_02811_b200 import build, graphgen


@pytest.fixture(scope="module", autouse=True)
def _built():
    build.build()


@pytest.mark.parametrize("scale,ef,seed,sym", [(1, 1, 0, True), (6, 4, 3, True), (10, 16, 1, True),
                                               (11, 8, 9, False)])
def test_rmat_matches_spec(scale, ef, seed, sym):
    n0, e0 = spec.rmat(scale, ef, seed, symmetrize=sym)
    n1, e1 = graphgen.rmat(scale, ef, seed, symmetrize=sym)
    assert n0 == n1 and np.array_equal(e0, e1)
    n2, e2 = graphgen.rmat(scale, ef, seed, symmetrize=sym, elem_bytes=4)
    assert np.array_equal(e0, e2.astype(np.int64))


def test_rmat_row_slices_concatenate():
    n, full = graphgen.rmat(9, 16, 5)
    parts = [graphgen.rmat(9, 16, 5, row_lo=lo, row_hi=hi)[1]
             for lo, hi in ((0, 1000), (1000, 9000), (9000, full.shape[0]))]
    assert np.array_equal(np.concatenate(parts), full)


def test_rmat_degree_skew_and_symmetry():
    n, e = graphgen.rmat(12, 16, 1)
    M = e.shape[0] // 2
    assert np.array_equal(e[:M, 0], e[M:, 1]) and np.array_equal(e[:M, 1], e[M:, 0])
    deg = np.bincount(e[:, 0], minlength=n)
    assert deg.max() > 20 * deg.mean()  # power-law-ish


@pytest.mark.parametrize("rows,cols,p,seed", [(1, 1, 0.55, 1), (1, 7, 0.5, 2), (5, 1, 0.9, 3),
                                              (64, 64, 0.55, 1), (300, 257, 0.55, 4)])
def test_grid_matches_spec(rows, cols, p, seed):
    n0, e0 = spec.grid(rows, cols, p, seed)
    n1, e1 = graphgen.grid(rows, cols, p, seed)
    assert n0 == n1 and np.array_equal(e0, e1)


def test_er_matches_spec():
    n0, e0 = spec.erdos_renyi(65536, 524288, 1)
    n1, e1 = graphgen.erdos_renyi(65536, 524288, 1)
    assert n0 == n1 and np.array_equal(e0, e1)
    assert (e1[:, 0] != e1[:, 1]).all()
    n2, e2 = graphgen.erdos_renyi(1000, 5000, 3)
    assert np.array_equal(e2, spec.erdos_renyi(1000, 5000, 3)[1])


@pytest.mark.parametrize("comps,seed", [(1, 1), (7, 2), (40, 1)])
def test_forest_matches_spec(comps, seed):
    assert np.array_equal(graphgen.forest_sizes(comps, seed), spec.forest_sizes(comps, seed))
    n0, e0 = spec.forest(comps, seed)
    n1, e1 = graphgen.forest(comps, seed)
    assert n0 == n1 and np.array_equal(e0, e1)


def test_permutation_is_bijection():
    for n in (1, 2, 3, 1000, 4096, 5003):
        p = spec.permute_ids(np.arange(n, dtype=np.uint64), n, spec.key(7, 2))
        assert np.array_equal(np.sort(p), np.arange(n, dtype=np.uint64))
