"""Numpy specification of the seeded synthetic inputs -- TEST INFRASTRUCTURE.

BASELINE.json's five configs are synthetic and none is produced by the
reference's own ``generate()`` (graph.py:277-332), so
this repo owns the generators.  They are defined by a counter-based RNG
(splitmix64 finaliser keyed by (seed, stream, index)) so that the product's
host C++ generator and its CUDA generator can reproduce the arrays bit for bit
at any scale; ``tests/test_gen.py`` checks the product generators against
this restatement.

Edge rows are returned as the reference's (m, 2) int64 array (graph.py:66).
"""

from __future__ import annotations

import math

import numpy as np

GOLD = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
ODD = [np.uint64(0x9E3779B97F4A7C15), np.uint64(0xBF58476D1CE4E5B9),
       np.uint64(0x94D049BB133111EB), np.uint64(0xD6E8FEB86659FD93)]

STREAM_RMAT, STREAM_PERM, STREAM_GRID, STREAM_ER, STREAM_FSIZE, STREAM_FTREE = 1, 2, 3, 4, 5, 6
MASK32 = np.uint64(0xFFFFFFFF)


def _u64(x):
    return np.asarray(x, dtype=np.uint64)


def mix(z):
    z = _u64(z)
    with np.errstate(over="ignore"):
        z = z ^ (z >> np.uint64(30))
        z = z * M1
        z = z ^ (z >> np.uint64(27))
        z = z * M2
        z = z ^ (z >> np.uint64(31))
    return z


def key(seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        return mix(_u64(seed & 0xFFFFFFFFFFFFFFFF) * GOLD + _u64(stream + 1))[()]


def rnd(k, idx):
    with np.errstate(over="ignore"):
        return mix(_u64(k) + (_u64(idx) + np.uint64(1)) * GOLD)


def perm_bits(n: int) -> int:
    return 0 if n <= 1 else int(n - 1).bit_length()


def _perm_pow2(x, pkey, k):
    if k == 0:
        return np.zeros_like(_u64(x))
    mask = np.uint64((1 << k) - 1)
    s = np.uint64((k + 1) // 2)
    x = _u64(x) & mask
    with np.errstate(over="ignore"):
        for r in range(4):
            kr = rnd(pkey, r) & mask
            x = (x * ODD[r] + kr) & mask
            x = x ^ (x >> s)
    return x


def permute_ids(x, n: int, pkey):
    """Keyed bijection on [0, n): 4-round multiply/xorshift permutation of the
    next power-of-two domain plus cycle walking."""
    k = perm_bits(n)
    y = _perm_pow2(x, pkey, k)
    bad = y >= np.uint64(n)
    while bad.any():
        y[bad] = _perm_pow2(y[bad], pkey, k)
        bad = y >= np.uint64(n)
    return y


def rmat_thresholds(a=0.57, b=0.19, c=0.19):
    return (int(a * 2 ** 32), int((a + b) * 2 ** 32), int((a + b + c) * 2 ** 32))


def rmat(scale: int, edgefactor: int = 16, seed: int = 1, symmetrize: bool = True,
         a=0.57, b=0.19, c=0.19, permute: bool = True) -> tuple[int, np.ndarray]:
    """Kronecker/RMAT: edge i draws its quadrant per bit level (MSB first)
    from (a, b, c, d); IDs permuted by the keyed bijection; symmetrised by
    appending (v, u) after all (u, v) rows; self-loops/duplicates kept."""
    n = 1 << scale
    M = edgefactor * n
    tA, tAB, tABC = (np.uint64(t) for t in rmat_thresholds(a, b, c))
    kr = key(seed, STREAM_RMAT)
    D = (scale + 1) // 2
    i = np.arange(M, dtype=np.uint64)
    u = np.zeros(M, dtype=np.uint64)
    v = np.zeros(M, dtype=np.uint64)
    d = None
    for lvl in range(scale):
        if lvl % 2 == 0:
            d = rnd(kr, i * np.uint64(D) + np.uint64(lvl // 2))
            r = d & MASK32
        else:
            r = d >> np.uint64(32)
        ub = (r >= tAB).astype(np.uint64)
        vb = (((r >= tA) & (r < tAB)) | (r >= tABC)).astype(np.uint64)
        u = (u << np.uint64(1)) | ub
        v = (v << np.uint64(1)) | vb
    if permute:
        pk = key(seed, STREAM_PERM)
        u = permute_ids(u, n, pk)
        v = permute_ids(v, n, pk)
    if symmetrize:
        src = np.concatenate([u, v])
        dst = np.concatenate([v, u])
    else:
        src, dst = u, v
    return n, np.stack([src, dst], axis=1).astype(np.int64)


def grid(rows: int, cols: int, p: float = 0.55, seed: int = 1,
         permute: bool = True) -> tuple[int, np.ndarray]:
    """rows x cols lattice; horizontal bonds (index r*(cols-1)+c) then
    vertical bonds (index R_h + r*cols + c); each kept iff the high 32 bits
    of its draw are < floor(p*2^32); IDs permuted."""
    n = rows * cols
    nh = rows * max(cols - 1, 0)
    nv = max(rows - 1, 0) * cols
    b = np.arange(nh + nv, dtype=np.uint64)
    keep = (rnd(key(seed, STREAM_GRID), b) >> np.uint64(32)) < np.uint64(int(p * 2 ** 32))
    b = b[keep].astype(np.int64)
    hor = b < nh
    bh = b[hor]
    bv = b[~hor] - nh
    su = np.empty(b.size, dtype=np.int64)
    sv = np.empty(b.size, dtype=np.int64)
    if cols > 1:
        su[hor] = (bh // (cols - 1)) * cols + bh % (cols - 1)
        sv[hor] = su[hor] + 1
    su[~hor] = bv
    sv[~hor] = bv + cols
    if permute:
        pk = key(seed, STREAM_PERM)
        su = permute_ids(su, n, pk).astype(np.int64)
        sv = permute_ids(sv, n, pk).astype(np.int64)
    return n, np.stack([su, sv], axis=1)


def erdos_renyi(n: int, m: int, seed: int = 1) -> tuple[int, np.ndarray]:
    """m i.i.d. uniform pairs (low/high 32 bits of draw i, mod n); self-loops
    dropped, duplicates kept, no canonicalisation."""
    d = rnd(key(seed, STREAM_ER), np.arange(m, dtype=np.uint64))
    u = (d & MASK32) % np.uint64(n)
    v = (d >> np.uint64(32)) % np.uint64(n)
    keep = u != v
    return n, np.stack([u[keep], v[keep]], axis=1).astype(np.int64)


def forest_sizes(components: int, seed: int = 1, lo: int = 2, hi: int = 100_000) -> np.ndarray:
    """Component sizes floor(exp(U(ln lo, ln hi))) with U from the high 53 bits."""
    d = rnd(key(seed, STREAM_FSIZE), np.arange(components, dtype=np.uint64))
    U = (d >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    s = np.floor(np.exp(math.log(lo) + U * (math.log(hi) - math.log(lo)))).astype(np.int64)
    return np.clip(s, lo, hi)


def forest(components: int, seed: int = 1, isolated_frac: float = 0.2,
           lo: int = 2, hi: int = 100_000) -> tuple[int, np.ndarray]:
    """Disjoint components (even index: path, odd index: random recursive
    tree with parent of local vertex j = draw(off+j) mod j) over contiguous
    pre-permutation ID ranges, then isolated vertices so they are
    `isolated_frac` of n, then all IDs permuted."""
    sizes = forest_sizes(components, seed, lo, hi)
    T = int(sizes.sum())
    iso = int(round(T * isolated_frac / (1.0 - isolated_frac)))
    n = T + iso
    offs = np.zeros(components + 1, dtype=np.int64)
    np.cumsum(sizes, out=offs[1:])
    kt = key(seed, STREAM_FTREE)
    us, vs = [], []
    for c in range(components):
        off, s = int(offs[c]), int(sizes[c])
        j = np.arange(1, s, dtype=np.int64)
        if c % 2 == 0:
            par = j - 1
        else:
            par = (rnd(kt, (off + j).astype(np.uint64)) % j.astype(np.uint64)).astype(np.int64)
        us.append(off + par)
        vs.append(off + j)
    u = np.concatenate(us) if us else np.zeros(0, np.int64)
    v = np.concatenate(vs) if vs else np.zeros(0, np.int64)
    pk = key(seed, STREAM_PERM)
    u = permute_ids(u.astype(np.uint64), n, pk).astype(np.int64)
    v = permute_ids(v.astype(np.uint64), n, pk).astype(np.int64)
    return n, np.stack([u, v], axis=1)


# ---------------------------------------------------------------- ingestion
INGEST_TEXT_CASES = ("edgelist_sparse", "edgelist_dense", "edgelist_err_nonint",
                     "edgelist_err_tokens", "edgelist_err_negative", "mtx_symmetric_real",
                     "mtx_general_pattern", "mtx_err_range", "mtx_err_count")


def ingest_text(case: str, seed: int = 1, lines: int = 60_000) -> str:
    """Seeded edge-list / Matrix Market text for the ingestion parity
    fixtures (tests/golden/ingest_large.json): comment and blank lines, tabs,
    CRLF endings, '+' signs, '_' digit grouping, leading zeros, reversed and
    repeated pairs, self-loops, no trailing newline; the error cases place one
    malformed line at a seeded position."""
    rng = np.random.default_rng([seed, INGEST_TEXT_CASES.index(case)])
    mtx = case.startswith("mtx")
    if case == "edgelist_sparse":
        pool = np.unique(rng.integers(0, 10**12, size=lines // 2))
    elif mtx:
        pool = np.arange(1, 40_001)
    else:
        pool = np.arange(0, lines // 3)
    u = pool[rng.integers(0, pool.size, size=lines)]
    v = pool[rng.integers(0, pool.size, size=lines)]
    dup = rng.random(lines) < 0.1
    u[dup], v[dup] = np.roll(v, 1)[dup], np.roll(u, 1)[dup]
    loops = rng.random(lines) < 0.01
    v[loops] = u[loops]

    def tok(x: int, r: float) -> str:
        if r < 0.03:
            return "+" + str(x)
        if r < 0.05 and x >= 1000:
            s = str(x)
            return s[:-3] + "_" + s[-3:]
        if r < 0.07:
            return "00" + str(x)
        return str(x)

    out = []
    if mtx:
        field = "real" if case == "mtx_symmetric_real" else "pattern"
        sym = "symmetric" if case == "mtx_symmetric_real" else "general"
        out.append(f"%%MatrixMarket matrix coordinate {field} {sym}")
        out.append("% generated by oracle/gen.py ingest_text")
        declared = lines + (1 if case == "mtx_err_count" else 0)
        out.append(f"{pool.size} {pool.size} {declared}")
    r = rng.random((lines, 4))
    for i in range(lines):
        if not mtx and r[i, 3] < 0.02:
            out.append("# comment " + str(i))
        if r[i, 3] > 0.99:
            out.append("")
        if mtx and r[i, 3] < 0.01:
            out.append("% note")
        sep = "\t" if r[i, 2] < 0.1 else (" " * (1 + int(r[i, 2] * 3)))
        line = tok(int(u[i]), r[i, 0]) + sep + tok(int(v[i]), r[i, 1])
        if case == "mtx_symmetric_real":
            line += f" {r[i, 2]:.4f}"
        if r[i, 2] > 0.95:
            line = "  " + line + " \r"
        out.append(line)
    bad = {"edgelist_err_nonint": "12 x7", "edgelist_err_tokens": "1 2 3",
           "edgelist_err_negative": "5 -3", "mtx_err_range": f"1 {pool.size + 1}"}
    if case in bad:
        pos = int(rng.integers(len(out) // 2, len(out)))
        out.insert(pos, bad[case])
    text = "\n".join(out)
    return text if int(rng.integers(0, 2)) else text + "\n"
