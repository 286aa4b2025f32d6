"""Pins of the CPU oracle (oracle/oracle.c) to things other than itself.

Each test names what fixes the expected value: a worked example printed in the
reference (tests/golden), an independent algorithm from the paper (Eq. 1-2 by
path enumeration, the minimax Floyd-Warshall variant, the MST-path property),
a library special case (scipy single linkage + cophenet), exact rational
arithmetic, or an invariant of the mathematics.  CPU only.
"""
import itertools
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from synth import generators as G

GOLD = os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def assert_bit_equal(a, b):
    a = np.asarray(a, np.float32)
    b = np.asarray(b, np.float32)
    assert a.shape == b.shape
    # canonical +0 everywhere on both sides (reading Q5): compare bits exactly
    diff = np.nonzero(bits(a) != bits(b))
    assert diff[0].size == 0, f"{diff[0].size} mismatches, first at {diff[0][0]},{diff[1][0] if len(diff) > 1 else ''}: {a[tuple(x[0] for x in diff)]} vs {b[tuple(x[0] for x in diff)]}"


REGIMES = ["uniform", "ties", "ints255", "negative", "signed_zero"]


# --------------------------------------------------------------------------
# worked examples printed in the reference
# --------------------------------------------------------------------------
def test_worked_examples_weights():
    g = json.load(open(GOLD))
    for c in g["cases"]:
        W = np.array(c["W"], np.float32)
        M = oracle.appd_weights(W, c["sense"])
        assert_bit_equal(M, np.array(c["M"], np.float32))
        assert_bit_equal(oracle.floyd(W, c["sense"]), np.array(c["M"], np.float32))
        if W.shape[0] <= 9:
            assert_bit_equal(oracle.brute(W, c["sense"]), np.array(c["M"], np.float32))
        if "mst" in c:
            eu, ev, ew = oracle.prim_weights(W, 1)
            got = sorted((min(u, v), max(u, v), float(w)) for u, v, w in zip(eu, ev, ew))
            assert got == sorted((a, b, float(w)) for a, b, w in c["mst"])


def test_worked_examples_points():
    g = json.load(open(GOLD))
    for c in g["points"]:
        X = np.array(c["X"], np.float32)
        assert_bit_equal(oracle.points_weights(X), np.array(c["W"], np.float32))
        assert_bit_equal(oracle.appd_points(X), np.array(c["M"], np.float32))


def test_write_counts_printed():
    g = json.load(open(GOLD))
    for c in g["write_counts"]:
        W = G.random_weights(c["n"], 3, "uniform")
        _, st = oracle.appd_weights(W, 1, with_stats=True)
        assert st["writes"] == c["writes"]


# --------------------------------------------------------------------------
# Eq. 1-2 by path enumeration (the definition itself)
# --------------------------------------------------------------------------
def _py_brute(W, sense):
    """Eq. 1-2 transcribed in Python over itertools.permutations (n <= 6)."""
    n = W.shape[0]
    M = np.zeros((n, n), np.float32)
    for i in range(n):
        for j in range(n):
            if i == j:
                continue
            others = [k for k in range(n) if k not in (i, j)]
            phi = []
            for r in range(len(others) + 1):
                for mid in itertools.permutations(others, r):
                    p = (i, *mid, j)
                    ws = [W[p[t], p[t + 1]] + np.float32(0) for t in range(len(p) - 1)]
                    phi.append(max(ws) if sense > 0 else min(ws))
            M[i, j] = min(phi) if sense > 0 else max(phi)
    return M


def test_c_brute_equals_python_brute():
    """The C path enumerator is itself checked against an itertools transcription of Eq. 1-2."""
    for n in range(1, 7):
        for seed in range(4):
            for kind in REGIMES:
                W = G.random_weights(n, seed, kind)
                for sense in (1, -1):
                    assert_bit_equal(oracle.brute(W, sense), _py_brute(W, sense))


@pytest.mark.parametrize("kind", REGIMES + ["huge"])
def test_algo4_equals_brute_force(kind):
    """Algorithm 4 == Eq. 2 on every n <= 8 (50 seeds at n = 8)."""
    for n in range(1, 9):
        seeds = range(50) if n == 8 else range(8)
        for seed in seeds:
            W = G.random_weights(n, seed, kind)
            for sense in (1, -1):
                want = oracle.brute(W, sense)
                assert_bit_equal(oracle.appd_weights(W, sense), want)
                assert_bit_equal(oracle.floyd(W, sense), want)


# --------------------------------------------------------------------------
# the paper's O(n^3) Floyd-Warshall variant and the MST-path property
# --------------------------------------------------------------------------
def test_algo4_equals_floyd_and_mst_path_200_seeds():
    """>= 200 seeded graphs, n in 2..64, both senses, bit-exact."""
    rs = np.random.default_rng(7)
    for seed in range(200):
        n = int(rs.integers(2, 65))
        kind = REGIMES[seed % len(REGIMES)]
        W = G.random_weights(n, seed, kind)
        for sense in (1, -1):
            assert_bit_equal(oracle.appd_weights(W, sense), oracle.floyd(W, sense))
        assert_bit_equal(oracle.appd_weights(W, 1), oracle.mst_path(W))


def test_c1_equals_floyd():
    W = G.config("C1")
    assert_bit_equal(oracle.appd_weights(W), oracle.floyd(W))


def test_mst_path_large():
    for n, kind in [(300, "uniform"), (700, "ties"), (1024, "negative")]:
        W = G.random_weights(n, 11, kind)
        assert_bit_equal(oracle.appd_weights(W), oracle.mst_path(W))


# --------------------------------------------------------------------------
# library special case: single linkage dendrogram read-off
# --------------------------------------------------------------------------
def _scipy_appd(W):
    from scipy.cluster.hierarchy import cophenet, linkage
    from scipy.spatial.distance import squareform

    Wd = np.asarray(W, np.float64).copy()
    np.fill_diagonal(Wd, 0.0)
    Z = linkage(squareform(Wd, checks=False), method="single")
    return squareform(cophenet(Z)).astype(np.float32)


@pytest.mark.parametrize("kind", ["uniform", "ties", "ints255"])
def test_scipy_single_linkage_cophenet(kind):
    for seed, n in [(0, 50), (1, 200), (2, 513)]:
        W = G.random_weights(n, seed, kind)
        assert_bit_equal(oracle.appd_weights(W), _scipy_appd(W))


def test_scipy_on_configs_c1_c2():
    W = G.config("C1")
    assert_bit_equal(oracle.appd_weights(W), _scipy_appd(W))
    X = G.config("C2")
    assert_bit_equal(oracle.appd_points(X), _scipy_appd(oracle.points_weights(X)))


# --------------------------------------------------------------------------
# invariants of the mathematics
# --------------------------------------------------------------------------
def check_invariants(W, M, sense=1, triples=None):
    n = W.shape[0]
    Wc = np.where(W == 0, np.float32(0), W).astype(np.float32)
    assert (bits(M) == bits(M.T)).all(), "symmetry"
    assert (bits(np.diag(M)) == 0).all(), "+0 diagonal"
    off = ~np.eye(n, dtype=bool)
    if sense > 0:
        assert (M[off] <= Wc[off]).all(), "M <= W"
    else:
        assert (M[off] >= Wc[off]).all(), "M >= W (widest)"
    eu, ev, ew = oracle.prim_weights(W, sense)
    vals = np.unique(M[off]) if n > 1 else np.array([], np.float32)
    assert len(vals) <= max(n - 1, 0)
    assert np.isin(vals, ew).all(), "every value is an MST edge weight"
    if n <= 128:
        # all triples: ultrametric M[i][j] <= max(M[i][k], M[k][j])  (dual for widest)
        # the diagonal is the empty path (-inf for minimax, +inf for widest); exclude it
        Mx = M.copy()
        np.fill_diagonal(Mx, -np.inf if sense > 0 else np.inf)
        for i in range(n):
            if sense > 0:
                bound = np.maximum(Mx[i][:, None], Mx)  # [k, j]: max(M[i][k], M[k][j])
                assert (Mx[i][None, :] <= bound).all()
            else:
                bound = np.minimum(Mx[i][:, None], Mx)
                assert (Mx[i][None, :] >= bound).all()
    else:
        rs = np.random.default_rng(0)
        t = triples or 200000
        i, j, k = rs.integers(0, n, (3, t))
        ok = (i != j) & (j != k) & (i != k)
        i, j, k = i[ok], j[ok], k[ok]
        if sense > 0:
            assert (M[i, j] <= np.maximum(M[i, k], M[k, j])).all()
        else:
            assert (M[i, j] >= np.minimum(M[i, k], M[k, j])).all()


@pytest.mark.parametrize("kind", REGIMES)
def test_invariants_and_write_once(kind):
    for n in (2, 3, 10, 100, 1000):
        W = G.random_weights(n, n + 1, kind)
        for sense in (1, -1):
            M, st = oracle.appd_weights(W, sense, with_stats=True)
            check_invariants(W, M, sense)
            assert st["writes"] == n * (n - 1) // 2
            assert st["traversed"] <= n * (n - 1) // 2 + n - 1


def test_mst_weight_is_minimal_by_enumeration():
    """Prim (R2) against all spanning trees for n <= 6: same total weight, both senses."""
    for n in range(2, 7):
        for seed in range(6):
            W = G.random_weights(n, seed, "ties" if seed % 2 else "uniform")
            edges = [(i, j) for i in range(n) for j in range(i + 1, n)]
            best_min, best_max = np.inf, -np.inf
            for sub in itertools.combinations(range(len(edges)), n - 1):
                parent = list(range(n))

                def find(x):
                    while parent[x] != x:
                        x = parent[x]
                    return x

                ok = True
                for e in sub:
                    a, b = find(edges[e][0]), find(edges[e][1])
                    if a == b:
                        ok = False
                        break
                    parent[a] = b
                if ok:
                    tot = sum(float(W[edges[e]]) for e in sub)
                    best_min = min(best_min, tot)
                    best_max = max(best_max, tot)
            _, _, ew = oracle.prim_weights(W, 1)
            assert abs(float(np.sum(ew.astype(np.float64))) - best_min) < 1e-9
            _, _, ew = oracle.prim_weights(W, -1)
            assert abs(float(np.sum(ew.astype(np.float64))) - best_max) < 1e-9


# --------------------------------------------------------------------------
# metamorphic identities
# --------------------------------------------------------------------------
def test_permutation_equivariance_with_ties():
    """relabelling invariance under ties, 50 seeds, n <= 32 (+ larger)."""
    for seed in range(50):
        n = 2 + seed % 31
        W = G.random_weights(n, seed, "ties")
        p = np.random.default_rng(seed).permutation(n)
        M = oracle.appd_weights(W)
        Mp = oracle.appd_weights(W[np.ix_(p, p)])
        assert_bit_equal(Mp, M[np.ix_(p, p)])
    X = G.random_points(300, 3, 1, "grid")
    p = np.random.default_rng(1).permutation(300)
    assert_bit_equal(oracle.appd_points(X[p]), oracle.appd_points(X)[np.ix_(p, p)])


def test_idempotence_and_monotone_commutation():
    for seed in range(30):
        n = 5 + seed * 3
        W = G.random_weights(n, seed, REGIMES[seed % len(REGIMES)])
        M = oracle.appd_weights(W)
        assert_bit_equal(oracle.appd_weights(M), M)  # APPD of an ultrametric is itself
        for f in (lambda a: np.floor(a), lambda a: a * np.float32(2), lambda a: np.minimum(a, np.float32(1))):
            fW = f(W).astype(np.float32)
            np.fill_diagonal(fW, 0)
            fM = f(M).astype(np.float32)
            np.fill_diagonal(fM, 0)
            assert_bit_equal(oracle.appd_weights(fW), fM + np.float32(0))


def test_widest_duality():
    """minimax(G) == -widest(-G) exactly (100 seeds, n <= 64); -0 canonicalised."""
    rs = np.random.default_rng(3)
    for seed in range(100):
        n = int(rs.integers(2, 65))
        W = G.random_weights(n, seed, REGIMES[seed % len(REGIMES)])
        a = oracle.appd_weights(W, 1)
        b = -oracle.appd_weights(-W, -1) + np.float32(0)
        assert_bit_equal(a, b)


def test_points_mode_equals_weights_mode_on_r1_weights():
    for kind in ("uniform", "blobs", "dups", "grid", "wide"):
        X = G.random_points(257, 5, 2, kind)
        assert_bit_equal(oracle.appd_points(X), oracle.appd_weights(oracle.points_weights(X)))


def test_sqrt_commutation_points():
    """Monotone commutation with f = sqrtf (App. A.4): APPD(sqrt(d2)) == sqrt(APPD(d2))."""
    for kind in ("uniform", "grid", "dups"):
        X = G.random_points(200, 4, 5, kind)
        W = oracle.points_weights(X)
        D2 = np.empty_like(W)
        for i in range(200):
            for j in range(200):
                D2[i, j] = oracle.r1_dist2(X[i], X[j]) if i != j else 0
        assert_bit_equal(np.sqrt(oracle.appd_weights(D2)), oracle.appd_weights(W))


def test_row_window_r5_equals_full():
    X = G.random_points(500, 3, 9, "dups")
    M = oracle.appd_points(X)
    for r0, R in [(0, 1), (0, 500), (123, 77), (499, 1)]:
        assert_bit_equal(oracle.appd_points_rows(X, r0, R), M[r0:r0 + R])
    W = G.random_weights(300, 4, "negative")
    Mw = oracle.appd_weights(W)
    assert_bit_equal(oracle.appd_weights_rows(W, 100, 50), Mw[100:150])


# --------------------------------------------------------------------------
# R1 weights: exact rational emulation of the pinned fmaf chain, fp64 bound
# --------------------------------------------------------------------------
def round_f32(q: Fraction) -> np.float32:
    """Round an exact rational to the nearest fp32, ties to even (IEEE-754 RN)."""
    if q == 0:
        return np.float32(0.0)
    s = -1 if q < 0 else 1
    a = abs(q)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    e = max(e, -126)
    ulp = Fraction(2) ** (e - 23)
    k = a / ulp
    fl = k.numerator // k.denominator
    rem = k - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return np.float32(s * float(fl * ulp))


def r1_exact(xi, xj):
    acc = Fraction(0)
    for a, b in zip(xi, xj):
        t = round_f32(Fraction(float(a)) - Fraction(float(b)))
        acc = Fraction(float(round_f32(Fraction(float(t)) * Fraction(float(t)) + acc)))
    return np.float32(float(acc))


def test_r1_matches_exact_rational_fma_chain():
    rs = np.random.default_rng(5)
    for trial in range(300):
        d = int(rs.integers(1, 9))
        scale = 10.0 ** rs.integers(-6, 6)
        xi = (rs.standard_normal(d) * scale).astype(np.float32)
        xj = (rs.standard_normal(d) * scale).astype(np.float32)
        assert bits(oracle.r1_dist2(xi, xj)) == bits(r1_exact(xi, xj))


def test_r1_double_rounding_case():
    """The fmaf step must round once.  Constructed case (search in DESIGN.md notes):
    t0 = 2047 * 2^-27 (t0^2 exact in fp32), t = 0x1.000ff8p+0: t^2 + t0^2 lies 2^-54
    above an fp32 midpoint whose lower neighbour is even.  A single rounding goes up;
    an fp64 emulation fl32(fl64(t*t + acc)) lands on the midpoint and goes down."""
    t0 = float.fromhex("0x1.ffcp-17")
    t = float.fromhex("0x1.000ff8p+0")
    exact = round_f32(Fraction(t) ** 2 + Fraction(t0) ** 2)
    emulated = np.float32(np.float64(t) * np.float64(t) + np.float64(np.float32(t0 * t0)))
    assert bits(exact) != bits(emulated)
    xi = np.array([t0, t], np.float32)
    xj = np.zeros(2, np.float32)
    assert bits(oracle.r1_dist2(xi, xj)) == bits(exact)
    assert bits(oracle.r1_dist2(xj, xi)) == bits(exact)


def test_r1_symmetry_zero_and_fp64_bound():
    for name, X in [("C2", G.config("C2")), ("C4s", G.config("C4", n=512)), ("C5s", G.config("C5", n=2048))]:
        n, d = X.shape
        rs = np.random.default_rng(1)
        rows = rs.integers(0, n, 64)
        Wb = oracle.points_weights(X, 0, n)[rows] if n <= 4096 else np.stack(
            [oracle.points_weights(X, int(r), 1)[0] for r in rows])
        bound = (d / 2 + 2) * 2.0 ** -24
        worst = 0.0
        for t, r in enumerate(rows):
            ref = np.sqrt(((X[r].astype(np.float64) - X.astype(np.float64)) ** 2).sum(1))
            got = Wb[t].astype(np.float64)
            nz = ref > 0
            assert (got[~nz] == 0).all()
            rel = np.abs(got[nz] - ref[nz]) / ref[nz]
            worst = max(worst, rel.max(initial=0))
            # symmetry, bitwise
            for c in rs.integers(0, n, 16):
                assert bits(oracle.r1_weight(X[r], X[c])) == bits(oracle.r1_weight(X[c], X[r]))
        assert worst <= bound and worst <= 1e-5, (name, worst, bound)


def test_dist_f64_exact_small():
    assert oracle.dist_f64(np.array([0, 0], np.float32), np.array([3, 4], np.float32)) == 5.0
    assert oracle.r1_weight(np.array([1, 2, 2], np.float32), np.zeros(3, np.float32)) == 3.0


# --------------------------------------------------------------------------
# NEXT-3: pluggable point metrics (Manhattan, Chebyshev)
# --------------------------------------------------------------------------
def _int_points(n, d, seed, lo=-50, hi=50):
    rs = np.random.default_rng(seed)
    return rs.integers(lo, hi + 1, size=(n, d)).astype(np.float32)


@pytest.mark.parametrize("metric", [1, 2])
def test_metric_points_equal_weights_path_on_integer_points(metric):
    """Integer coordinates make every fp32 operation of L1 / L-inf exact, so the weight
    matrix is fixed by integer arithmetic (numpy int64) independently of the oracle's
    metric code; the points path must then equal Algorithm 4 on that W, and the
    minimax Floyd-Warshall variant on it."""
    for t, (n, d) in enumerate([(2, 1), (3, 2), (7, 3), (40, 2), (200, 5), (333, 8)]):
        X = _int_points(n, d, 60 + t)
        D = np.abs(X[:, None, :].astype(np.int64) - X[None, :, :].astype(np.int64))
        W = (D.sum(-1) if metric == 1 else D.max(-1)).astype(np.float32)
        np.fill_diagonal(W, 0.0)
        assert_bit_equal(oracle.points_weights(X, metric=metric), W)
        M = oracle.appd_points(X, metric=metric)
        assert_bit_equal(M, oracle.appd_weights(W))
        if n <= 64:
            assert_bit_equal(M, oracle.floyd(W))
        if n <= 7:
            assert_bit_equal(M, oracle.brute(W))


def test_metric_worked_example():
    """(0,0), (2,2), (4,0): Manhattan distances 4, 4, 4; Chebyshev 2, 4, 2; Euclidean
    sqrt 8, 4, sqrt 8 -> every off-diagonal APPD entry is 4, 2 and sqrtf(8)."""
    X = np.array([[0, 0], [2, 2], [4, 0]], np.float32)
    off = ~np.eye(3, dtype=bool)
    for metric, want in [(1, 4.0), (2, 2.0), (0, float(np.sqrt(np.float32(8.0))))]:
        M = oracle.appd_points(X, metric=metric)
        assert (M[off] == np.float32(want)).all(), (metric, M)
        assert (bits(np.diag(M)) == 0).all()


def test_metrics_coincide_in_one_dimension():
    """d = 1: |x - y| for all three metrics (sqrtf of a correctly rounded square of t is
    |t| in round-to-nearest without overflow or underflow)."""
    rs = np.random.default_rng(5)
    X = (rs.standard_normal((150, 1)) * 10).astype(np.float32)
    M0 = oracle.appd_points(X)
    for metric in (1, 2):
        assert_bit_equal(oracle.appd_points(X, metric=metric), M0)


def test_overflowing_distances_are_infinite_edges():
    """Reading Q14: points whose squared distance overflows fp32 are joined by an edge of
    weight +inf (the graph is complete).  Closed form: the ordinary half keeps
    its own APPD, every entry across the halves and between huge points is +inf."""
    rs = np.random.default_rng(8)
    X = (rs.standard_normal((120, 5)) * 1e20).astype(np.float32)
    X[:60] *= np.float32(1e-20)
    M = oracle.appd_points(X)
    assert_bit_equal(M[:60, :60], oracle.appd_points(X[:60]))
    assert np.isinf(M[:60, 60:]).all() and np.isinf(M[60:, :60]).all()
    off = ~np.eye(60, dtype=bool)
    assert np.isinf(M[60:, 60:][off]).all() and (bits(np.diag(M)) == 0).all()


# --------------------------------------------------------------------------
# NEXT-3: fp64 weights.  Pinned to an independent algorithm written here (the
# minimax / widest closure of Floyd-Warshall, P:L44 / S:L235, in numpy float64), to a
# three-vertex case whose answer is fixed by Eq. 1-2 by hand, and to the pinned fp32
# oracle on fp32-representable inputs.
# --------------------------------------------------------------------------
def floyd_closure_f64(W, sense):
    M = np.where(W == 0, 0.0, W).astype(np.float64)
    n = M.shape[0]
    for k in range(n):
        via = np.maximum(M[:, k:k + 1], M[k:k + 1, :]) if sense > 0 else np.minimum(M[:, k:k + 1], M[k:k + 1, :])
        M = np.minimum(M, via) if sense > 0 else np.maximum(M, via)
    np.fill_diagonal(M, 0.0)
    return M


def assert_f64_bit_equal(a, b):
    a = np.asarray(a, np.float64) + 0.0  # canonical +0 (reading Q5)
    b = np.asarray(b, np.float64) + 0.0
    assert a.shape == b.shape
    bad = np.nonzero(a.view(np.uint64) != b.view(np.uint64))
    assert bad[0].size == 0, f"{bad[0].size} mismatches, first at {bad[0][0]},{bad[1][0]}: {a[bad[0][0], bad[1][0]]!r} vs {b[bad[0][0], bad[1][0]]!r}"


@pytest.mark.parametrize("kind", ["uniform", "fine_ties", "negative", "signed_zero", "huge"])
@pytest.mark.parametrize("sense", [1, -1])
def test_f64_equals_floyd_closure(kind, sense):
    for seed in range(4):
        W = G.random_weights_f64(37 + 5 * seed, seed, kind)
        assert_f64_bit_equal(oracle.appd_weights_f64(W, sense), floyd_closure_f64(W, sense))


def test_f64_three_vertex_by_hand():
    # Eq. 1-2: the path 0-2-1 has max edge 1 + 2^-41 < 1 + 2^-40 = w01, so d(0,1) = 1 + 2^-41;
    # in fp32 every weight here rounds to 1.0 (a plausible truncation would give 1.0)
    a, b = 1.0 + 2.0 ** -40, 1.0 + 2.0 ** -41
    W = np.array([[0, a, b], [a, 0, 1.0], [b, 1.0, 0]], np.float64)
    M = oracle.appd_weights_f64(W, 1)
    assert M[0, 1] == b and M[1, 0] == b and M[0, 2] == b and M[1, 2] == 1.0
    Mw = oracle.appd_weights_f64(W, -1)  # widest: best bottleneck between 0 and 1 is the edge itself
    assert Mw[0, 1] == a and Mw[1, 2] == b and Mw[0, 2] == b
    eu, ev, ew = oracle.prim_weights_f64(W, 1)
    assert sorted(ew.tolist()) == [1.0, b]


@pytest.mark.parametrize("kind", REGIMES)
def test_f64_equals_f32_on_representable_inputs(kind):
    W = G.random_weights(48, 7, kind)
    M32 = oracle.appd_weights(W, 1)
    M64 = oracle.appd_weights_f64(W.astype(np.float64), 1)
    assert_f64_bit_equal(M64, M32.astype(np.float64))


# --------------------------------------------------------------------------
# round 2 pins: the L1 / L-inf chains on non-integer inputs (exact rational
# arithmetic), and Prim (R2) against an independent Kruskal (no oracle code)
# --------------------------------------------------------------------------
def _metric_pair(xi, xj, metric):
    X = np.stack([xi, xj]).astype(np.float32)
    return oracle.points_weights(X, metric=metric)[0, 1]


def l1_exact(xi, xj):
    """S:L80 / DESIGN Q6 (metric 1): acc = +0; acc = fl32(acc + |fl32(x_k - y_k)|), k in order."""
    acc = Fraction(0)
    for a, b in zip(xi, xj):
        t = abs(Fraction(float(round_f32(Fraction(float(a)) - Fraction(float(b))))))
        acc = Fraction(float(round_f32(acc + t)))
    return np.float32(float(acc))


def linf_exact(xi, xj):
    """metric 2: max over k of |fl32(x_k - y_k)| (a max of exactly rounded differences)."""
    return np.float32(max(float(abs(Fraction(float(round_f32(Fraction(float(a)) - Fraction(float(b)))))))
                          for a, b in zip(xi, xj)))


def test_l1_matches_exact_rational_chain():
    """300 random non-integer cases across magnitudes: every fp32 subtraction and every
    partial sum rounds, so a double accumulator, a different summation order or an
    unrounded difference changes some result bit."""
    rs = np.random.default_rng(77)
    for trial in range(300):
        d = int(rs.integers(1, 17))
        scale = 10.0 ** rs.integers(-5, 6)
        xi = (rs.standard_normal(d) * scale).astype(np.float32)
        xj = (rs.standard_normal(d) * scale * (10.0 ** rs.integers(-2, 3))).astype(np.float32)
        assert bits(_metric_pair(xi, xj, 1)) == bits(l1_exact(xi, xj)), (trial, xi, xj)
        assert bits(_metric_pair(xj, xi, 1)) == bits(l1_exact(xj, xi))


def test_l1_order_sensitive_case():
    """A case where the summation order decides the result: 1 + 2^-24 + 2^-24 is 1 in
    k order (each add ties to even) but 1 + 2^-23 if the small terms were summed first."""
    xi = np.array([1.0, 2.0 ** -24, 2.0 ** -24], np.float32)
    xj = np.zeros(3, np.float32)
    assert _metric_pair(xi, xj, 1) == np.float32(1.0)
    assert bits(l1_exact(xi, xj)) == bits(np.float32(1.0))
    xr = xi[::-1].copy()
    assert _metric_pair(xr, xj, 1) == np.float32(1.0 + 2.0 ** -23)


def test_linf_matches_exact_rational_max():
    rs = np.random.default_rng(78)
    for trial in range(300):
        d = int(rs.integers(1, 17))
        scale = 10.0 ** rs.integers(-5, 6)
        xi = (rs.standard_normal(d) * scale).astype(np.float32)
        xj = (rs.standard_normal(d) * scale * (10.0 ** rs.integers(-2, 3))).astype(np.float32)
        assert bits(_metric_pair(xi, xj, 2)) == bits(linf_exact(xi, xj)), (trial, xi, xj)
    # the rounded difference, not |x| - |y| or an fp64 difference: 1 - (-2^-30) rounds to 1
    assert _metric_pair(np.array([1.0], np.float32), np.array([-(2.0 ** -30)], np.float32), 2) == np.float32(1.0)


def kruskal_numpy(W):
    """Kruskal's algorithm written here (not in oracle/): edges by (weight, i, j), union-find."""
    n = W.shape[0]
    iu, ju = np.triu_indices(n, 1)
    order = np.lexsort((ju, iu, W[iu, ju].astype(np.float64)))
    parent = list(range(n))

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    tree = []
    for e in order:
        a, b = find(int(iu[e])), find(int(ju[e]))
        if a != b:
            parent[a] = b
            tree.append((int(iu[e]), int(ju[e]), W[iu[e], ju[e]]))
    return tree


def tree_path_appd(n, tree):
    """APPD by the MST-path property: the largest weight on each tree path (numpy BFS)."""
    adj = [[] for _ in range(n)]
    for u, v, w in tree:
        adj[u].append((v, w))
        adj[v].append((u, w))
    M = np.zeros((n, n), np.float32)
    for s in range(n):
        seen = np.zeros(n, bool)
        seen[s] = True
        stack = [(s, np.float32(-np.inf))]
        while stack:
            x, mx = stack.pop()
            for y, w in adj[x]:
                if not seen[y]:
                    seen[y] = True
                    m2 = max(mx, w)
                    M[s, y] = m2
                    stack.append((y, m2))
    return M


@pytest.mark.parametrize("kind", ["uniform", "ties", "ints255", "negative"])
def test_prim_against_independent_kruskal(kind):
    """R2 (Prim) pinned without going through oracle code twice: Prim's n-1 edges
    form a spanning tree of W's own entries whose sorted weight multiset equals an
    independent Kruskal's (all MSTs share it), and Algorithm 4 equals the path maxima of
    the Kruskal tree -- so an error in prim() shared by the oracle's MST-path
    checker cannot hide."""
    for t, n in enumerate([2, 3, 5, 9, 17, 33, 64]):
        W = G.random_weights(n, 900 + t, kind)
        eu, ev, ew = oracle.prim_weights(W, 1)
        assert len(ew) == n - 1
        parent = list(range(n))

        def find(x):
            while parent[x] != x:
                x = parent[x]
            return x

        for u, v, w in zip(eu, ev, ew):
            assert u != v and bits(np.float32(w) + np.float32(0)) == bits(W[u, v] + np.float32(0))
            a, b = find(int(u)), find(int(v))
            assert a != b, "Prim closed a cycle"
            parent[a] = b
        kt = kruskal_numpy(W)
        assert sorted(float(x) for x in ew) == sorted(float(w) for _, _, w in kt)
        assert_bit_equal(oracle.appd_weights(W), tree_path_appd(n, kt) + np.float32(0))


# --------------------------------------------------------------------------
# fault injection: the checks that pin results must catch a corrupted APPD --
# one entry changed to another MST weight, one merge height changed, two leaves swapped
# in the leaf order -- so a GPU fault of that shape cannot pass as parity
# --------------------------------------------------------------------------
def _fill_from_dendrogram(pi, h, sense=1):
    """M[pi_a][pi_b] = max (min for widest) of h[a..b-1] -- the fill's identity (App. A.2)."""
    n = len(pi)
    M = np.zeros((n, n), np.float32)
    for a in range(n):
        run = np.float32(-np.inf if sense > 0 else np.inf)
        for b in range(a + 1, n):
            run = max(run, h[b - 1]) if sense > 0 else min(run, h[b - 1])
            M[pi[a], pi[b]] = M[pi[b], pi[a]] = run
    return M


def test_corruptions_are_caught():
    W = G.random_weights(40, 77, "uniform")
    M = oracle.appd_weights(W)
    check_invariants(W, M)
    # the leaf-order identity reproduces the oracle from a Prim order (App. A.3) ...
    eu, ev, ew = oracle.prim_weights(W, 1)
    order = [0] + [int(v) for v in ev]
    pi = np.array(order, np.int32)
    h = np.array(ew, np.float32)
    assert (bits(_fill_from_dendrogram(pi, h)) == bits(M)).all()
    # ... and each corruption below changes bits that parity compares, or breaks an invariant
    bad = M.copy()
    i, j = 3, 17
    other = np.float32(ew[(np.searchsorted(np.sort(ew), M[i, j]) + 1) % len(ew)])
    bad[i, j] = bad[j, i] = other  # another MST weight, still symmetric: parity sees it
    assert (bits(bad) != bits(M)).any()
    one_sided = M.copy()
    one_sided[i, j] = other  # a one-sided write: the invariants see it without the oracle
    with pytest.raises(AssertionError):
        check_invariants(W, one_sided)
    h2 = h.copy()
    h2[10] = np.float32(h2[10] * 0.5)  # one merge height
    assert (bits(_fill_from_dendrogram(pi, h2)) != bits(M)).any()
    pi2 = pi.copy()
    pi2[[5, 30]] = pi2[[30, 5]]  # two leaves swapped
    assert (bits(_fill_from_dendrogram(pi2, h)) != bits(M)).any()


def test_oracle_under_sanitizers(tmp_path):
    """The oracle's C code under -fsanitize=address,undefined: Algorithm 4, the row windows,
    Floyd, brute force and the points path on small inputs, checked against each other
    (tests/oracle_san_main.c); any out-of-bounds access or UB aborts the run."""
    import subprocess

    here = os.path.dirname(os.path.abspath(__file__))
    exe = tmp_path / "oracle_san"
    cmd = ["gcc", "-O1", "-g", "-std=c11", "-ffp-contract=off", "-mfma", "-fsanitize=address,undefined",
           "-fno-sanitize-recover=all", os.path.join(here, "oracle_san_main.c"),
           os.path.join(os.path.dirname(here), "oracle", "oracle.c"), "-lm", "-o", str(exe)]
    subprocess.check_call(cmd)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ok" in out.stdout
