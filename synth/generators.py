"""Seeded generators for the five BASELINE.json configurations and for test inputs.

Conventions (SPEC S:L339 names splitmix64):
  * draw i (0-based) of stream ``seed`` is splitmix64 output number i+1, i.e.
    z = seed + (i+1)*0x9E3779B97F4A7C15 (mod 2^64) followed by the two
    xor-shift-multiply rounds.  The stream is counter based, so it vectorises.
  * u53  = (z >> 11) * 2^-53                        fp64 in [0, 1)
  * u24  = (z >> 40) * 2^-24                        fp32 in [0, 1), exact
  * open = ((z >> 41) * 2 + 1) * 2^-24              fp32 in (0, 1), exact
  * bounded(m) = ((z >> 32) * m) >> 32              integer in [0, m)
  * N()  = sqrt(-2 ln(1 - u53)) * cos(2 pi u53)     two fresh draws, no caching
  * Fisher-Yates: for i = n-1 .. 1: swap(i, bounded(i+1))

``ln`` and ``cos`` are evaluated with plain +,-,*,/ series (below) rather than
libm or numpy's SIMD transcendental kernels, so the bytes are identical on any
IEEE-754 machine (the GPU box's host included).  All values are computed in
fp64 and rounded once to fp32.
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
LN2 = 0.6931471805599453
TWO_PI = 6.283185307179586


def splitmix_block(seed: int, start: int, count: int) -> np.ndarray:
    """Draws start .. start+count-1 of the splitmix64 stream seeded with ``seed``."""
    i = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + i * GAMMA
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


class SplitMix64:
    """Sequential cursor over the counter-based stream."""

    def __init__(self, seed: int):
        self.seed = int(seed)
        self.pos = 0

    def raw(self, count: int) -> np.ndarray:
        z = splitmix_block(self.seed, self.pos, count)
        self.pos += count
        return z

    def u53(self, count: int) -> np.ndarray:
        return (self.raw(count) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)

    def u24(self, count: int) -> np.ndarray:
        return ((self.raw(count) >> np.uint64(40)).astype(np.float64) * (2.0 ** -24)).astype(np.float32)

    def open01(self, count: int) -> np.ndarray:
        z = self.raw(count) >> np.uint64(41)
        return ((z.astype(np.float64) * 2.0 + 1.0) * (2.0 ** -24)).astype(np.float32)

    def bounded(self, m: int, count: int) -> np.ndarray:
        z = self.raw(count) >> np.uint64(32)
        return ((z * np.uint64(m)) >> np.uint64(32)).astype(np.int64)

    def normal(self, count: int) -> np.ndarray:
        """count standard normals; each uses two consecutive draws (u1, u2)."""
        u = self.u53(2 * count).reshape(count, 2)
        return np.sqrt(-2.0 * det_log(1.0 - u[:, 0])) * det_cos2pi(u[:, 1])

    def shuffle_rows(self, a: np.ndarray) -> np.ndarray:
        n = a.shape[0]
        if n < 2:
            return a
        idx = np.arange(n)
        js = self.bounded_seq(n)
        for i in range(n - 1, 0, -1):
            j = js[n - 1 - i]
            idx[i], idx[j] = idx[j], idx[i]
        return a[idx]

    def bounded_seq(self, n: int) -> np.ndarray:
        """The n-1 Fisher-Yates draws bounded(i+1) for i = n-1 .. 1, in that order."""
        z = self.raw(n - 1) >> np.uint64(32)
        m = np.arange(n, 1, -1, dtype=np.uint64)  # i+1 for i = n-1..1
        return ((z * m) >> np.uint64(32)).astype(np.int64)


def det_log(x: np.ndarray) -> np.ndarray:
    """Natural log for x in (0, 1] with +,-,*,/ only (atanh series), fp64."""
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)  # x = m * 2^e, m in [0.5, 1)
    small = m < 0.7071067811865476
    m = np.where(small, m * 2.0, m)
    e = np.where(small, e - 1, e).astype(np.float64)
    s = (m - 1.0) / (m + 1.0)  # |s| <= 0.1716
    s2 = s * s
    acc = np.zeros_like(s)
    for k in range(15, -1, -1):  # sum_{k} s^(2k+1)/(2k+1), Horner in s^2
        acc = acc * s2 + 1.0 / (2 * k + 1)
    return e * LN2 + 2.0 * s * acc


def _cos_poly(t):
    t2 = t * t
    acc = np.zeros_like(t)
    for k in range(11, -1, -1):
        fact = 1.0
        for q in range(1, 2 * k + 1):
            fact *= q
        acc = acc * t2 + ((-1.0) ** k) / fact
    return acc


def _sin_poly(t):
    t2 = t * t
    acc = np.zeros_like(t)
    for k in range(11, -1, -1):
        fact = 1.0
        for q in range(1, 2 * k + 2):
            fact *= q
        acc = acc * t2 + ((-1.0) ** k) / fact
    return acc * t


def det_cos2pi(u: np.ndarray) -> np.ndarray:
    """cos(2 pi u) for u in [0, 1) with +,-,*,/ only, fp64."""
    u = np.asarray(u, dtype=np.float64)
    u = np.where(u > 0.5, 1.0 - u, u)  # cos(2pi u) = cos(2pi(1-u)); u in [0, 0.5]
    sign = np.where(u > 0.25, -1.0, 1.0)
    u = np.where(u > 0.25, 0.5 - u, u)  # u in [0, 0.25]
    use_sin = u > 0.125
    v = np.where(use_sin, 0.25 - u, u)  # v in [0, 0.125]; angle <= pi/4
    t = v * TWO_PI
    return sign * np.where(use_sin, _sin_poly(t), _cos_poly(t))


# ----------------------------------------------------------------------------
# The five BASELINE.json configurations
# ----------------------------------------------------------------------------

def _upper_to_symmetric(n: int, draw_row) -> np.ndarray:
    W = np.zeros((n, n), dtype=np.float32)
    for i in range(n - 1):
        W[i, i + 1:] = draw_row(i, n - 1 - i)
    W += W.T
    return W


def c1_weights(n: int = 256, seed: int = 0) -> np.ndarray:
    """C1: W[i][j] = W[j][i] = open(0,1) fp32 for i<j in row-major order; +0 diagonal."""
    rng = SplitMix64(seed)
    return _upper_to_symmetric(n, lambda i, c: rng.open01(c))


def c3_weights(n: int = 16384, seed: int = 2) -> np.ndarray:
    """C3: W = 1 + bounded(255) (integers 1..255 as fp32) for i<j row-major; +0 diagonal."""
    W = np.zeros((n, n), dtype=np.float32)
    rng = SplitMix64(seed)
    block = 256
    for i0 in range(0, n - 1, block):
        i1 = min(n - 1, i0 + block)
        counts = [n - 1 - i for i in range(i0, i1)]
        vals = (1 + rng.bounded(255, int(sum(counts)))).astype(np.float32)
        p = 0
        for i, c in zip(range(i0, i1), counts):
            W[i, i + 1:] = vals[p:p + c]
            p += c
    W += W.T
    return W


def c2_points(n: int = 4096, seed: int = 1) -> np.ndarray:
    """C2: 5 isotropic Gaussian blobs (centres U[-10,10]^2, sigma 0.8, equal sizes) + 5% U[-12,12]^2 noise."""
    rng = SplitMix64(seed)
    n_noise = int(round(0.05 * n))
    n_blob = n - n_noise
    sizes = [n_blob // 5 + (1 if k < n_blob % 5 else 0) for k in range(5)]
    centres = (-10.0 + 20.0 * rng.u53(10)).reshape(5, 2)
    pts = []
    for k in range(5):
        z = rng.normal(2 * sizes[k]).reshape(sizes[k], 2)
        pts.append(centres[k] + 0.8 * z)
    pts.append((-12.0 + 24.0 * rng.u53(2 * n_noise)).reshape(n_noise, 2))
    X = np.concatenate(pts).astype(np.float32)
    return rng.shuffle_rows(X)


def c4_points(n: int = 65536, d: int = 64, seed: int = 3, k: int = 32) -> np.ndarray:
    """C4: k-component Gaussian mixture, means N(0, 25 I), sigma_k ~ U[0.5, 2], weights Dirichlet(1)."""
    rng = SplitMix64(seed)
    mu = 5.0 * rng.normal(k * d).reshape(k, d)
    sigma = 0.5 + 1.5 * rng.u53(k)
    E = -det_log(1.0 - rng.u53(k))
    cdf = np.cumsum(E) / np.cumsum(E)[-1]
    per_point = 1 + 2 * d
    z = rng.raw(n * per_point).reshape(n, per_point)
    u = (z[:, 0] >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    comp = np.minimum(np.searchsorted(cdf, u, side="right"), k - 1)  # first kk with u < cdf[kk]
    uu = (z[:, 1:] >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    u1 = uu[:, 0::2]
    u2 = uu[:, 1::2]
    nz = np.sqrt(-2.0 * det_log(1.0 - u1)) * det_cos2pi(u2)
    X = mu[comp] + sigma[comp, None] * nz
    return X.astype(np.float32)


def c5_points(n: int = 131072, d: int = 16, seed: int = 4) -> np.ndarray:
    """C5: U[0,1]^d rows with 1% exact duplicate rows (zero-weight edges), then shuffled."""
    rng = SplitMix64(seed)
    n_dup = int(round(0.01 * n))
    n_base = n - n_dup
    base = rng.u24(n_base * d).reshape(n_base, d)
    src = rng.bounded(n_base, n_dup)
    X = np.concatenate([base, base[src]])
    return rng.shuffle_rows(X)


CONFIGS = {
    "C1": dict(mode="weights", n=256, seed=0, desc="weights U(0,1), n=256"),
    "C2": dict(mode="points", n=4096, d=2, seed=1, desc="points 5 blobs + 5% noise, n=4096, d=2"),
    "C3": dict(mode="weights", n=16384, seed=2, desc="weights integers 1..255, n=16384"),
    "C4": dict(mode="points", n=65536, d=64, seed=3, desc="points 32-GMM, n=65536, d=64"),
    "C5": dict(mode="points", n=131072, d=16, seed=4, desc="points U[0,1]^16 + 1% duplicates, n=131072"),
}


def config(name: str, n: int | None = None):
    """Input array of a configuration; ``n`` overrides the size (same recipe, smaller)."""
    c = CONFIGS[name]
    nn = c["n"] if n is None else n
    if name == "C1":
        return c1_weights(nn, c["seed"])
    if name == "C2":
        return c2_points(nn, c["seed"])
    if name == "C3":
        return c3_weights(nn, c["seed"])
    if name == "C4":
        return c4_points(nn, c["d"], c["seed"])
    if name == "C5":
        return c5_points(nn, c["d"], c["seed"])
    raise KeyError(name)


# ----------------------------------------------------------------------------
# Test inputs (parity and edge cases)
# ----------------------------------------------------------------------------

def random_weights(n: int, seed: int, kind: str = "uniform") -> np.ndarray:
    """Symmetric fp32 weight matrix with +0 diagonal.

    kinds: uniform (open (0,1)), ties (integers 1..4), ints255 (1..255),
    negative (integers -3..3, includes zeros and negatives), signed_zero
    (values in {-0, +0, 1, 2}; stored -0 entries exercise canonicalisation),
    huge (magnitudes spanning 1e-30 .. 1e30).
    """
    rng = SplitMix64(1000003 * seed + 17)
    if kind == "uniform":
        f = lambda i, c: rng.open01(c)
    elif kind == "ties":
        f = lambda i, c: (1 + rng.bounded(4, c)).astype(np.float32)
    elif kind == "ints255":
        f = lambda i, c: (1 + rng.bounded(255, c)).astype(np.float32)
    elif kind == "negative":
        f = lambda i, c: (rng.bounded(7, c) - 3).astype(np.float32)
    elif kind == "signed_zero":
        f = lambda i, c: (rng.bounded(3, c)).astype(np.float32)
    elif kind == "huge":
        f = lambda i, c: (10.0 ** (rng.u53(c) * 60.0 - 30.0)).astype(np.float32)
    else:
        raise KeyError(kind)
    W = _upper_to_symmetric(n, f)
    if kind == "signed_zero":
        zero = W == 0
        W[zero] = np.float32(-0.0)  # -0 both triangles (symmetric bitwise), diagonal too
    return W


def random_weights_f64(n: int, seed: int, kind: str = "uniform") -> np.ndarray:
    """Symmetric fp64 weight matrix with +0 diagonal (NEXT-3, S:L77 fp64 weights).

    kinds: uniform (u53 on [0, 1)), fine_ties (1 + k 2^-40 with k in 0..7: distinct in
    fp64, all one value in fp32, with ties), negative (integers -3..3 plus k 2^-45),
    signed_zero (values in {-0, +0, 1, 1 + 2^-50}), huge (magnitudes 1e-300 .. 1e300).
    """
    rng = SplitMix64(1000033 * seed + 29)
    W = np.zeros((n, n), dtype=np.float64)
    for i in range(n - 1):
        c = n - 1 - i
        if kind == "uniform":
            row = rng.u53(c)
        elif kind == "fine_ties":
            row = 1.0 + rng.bounded(8, c).astype(np.float64) * 2.0 ** -40
        elif kind == "negative":
            row = (rng.bounded(7, c).astype(np.float64) - 3.0) + rng.bounded(3, c).astype(np.float64) * 2.0 ** -45
        elif kind == "signed_zero":
            row = np.array([0.0, 0.0, 1.0, 1.0 + 2.0 ** -50])[rng.bounded(4, c)]
        elif kind == "huge":
            row = 10.0 ** (rng.u53(c) * 600.0 - 300.0)
        else:
            raise KeyError(kind)
        W[i, i + 1:] = row
    W += W.T
    if kind == "signed_zero":
        W[W == 0] = -0.0  # -0 both triangles (symmetric bitwise), diagonal too
    return W


def random_points(n: int, d: int, seed: int, kind: str = "uniform") -> np.ndarray:
    """n x d fp32 points.

    kinds: uniform (u24), blobs (Gaussian blobs), dups (10% exact duplicate
    rows), grid (small integer coordinates: heavy distance ties), wide
    (magnitudes around 1e4 with fine offsets), clumps (about n/64 distinct
    points, each repeated ~64 times: masses of zero-weight edges).
    """
    rng = SplitMix64(7919 * seed + 5)
    if kind == "uniform":
        return rng.u24(n * d).reshape(n, d)
    if kind == "blobs":
        k = 4
        c = (-10.0 + 20.0 * rng.u53(k * d)).reshape(k, d)
        lab = rng.bounded(k, n)
        return (c[lab] + 0.7 * rng.normal(n * d).reshape(n, d)).astype(np.float32)
    if kind == "dups":
        nb = max(1, n - n // 10)
        base = rng.u24(nb * d).reshape(nb, d)
        src = rng.bounded(nb, n - nb)
        return rng.shuffle_rows(np.concatenate([base, base[src]]))
    if kind == "grid":
        return rng.bounded(4, n * d).reshape(n, d).astype(np.float32)
    if kind == "wide":
        return (1.0e4 + rng.u53(n * d) * 3.0).reshape(n, d).astype(np.float32)
    if kind == "clumps":
        nb = max(1, n // 64)
        base = rng.u24(nb * d).reshape(nb, d)
        return np.ascontiguousarray(base[rng.bounded(nb, n)])
    raise KeyError(kind)
