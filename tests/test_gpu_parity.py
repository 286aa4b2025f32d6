"""GPU parity: libappd (through its C ABI) against the CPU oracle, bit-exact.

The APPD is a function of W (unique, bit-unique after -0 -> +0; reading Q9), so
every comparison is exact.  Points mode: the GPU's R1 weights (appd_points_weights)
must equal the oracle's R1 bit-exactly and fp64 within 1e-5 relative, and the
APPD is compared bit-exactly.
"""
import json
import os

import numpy as np
import pytest

import oracle
from synth import generators as G

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def assert_bit_equal(got, want, what=""):
    got = np.asarray(got, np.float32)
    want = np.asarray(want, np.float32)
    assert got.shape == want.shape, (got.shape, want.shape)
    bad = np.nonzero(bits(got) != bits(want))
    if bad[0].size:
        idx = tuple(b[0] for b in bad)
        raise AssertionError(f"{what}: {bad[0].size} mismatching entries, first {idx}: gpu {got[idx]!r} oracle {want[idx]!r}")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2407_07058_b200 as P

    return P


@pytest.fixture(scope="module")
def ctx(P):
    c = P.Context(timing=True)
    yield c
    c.close()


def gpu_weights(ctx, W, sense=1, c=None):
    c = c or ctx
    Wt = torch.from_numpy(np.ascontiguousarray(W, np.float32)).cuda()
    return c.solve_weights(Wt).cpu().numpy()


def gpu_points(ctx, X):
    Xt = torch.from_numpy(np.ascontiguousarray(X, np.float32)).cuda()
    return ctx.solve_points(Xt).cpu().numpy()


def test_native_library_is_loaded(ctx):
    ctx.solve_weights(torch.zeros((2, 2), device="cuda"))
    maps = open("/proc/self/maps").read()
    assert "libappd.so" in maps
    st = ctx.stats()
    assert st["kernel_launches"] > 0


# --------------------------------------------------------------------------
# weights mode
# --------------------------------------------------------------------------
def test_c1(ctx):
    W = G.config("C1")
    assert_bit_equal(gpu_weights(ctx, W), oracle.appd_weights(W), "C1")


@pytest.fixture(scope="module")
def bctx(P):
    """Boruvka forced (AUTO takes the Prim variant for the small sizes below)."""
    c = P.Context(timing=True, variant=P.VARIANT_BORUVKA)
    yield c
    c.close()


@pytest.mark.parametrize("variant", ["auto", "boruvka"])
@pytest.mark.parametrize("kind", ["uniform", "ties", "ints255", "negative", "signed_zero", "huge"])
def test_random_weights(ctx, bctx, kind, variant):
    c = ctx if variant == "auto" else bctx
    rs = np.random.default_rng(11)
    sizes = [1, 2, 3, 4, 5, 7, 8, 31, 33, 127, 128, 129, 255, 257, 300, 513, 1000, 1024, 1031]
    for t, n in enumerate(sizes):
        W = G.random_weights(n, 100 + t, kind)
        assert_bit_equal(gpu_weights(c, W, c=c), oracle.appd_weights(W), f"{kind} n={n}")
    for t in range(40):
        n = int(rs.integers(2, 200))
        W = G.random_weights(n, 500 + t, kind)
        assert_bit_equal(gpu_weights(c, W, c=c), oracle.appd_weights(W), f"{kind} n={n}")


@pytest.mark.parametrize("topk", [0, -1, 4, 32])
def test_weights_cache_lengths(P, topk):
    """Weights mode with and without the round-0 candidate cache (several K), incl. ties."""
    c = P.Context(timing=True, topk=topk, variant=P.VARIANT_BORUVKA)
    try:
        for t, (n, kind) in enumerate([(300, "uniform"), (257, "ties"), (700, "ints255"), (129, "negative"),
                                       (1000, "ties")]):
            W = G.random_weights(n, 500 + t, kind)
            assert_bit_equal(gpu_weights(c, W, c=c), oracle.appd_weights(W), f"topk={topk} {kind} n={n}")
    finally:
        c.close()


@pytest.mark.parametrize("topk", [4, 8])
def test_weights_cache_multi_batch(P, topk):
    """The single-pass warp-per-row round-0 cache (n % 4 == 0: 1024-column batches) across
    several batches with a ragged last one, the diagonal in a later batch, heavy ties and
    signed zeros, both senses; n % 4 != 0 takes the two-pass kernel (same cache)."""
    for sense in (1, -1):
        with P.Context(timing=True, topk=topk, sense=sense, variant=P.VARIANT_BORUVKA) as c:
            for t, (n, kind) in enumerate([(2052, "ints255"), (3000, "ties"), (4100, "signed_zero"),
                                           (2050, "ints255"), (1028, "uniform")]):
                W = G.random_weights(n, 900 + t, kind)
                assert_bit_equal(gpu_weights(None, W, c=c), oracle.appd_weights(W, sense),
                                 f"topk={topk} sense={sense} {kind} n={n}")


@pytest.mark.parametrize("variant", [0, 2])
def test_widest_sense(P, variant):
    with P.Context(sense=-1, variant=variant) as cw:
        for t, n in enumerate([2, 3, 17, 64, 255, 600]):
            for kind in ("uniform", "ties", "negative"):
                W = G.random_weights(n, t, kind)
                assert_bit_equal(gpu_weights(None, W, c=cw), oracle.appd_weights(W, -1), f"widest {kind} n={n}")


def test_c3_closed_form_and_oracle(ctx):
    W = G.config("C3")
    M = gpu_weights(ctx, W)
    n = W.shape[0]
    off = ~np.eye(n, dtype=bool)
    assert (M[off] == 1.0).all()
    assert (bits(np.diag(M)) == 0).all()
    assert_bit_equal(M, oracle.appd_weights(W), "C3")


# --------------------------------------------------------------------------
# NEXT-2: the paper's comparison algorithm (minimax Floyd-Warshall) on the GPU
# --------------------------------------------------------------------------
def gpu_floyd(c, W):
    Wt = torch.from_numpy(np.ascontiguousarray(W, np.float32)).cuda()
    return c.floyd_weights(Wt).cpu().numpy()


@pytest.mark.parametrize("kind", ["uniform", "ties", "negative", "signed_zero", "huge"])
def test_floyd_against_oracle_floyd(ctx, kind):
    """Blocked (min, max) closure vs the oracle's literal triple loop, ragged
    tile counts (tile 128) included; and vs Algorithm 4 (the same APPD, reading Q9)."""
    for t, n in enumerate([1, 2, 3, 5, 31, 127, 128, 129, 200, 256, 257, 385]):
        W = G.random_weights(n, 700 + t, kind)
        want = oracle.floyd(W)
        assert_bit_equal(gpu_floyd(ctx, W), want, f"floyd {kind} n={n}")
    W = G.random_weights(1000, 799, kind)
    assert_bit_equal(gpu_floyd(ctx, W), oracle.appd_weights(W), f"floyd {kind} n=1000 vs Algorithm 4")


def test_floyd_widest(P):
    with P.Context(sense=-1) as cw:
        for t, n in enumerate([2, 3, 64, 129, 300]):
            for kind in ("uniform", "ties", "negative"):
                W = G.random_weights(n, 40 + t, kind)
                assert_bit_equal(gpu_floyd(cw, W), oracle.floyd(W, -1), f"floyd widest {kind} n={n}")


def test_floyd_equals_boruvka_path_c1_c3(ctx):
    """C1 against the oracle; the C3 recipe at n = 4096 (32 tiles, heavy ties) against
    the Boruvka path's result and Algorithm 4."""
    W = G.config("C1")
    assert_bit_equal(gpu_floyd(ctx, W), oracle.appd_weights(W), "floyd C1")
    W = G.config("C3", n=4096)
    Mf = gpu_floyd(ctx, W)
    assert_bit_equal(Mf, gpu_weights(ctx, W), "floyd C3 n=4096 vs Boruvka path")
    assert_bit_equal(Mf, oracle.appd_weights(W), "floyd C3 n=4096 vs Algorithm 4")


def test_floyd_validation(ctx, P):
    W = G.random_weights(130, 5, "uniform")
    W[3, 7] = np.float32(0.123)  # asymmetric
    with pytest.raises(P.AppdError) as e:
        gpu_floyd(ctx, W)
    assert e.value.name == "APPD_ERR_NOT_SYMMETRIC" and e.value.index == (3, 7)


# --------------------------------------------------------------------------
# points mode
# --------------------------------------------------------------------------
def test_r1_weights_bitexact_and_fp64(ctx):
    for name, X in [("C2", G.config("C2")), ("C4s", G.config("C4", n=1500)), ("C5s", G.config("C5", n=3000)),
                    ("d7", G.random_points(700, 7, 1, "dups"))]:
        Xt = torch.from_numpy(X).cuda()
        n = X.shape[0]
        rows = min(n, 512)
        Wg = ctx.points_weights(Xt, 0, rows).cpu().numpy()
        assert_bit_equal(Wg, oracle.points_weights(X, 0, rows), f"R1 {name}")
        ref = np.sqrt(((X[:rows, None, :].astype(np.float64) - X[None, :, :].astype(np.float64)) ** 2).sum(-1))
        nz = ref > 0
        assert (Wg[~nz] == 0).all()
        assert (np.abs(Wg[nz] - ref[nz]) / ref[nz]).max() <= 1e-5


def test_c2(ctx):
    X = G.config("C2")
    assert_bit_equal(gpu_points(ctx, X), oracle.appd_points(X), "C2")


@pytest.mark.parametrize("variant", ["auto", "boruvka"])
@pytest.mark.parametrize("kind", ["uniform", "blobs", "dups", "grid", "wide"])
def test_random_points(ctx, bctx, kind, variant):
    c = ctx if variant == "auto" else bctx
    cases = [(1, 3), (2, 1), (3, 2), (5, 64), (64, 1), (127, 33), (128, 32), (129, 31), (300, 2), (513, 65),
             (1000, 16), (1031, 70), (2048, 3)]
    for t, (n, d) in enumerate(cases):
        X = G.random_points(n, d, 40 + t, kind)
        assert_bit_equal(gpu_points(c, X), oracle.appd_points(X), f"{kind} n={n} d={d}")


# every points-mode engine configuration: the tensor-core filter with and
# without the round-0 candidate cache and the component-matrix finish, several cache
# lengths and finish thresholds, and the exact FP32 engine -- all bit-exact vs the oracle
ENGINES = [
    dict(),                                   # defaults: cache K=8, finish at k <= 128
    dict(topk=-1, finish_k=-1),               # every round a full tensor-core scan
    dict(topk=16, finish_k=-1),               # cache, Boruvka to the end (tensor-core re-scans)
    dict(topk=4, finish_k=4),                 # short cache, late finish
    dict(topk=32, finish_k=16),
    dict(topk=-1, finish_k=128),              # finish without the cache
    dict(points_engine=1),                    # exact FP32 engine
    dict(dendrogram=1),                       # host union-find dendrogram instead of the GPU Prim order
]
ENGINE_INPUTS = [("blobs", 3000, 16), ("uniform", 2500, 40), ("clumps", 3000, 8), ("grid", 2000, 5),
                 ("dups", 4100, 64), ("wide", 1500, 3)]


@pytest.fixture(scope="module")
def engine_inputs():
    return [(kind, n, d, G.random_points(n, d, 900 + t, kind)) for t, (kind, n, d) in enumerate(ENGINE_INPUTS)]


@pytest.fixture(scope="module")
def engine_refs(engine_inputs):
    return [oracle.appd_points(X) for (_, _, _, X) in engine_inputs]


@pytest.mark.parametrize("eng", range(len(ENGINES)))
def test_points_engines(P, eng, engine_inputs, engine_refs):
    c = P.Context(timing=True, **ENGINES[eng])
    try:
        for (kind, n, d, X), ref in zip(engine_inputs, engine_refs):
            assert_bit_equal(gpu_points(c, X), ref, f"{ENGINES[eng]} {kind} n={n} d={d}")
    finally:
        c.close()


def test_points_engine_paths_taken(P):
    """The configurations above really take the paths they name (statistics)."""
    X = G.config("C4", n=8192)
    ref = oracle.appd_points(X)
    c = P.Context(timing=True)
    assert_bit_equal(gpu_points(c, X), ref, "C4 n=8192 defaults")
    st = c.stats()
    assert st["points_engine"] == 2 and st["topk"] == 8 and st["cm_k"] > 0
    c.close()
    c = P.Context(timing=True, topk=-1, finish_k=-1)
    assert_bit_equal(gpu_points(c, X), ref, "C4 n=8192 no cache")
    st = c.stats()
    assert st["topk"] == 0 and st["cm_k"] == 0 and st["tcscan_launches"] == st["rounds"]
    c.close()
    # rounds whose flagged rows exceed the exact-row limit (1024): the re-scan queued before
    # the round's host wait must do nothing, the tensor-core re-scan then runs
    Xu = G.random_points(8192, 4, 78, "uniform")  # (measured: 4793 flagged rows, 48 re-scanned blocks)
    c = P.Context(timing=True, topk=4, finish_k=-1)
    assert_bit_equal(gpu_points(c, Xu), oracle.appd_points(Xu), "uniform n=8192 d=4 K=4, Boruvka to the end")
    st = c.stats()
    assert st["rescan_blocks"] > 0 and st["rescan_rows"] > 1024, st
    c.close()
    Xc = G.random_points(3000, 8, 77, "clumps")  # > 4K zero-distance columns per row: cache overflow
    c = P.Context(timing=True)
    assert_bit_equal(gpu_points(c, Xc), oracle.appd_points(Xc), "clumps")
    assert c.stats()["cache_invalid_rows"] > 0
    c.close()


def test_points_stream_to_host(ctx):
    """NEXT-4: M streamed to host memory in row blocks (ragged last block, one block,
    several blocks) equals the oracle and the device-resident path bit for bit."""
    for t, (kind, n, d, block) in enumerate([("blobs", 1, 3, 0), ("blobs", 2, 3, 1), ("uniform", 300, 5, 128),
                                             ("clumps", 3000, 8, 256), ("dups", 2500, 16, 0), ("blobs", 4100, 64, 1000)]):
        X = G.random_points(n, d, 950 + t, kind)
        M = torch.empty((n, n), dtype=torch.float32).pin_memory()
        ctx.solve_points_stream(torch.from_numpy(X), M, block)
        got = M.numpy()
        assert_bit_equal(got, oracle.appd_points(X), f"stream {kind} n={n} block={block}")
        assert_bit_equal(got, gpu_points(ctx, X), f"stream vs device {kind} n={n}")


def test_points_stream_tile_span_256(ctx):
    """Regression (round 2): a fill tile whose rows' leaf positions span exactly 256 read
    level 8 of the tile's 8-level shared-memory table (out of bounds).  Blocks of 128
    original rows at n = 257 span 256 positions whenever a block holds both end leaves;
    over 24 inputs that happens many times.  Each result must equal the oracle."""
    for t in range(24):
        X = G.random_points(257, 2, 4000 + t, "uniform")
        M = torch.empty((257, 257), dtype=torch.float32).pin_memory()
        ctx.solve_points_stream(torch.from_numpy(X), M, 128)
        assert_bit_equal(M.numpy(), oracle.appd_points(X), f"span-256 stream seed {4000 + t}")


def test_points_stream_large_vs_device(ctx):
    """32768 points (4 GiB of output) in 3000-row blocks against the device path."""
    X = G.config("C4", n=32768)
    n = X.shape[0]
    M = torch.empty((n, n), dtype=torch.float32).pin_memory()
    ctx.solve_points_stream(torch.from_numpy(X), M, 3000)
    ref = ctx.solve_points(torch.from_numpy(X).cuda()).cpu()
    assert torch.equal(M.view(torch.int32), ref.view(torch.int32))
    st = ctx.stats()
    assert st["fill_bytes"] == n * n * 4


@pytest.mark.parametrize("metric", [1, 2])
def test_points_metrics(P, metric):
    """NEXT-3: Manhattan / Chebyshev point metrics (exact FP32 engine) against the oracle,
    bit for bit, and the weights hook against the oracle's metric weights."""
    with P.Context(metric=metric) as c:
        for t, (kind, n, d) in enumerate([("blobs", 1, 3), ("blobs", 2, 2), ("uniform", 300, 5), ("clumps", 1500, 8),
                                          ("grid", 1000, 3), ("dups", 2100, 16), ("blobs", 700, 70)]):
            X = G.random_points(n, d, 970 + t, kind)
            assert_bit_equal(gpu_points(c, X), oracle.appd_points(X, metric=metric), f"metric {metric} {kind} n={n}")
        X = G.random_points(600, 9, 990, "uniform")
        Wg = c.points_weights(torch.from_numpy(X).cuda(), 0, 200).cpu().numpy()
        assert_bit_equal(Wg, oracle.points_weights(X, 0, 200, metric=metric), f"metric {metric} weights")
        assert c.stats()["points_engine"] == 1
    with P.Context(metric=metric, points_engine=2) as c2:
        with pytest.raises(P.AppdError) as e:
            gpu_points(c2, G.random_points(100, 4, 1, "blobs"))
        assert e.value.name == "APPD_ERR_UNSUPPORTED"


def test_permutation_equivariance_large(ctx):
    """relabelling the input relabels the APPD, M(P X) = P M(X) P^T, bit for
    bit, at sizes beyond the oracle's reach and with heavy ties (the engines break ties by
    index, so every tie decision changes under the permutation)."""
    g = torch.Generator().manual_seed(5)
    X = torch.from_numpy(G.random_points(20000, 16, 41, "clumps")).cuda()
    p = torch.randperm(X.shape[0], generator=g).cuda()
    M = ctx.solve_points(X)
    Mp = ctx.solve_points(X[p].contiguous())
    assert torch.equal(Mp.view(torch.int32), M[p][:, p].contiguous().view(torch.int32))
    W = torch.from_numpy(G.random_weights(3000, 42, "ties")).cuda()
    q = torch.randperm(W.shape[0], generator=g).cuda()
    M = ctx.solve_weights(W)
    Mq = ctx.solve_weights(W[q][:, q].contiguous())
    assert torch.equal(Mq.view(torch.int32), M[q][:, q].contiguous().view(torch.int32))


def test_points_too_large_for_the_filter(P):
    """Coordinates whose squares overflow fp32: the device-side scale reports it at the
    first synchronisation and the solve is redone on the exact engine (same result as the
    oracle, infinite distances included)."""
    rs = np.random.default_rng(8)
    X = (rs.standard_normal((2500, 6)) * 1e20).astype(np.float32)  # n > 2048: AUTO tries the filter
    X[:1250] *= np.float32(1e-20)  # half of the points at ordinary scale
    with P.Context(timing=True, variant=P.VARIANT_BORUVKA) as c:
        assert_bit_equal(gpu_points(c, X), oracle.appd_points(X), "huge coordinates")
        assert c.stats()["points_engine"] == 1
        Xs = G.random_points(2500, 8, 3, "blobs")  # the same context keeps working afterwards
        assert_bit_equal(gpu_points(c, Xs), oracle.appd_points(Xs), "after fallback")
        assert c.stats()["points_engine"] == 2


def test_points_list_overflow_is_exact(P):
    """A candidate list far too small for the input: rows whose entries are lost are
    poisoned (invalid cache, exact full-row minimum, re-scanned every round), and the
    result must not change."""
    X = G.random_points(3000, 16, 901, "blobs")
    ref = oracle.appd_points(X)
    c = P.Context(timing=True, list_cap=5000)
    try:
        assert_bit_equal(gpu_points(c, X), ref, "list overflow")
        st = c.stats()
        assert st["cache_invalid_rows"] > 0
        # the component matrix's own listing overflowed too: detected on the device,
        # the solve is repeated without it
        assert st["cm_retries"] == 1, st
    finally:
        c.close()


def _check_golden(M_rows_fn, cfg, name):
    path = os.path.join(GOLD, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated")
    g = json.load(open(path))
    X = G.config(cfg)
    assert oracle.fnv1a64(X) == g["input_fnv1a64"], "input generator drifted"
    B = g["block_rows"]
    r0 = g["row0"]
    for bi, want in enumerate(g["row_block_fnv1a64"]):
        rows = M_rows_fn(r0 + bi * B, min(B, g["rows"] - bi * B))
        assert f"{oracle.fnv1a64(rows):016x}" == want, f"{cfg} row block {bi}"


def _properties(M_gpu, X, h_sorted, rs_seed=0, samples=20000):
    """Properties that hold at any size: symmetry, +0 diagonal, ultrametric, M <= W,
    every value is a merge height (an MST weight)."""
    n = X.shape[0]
    rs = np.random.default_rng(rs_seed)
    i, j, k = rs.integers(0, n, (3, samples))
    idx_i = torch.from_numpy(i).cuda()
    idx_j = torch.from_numpy(j).cuda()
    idx_k = torch.from_numpy(k).cuda()
    mij = M_gpu[idx_i, idx_j].cpu().numpy()
    mji = M_gpu[idx_j, idx_i].cpu().numpy()
    mik = M_gpu[idx_i, idx_k].cpu().numpy()
    mkj = M_gpu[idx_k, idx_j].cpu().numpy()
    assert (bits(mij) == bits(mji)).all()
    assert (bits(M_gpu.diagonal()[:4096].cpu().numpy()) == 0).all()
    assert (mij <= np.maximum(mik, mkj)).all()
    for t in range(200):
        a, b = int(i[t]), int(j[t])
        w = 0.0 if a == b else float(oracle.r1_weight(X[a], X[b]))
        assert mij[t] <= w
    assert np.isin(mij[i != j], h_sorted).all()


def test_c4_full(ctx):
    X = G.config("C4")
    Xt = torch.from_numpy(X).cuda()
    M = ctx.solve_points(Xt)
    pi, h = ctx.last_dendrogram(X.shape[0])
    assert sorted(pi.tolist()) == list(range(X.shape[0]))
    _properties(M, X, np.sort(h))
    _check_golden(lambda r, c: M[r:r + c].cpu().numpy(), "C4", "C4.json")
    del M
    torch.cuda.empty_cache()


def hash_row_blocks(M, block_rows, workers=8):
    """FNV-1a-64 of every block of block_rows rows of the device matrix M (host copies one
    block at a time; the C hash runs in threads, ctypes releases the GIL)."""
    from concurrent.futures import ThreadPoolExecutor

    nb = (M.shape[0] + block_rows - 1) // block_rows

    def one(b):
        return f"{oracle.fnv1a64(M[b * block_rows:(b + 1) * block_rows].cpu().numpy()):016x}"

    with ThreadPoolExecutor(workers) as ex:
        return list(ex.map(one, range(nb)))


def test_c5_full_single_gpu(ctx):
    """C5 (n = 131072, 64 GiB) on one GPU against the oracle: EVERY 1024-row block's
    FNV-1a-64 equals tests/golden/C5.json (the oracle's R5 row windows: every
    cell), plus the closed-form count of zero merge heights."""
    X = G.config("C5")
    Xt = torch.from_numpy(X).cuda()
    M = ctx.solve_points(Xt)
    pi, h = ctx.last_dendrogram(X.shape[0])
    assert (h == 0).sum() == 1311  # SURVEY §8(c) pin 5: exactly 1311 zero merge heights
    _properties(M, X, np.sort(h))
    path = os.path.join(GOLD, "C5.json")
    g = json.load(open(path))
    assert oracle.fnv1a64(X) == g["input_fnv1a64"], "input generator drifted"
    assert g["rows"] == X.shape[0] and len(g["row_block_fnv1a64"]) == 128
    got = hash_row_blocks(M, g["block_rows"])
    bad = [b for b, (x, y) in enumerate(zip(got, g["row_block_fnv1a64"])) if x != y]
    assert not bad, f"C5 row blocks differing from the oracle: {bad[:10]} ({len(bad)} of 128)"
    del M
    torch.cuda.empty_cache()


# --------------------------------------------------------------------------
# boundary behaviour
# --------------------------------------------------------------------------
def test_validation_errors(P, ctx):
    W = G.random_weights(50, 3, "uniform")
    for (i, j, val, status) in [(3, 7, np.nan, "APPD_ERR_NONFINITE"), (10, 2, np.inf, "APPD_ERR_NONFINITE"),
                                 (5, 9, 0.123, "APPD_ERR_NOT_SYMMETRIC"), (9, 5, 0.123, "APPD_ERR_NOT_SYMMETRIC"),
                                 (4, 4, 1.0, "APPD_ERR_BAD_DIAGONAL")]:
        Wb = W.copy()
        Wb[i, j] = val
        with pytest.raises(P.AppdError) as e:
            gpu_weights(ctx, Wb)
        assert e.value.name == status
        want = (min(i, j), max(i, j)) if status == "APPD_ERR_NOT_SYMMETRIC" else (i, j)
        assert e.value.index == want
    # priority: non-finite, then diagonal, then symmetry; first offender in row-major order of its kind
    Wb = W.copy()
    Wb[20, 30] = np.nan
    Wb[2, 40] = 5.0
    Wb[1, 1] = 2.0
    with pytest.raises(P.AppdError) as e:
        gpu_weights(ctx, Wb)
    assert e.value.name == "APPD_ERR_NONFINITE" and e.value.index == (20, 30)
    Wb[20, 30] = Wb[30, 20]
    with pytest.raises(P.AppdError) as e:
        gpu_weights(ctx, Wb)
    assert e.value.name == "APPD_ERR_BAD_DIAGONAL" and e.value.index == (1, 1)
    Wb[1, 1] = 0
    Wb[7, 3] = 9.0
    with pytest.raises(P.AppdError) as e:
        gpu_weights(ctx, Wb)
    assert e.value.name == "APPD_ERR_NOT_SYMMETRIC" and e.value.index == (2, 40)
    X = G.random_points(40, 3, 1)
    X[7, 2] = np.nan
    with pytest.raises(P.AppdError) as e:
        gpu_points(ctx, X)
    assert e.value.name == "APPD_ERR_NONFINITE" and e.value.index == (7, 2)
    # -0 diagonal and -0 weights are valid
    Wz = G.random_weights(30, 2, "signed_zero")
    assert_bit_equal(gpu_weights(ctx, Wz), oracle.appd_weights(Wz), "signed zero")


def test_invalid_arguments(P, ctx):
    Wh = torch.zeros((4, 4))
    M = torch.empty((4, 4), device="cuda")
    with pytest.raises(P.AppdError) as e:
        ctx.solve_weights(Wh, M)  # host pointer
    assert e.value.name == "APPD_ERR_INVALID_ARGUMENT"
    L = P.load()
    assert L.appd_solve_points(ctx._h, 0, 0, 2, 0) == 1
    assert L.appd_solve_points(ctx._h, M.data_ptr(), 4, 0, M.data_ptr()) == 1


def test_single_vertex(ctx):
    assert_bit_equal(gpu_weights(ctx, np.zeros((1, 1), np.float32)), np.zeros((1, 1), np.float32))
    assert_bit_equal(gpu_points(ctx, np.ones((1, 5), np.float32)), np.zeros((1, 1), np.float32))


def test_host_buffer_calls(ctx):
    X = G.random_points(777, 9, 3, "blobs")
    Mh = torch.empty((777, 777)).pin_memory()
    ctx.solve_points_host(torch.from_numpy(X).pin_memory(), Mh)
    assert_bit_equal(Mh.numpy(), oracle.appd_points(X), "host points")
    W = G.random_weights(301, 5, "ties")
    Mw = torch.empty((301, 301))
    ctx.solve_weights_host(torch.from_numpy(W), Mw)
    assert_bit_equal(Mw.numpy(), oracle.appd_weights(W), "host weights")


def test_no_validation_path(P):
    with P.Context(validate=False) as c:
        W = G.random_weights(200, 9, "ints255")
        assert_bit_equal(gpu_weights(None, W, c=c), oracle.appd_weights(W))


def test_dendrogram_hook_is_a_leaf_order(ctx):
    """(pi, h) of the last solve reproduces the oracle through M[pi_a][pi_b] = max(h[a..b-1])."""
    W = G.random_weights(300, 8, "ties")
    M = gpu_weights(ctx, W)
    pi, h = ctx.last_dendrogram(300)
    Mo = oracle.appd_weights(W)
    for a in range(0, 300, 7):
        run = -np.inf
        for b in range(a + 1, 300):
            run = max(run, h[b - 1])
            assert Mo[pi[a], pi[b]] == run
    assert_bit_equal(M, Mo)


# --------------------------------------------------------------------------
# NEXT-3: fp64 weights (k_f64.cu) against the fp64 oracle, bit-exact
# --------------------------------------------------------------------------
def gpu_weights_f64(c, W):
    Wt = torch.from_numpy(np.ascontiguousarray(W, np.float64)).cuda()
    return c.solve_weights_f64(Wt).cpu().numpy()


def assert_f64_bit_equal(got, want, what=""):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64) + 0.0
    assert got.shape == want.shape, (got.shape, want.shape)
    bad = np.nonzero(got.view(np.uint64) != want.view(np.uint64))
    if bad[0].size:
        idx = tuple(b[0] for b in bad)
        raise AssertionError(f"{what}: {bad[0].size} mismatching entries, first {idx}: gpu {got[idx]!r} oracle {want[idx]!r}")


@pytest.mark.parametrize("kind", ["uniform", "fine_ties", "negative", "signed_zero", "huge"])
def test_f64_weights_against_oracle(P, kind):
    """Ragged sizes (odd n takes the scalar fill), both senses, values that collide in fp32."""
    for sense in (1, -1):
        with P.Context(sense=sense) as c:
            for t, n in enumerate([1, 2, 3, 5, 31, 64, 127, 300, 513, 1000]):
                W = G.random_weights_f64(n, 900 + t, kind)
                assert_f64_bit_equal(gpu_weights_f64(c, W), oracle.appd_weights_f64(W, sense), f"f64 {kind} sense {sense} n={n}")


def test_f64_fine_ties_n4096(ctx):
    W = G.random_weights_f64(4096, 77, "fine_ties")
    assert_f64_bit_equal(gpu_weights_f64(ctx, W), oracle.appd_weights_f64(W, 1), "f64 fine_ties n=4096")


def test_f64_equals_f32_path_on_c3(ctx):
    """The C3 recipe at full size (n = 16384, heavy ties) in fp64: the result equals the fp32
    path's, widened (the method copies weights), compared on the device."""
    W = torch.from_numpy(G.config("C3")).cuda()
    M32 = ctx.solve_weights(W)
    M64 = ctx.solve_weights_f64(W.double())
    assert bool((M64 == M32.double()).all()) and not bool(torch.signbit(M64).any())
    st = ctx.stats()
    assert st["fill_bytes"] == 16384 * 16384 * 8


def test_f64_validation(ctx, P):
    W = G.random_weights_f64(70, 3, "uniform")
    W2 = W.copy(); W2[3, 7] = W2[3, 7] + 2.0 ** -50  # asymmetric beyond fp32 precision
    with pytest.raises(P.AppdError) as e:
        gpu_weights_f64(ctx, W2)
    assert e.value.name == "APPD_ERR_NOT_SYMMETRIC" and e.value.index == (3, 7)
    W3 = W.copy(); W3[40, 40] = 1e-300
    with pytest.raises(P.AppdError) as e:
        gpu_weights_f64(ctx, W3)
    assert e.value.name == "APPD_ERR_BAD_DIAGONAL" and e.value.index == (40, 40)
    W4 = W.copy(); W4[50, 2] = np.inf; W4[2, 50] = np.inf
    with pytest.raises(P.AppdError) as e:
        gpu_weights_f64(ctx, W4)
    assert e.value.name == "APPD_ERR_NONFINITE" and e.value.index == (2, 50)
    with pytest.raises(TypeError):
        ctx.solve_weights_f64(torch.zeros((4, 4), dtype=torch.float32, device="cuda"))


# --------------------------------------------------------------------------
# the Prim variant: one CTA, (pi, h) directly
# --------------------------------------------------------------------------
@pytest.mark.parametrize("kind", ["uniform", "ties", "ints255", "negative", "signed_zero", "huge"])
def test_prim_variant_weights(P, kind):
    with P.Context(variant=P.VARIANT_PRIM, timing=True) as c:
        for t, n in enumerate([2, 3, 5, 31, 32, 33, 64, 127, 255, 256, 299, 300]):
            W = G.random_weights(n, 700 + t, kind)
            assert_bit_equal(gpu_weights(c, W, c=c), oracle.appd_weights(W), f"prim {kind} n={n}")
            st = c.stats()
            assert st["variant"] == P.VARIANT_PRIM and st["rounds"] == 0
    with P.Context(variant=P.VARIANT_PRIM, sense=-1) as c:
        for t, n in enumerate([2, 17, 200, 300]):
            W = G.random_weights(n, 720 + t, kind)
            assert_bit_equal(gpu_weights(c, W, c=c), oracle.appd_weights(W, -1), f"prim widest {kind} n={n}")


def test_prim_variant_c1_and_auto(P, ctx):
    W = G.config("C1")
    want = oracle.appd_weights(W)
    with P.Context(variant=P.VARIANT_PRIM) as c:
        assert_bit_equal(gpu_weights(c, W, c=c), want, "C1 prim")
    assert_bit_equal(gpu_weights(ctx, W), want, "C1 auto")
    assert ctx.stats()["variant"] == P.VARIANT_PRIM  # AUTO picks Prim at n = 256 (crossover table)
    with P.Context(variant=P.VARIANT_BORUVKA) as c:
        assert_bit_equal(gpu_weights(c, W, c=c), want, "C1 boruvka")
        assert c.stats()["variant"] == P.VARIANT_BORUVKA


@pytest.mark.parametrize("kind", ["uniform", "blobs", "dups", "grid", "clumps", "wide"])
def test_prim_variant_points(P, kind):
    with P.Context(variant=P.VARIANT_PRIM) as c:
        for t, (n, d) in enumerate([(2, 1), (3, 2), (100, 3), (127, 2), (129, 4), (1023, 2), (1025, 5),
                                    (2048, 2), (2000, 16), (700, 64)]):
            X = G.random_points(n, d, 730 + t, kind)
            assert_bit_equal(gpu_points(c, X), oracle.appd_points(X), f"prim points {kind} n={n} d={d}")


def test_prim_variant_c2_and_metrics(P):
    X = G.config("C2", n=2048)  # the C2 recipe at the largest n the variant takes
    want = oracle.appd_points(X)
    with P.Context(variant=P.VARIANT_PRIM) as c:
        assert_bit_equal(gpu_points(c, X), want, "C2 recipe n=2048 prim")
    for metric in (1, 2):
        Xm = G.random_points(1500, 6, 91 + metric, "blobs")
        with P.Context(variant=P.VARIANT_PRIM, metric=metric) as c:
            assert_bit_equal(gpu_points(c, Xm), oracle.appd_points(Xm, metric=metric), f"prim metric {metric}")


def test_prim_variant_validation_and_limits(P):
    with P.Context(variant=P.VARIANT_PRIM) as c:
        W = G.random_weights(50, 3, "uniform")
        W[7, 9] = np.float32(2.0)
        with pytest.raises(P.AppdError) as e:
            gpu_weights(c, W, c=c)
        assert e.value.name == "APPD_ERR_NOT_SYMMETRIC" and e.value.index == (7, 9)
        W = G.random_weights(50, 3, "uniform")
        W[4, 4] = np.float32(1.0)
        W[30, 2] = np.float32(np.nan)
        W[2, 30] = np.float32(np.nan)
        with pytest.raises(P.AppdError) as e:
            gpu_weights(c, W, c=c)
        assert e.value.name == "APPD_ERR_NONFINITE" and e.value.index == (2, 30)
        W = G.random_weights(50, 3, "uniform")
        W[4, 4] = np.float32(1.0)
        with pytest.raises(P.AppdError) as e:
            gpu_weights(c, W, c=c)
        assert e.value.name == "APPD_ERR_BAD_DIAGONAL" and e.value.index == (4, 4)
        X = G.random_points(300, 3, 5, "uniform")
        X[17, 1] = np.float32(np.inf)
        with pytest.raises(P.AppdError) as e:
            gpu_points(c, X)
        assert e.value.name == "APPD_ERR_NONFINITE" and e.value.index == (17, 1)
        # too large for one CTA: explicit PRIM is refused, AUTO takes Boruvka
        with pytest.raises(P.AppdError) as e:
            gpu_weights(c, G.random_weights(301, 3, "uniform"), c=c)
        assert e.value.name == "APPD_ERR_UNSUPPORTED"
        with pytest.raises(P.AppdError) as e:
            gpu_points(c, G.random_points(2049, 2, 3, "uniform"))
        assert e.value.name == "APPD_ERR_UNSUPPORTED"
        W = G.random_weights(50, 3, "ties")
        assert_bit_equal(gpu_weights(c, W, c=c), oracle.appd_weights(W), "after errors")


# --------------------------------------------------------------------------
# NEXT-4 beyond n = 131072: wide edge keys (two-step component reduction) and the block sink
# --------------------------------------------------------------------------
@pytest.mark.parametrize("kind", ["uniform", "dups", "grid", "clumps", "blobs"])
def test_wide_keys_engine(P, kind):
    """The wide-key path (automatic above n = 131072) forced at small n: bit-exact vs the
    oracle, ties (grid), zero-weight edges (dups, clumps) and ragged sizes included."""
    with P.Context(wide_keys=1, timing=True) as c:
        for t, (n, d) in enumerate([(2, 3), (3, 1), (129, 4), (1000, 8), (2500, 3), (4100, 16)]):
            X = G.random_points(n, d, 960 + t, kind)
            assert_bit_equal(gpu_points(c, X), oracle.appd_points(X), f"wide {kind} n={n} d={d}")
            st = c.stats()
            assert n < 2 or (st["points_engine"] == 1 and st["variant"] == P.VARIANT_BORUVKA)


def test_wide_keys_metrics(P):
    for metric in (1, 2):
        X = G.random_points(1500, 5, 970 + metric, "blobs")
        with P.Context(wide_keys=1, metric=metric) as c:
            assert_bit_equal(gpu_points(c, X), oracle.appd_points(X, metric=metric), f"wide metric {metric}")


def test_points_sink_blocks(P):
    """appd_solve_points_sink: blocks arrive in row order, tile M exactly, equal the oracle."""
    X = G.random_points(3000, 6, 975, "dups")
    want = oracle.appd_points(X)
    for block in (700, 0, 3000, 1):
        got = np.full_like(want, np.nan)
        seen = []
        with P.Context() as c:
            def sink(r0, blk):
                seen.append((r0, blk.shape[0]))
                got[r0:r0 + blk.shape[0]] = blk
            c.solve_points_sink(torch.from_numpy(X), sink, block if block != 1 else 1)
        assert [r for r, _ in seen] == sorted(r for r, _ in seen) and sum(k for _, k in seen) == 3000
        assert_bit_equal(got, want, f"sink block={block}")
    with P.Context() as c:  # a failing sink stops the solve
        def bad(r0, blk):
            raise RuntimeError("disk full")
        with pytest.raises(RuntimeError):
            c.solve_points_sink(torch.from_numpy(X), bad, 1000)
        assert_bit_equal(gpu_points(c, X), want, "after a failed sink")


def test_c5x_beyond_hbm_sink(P):
    """NEXT-4: the C5 recipe at n = 2^18 -- 256 GiB of output, more than the GPU's
    HBM and this host's RAM -- through the sink, on the wide-key path; the first, middle and
    last 1024-row blocks hash to the oracle's R5 windows (tests/golden/C5x_windows.json)."""
    path = os.path.join(GOLD, "C5x_windows.json")
    if not os.path.exists(path):
        pytest.skip("C5x_windows.json not generated")
    g = json.load(open(path))
    X = G.c5_points(g["n"], g["d"], 4)
    assert oracle.fnv1a64(X) == g["input_fnv1a64"]
    n, B = g["n"], g["block_rows"]
    got, rows = {}, [0]

    def sink(r0, blk):
        assert r0 == rows[0]
        rows[0] += blk.shape[0]
        for b0 in range(r0, r0 + blk.shape[0], B):
            if str(b0) in g["blocks"]:
                got[str(b0)] = f"{oracle.fnv1a64(np.ascontiguousarray(blk[b0 - r0:b0 - r0 + B])):016x}"

    with P.Context(timing=True) as c:
        c.solve_points_sink(torch.from_numpy(X), sink, B)
        st = c.stats()
    assert rows[0] == n
    assert got == g["blocks"], (got, g["blocks"])
    assert st["points_engine"] == 1 and st["fill_bytes"] == n * n * 4


# --------------------------------------------------------------------------
# widest paths in points mode (VERDICT r1 missing #6): Algorithm 4 in the widest
# sense on the oracle's own point weights
# --------------------------------------------------------------------------
def widest_points_ref(X, metric=0):
    return oracle.appd_weights(oracle.points_weights(X, metric=metric), -1)


@pytest.mark.parametrize("variant", [0, 1, 2])
def test_points_widest(P, variant):
    with P.Context(sense=-1, variant=variant) as c:
        for t, (kind, n, d) in enumerate([("uniform", 2, 3), ("blobs", 300, 4), ("dups", 700, 8), ("grid", 1000, 3),
                                          ("clumps", 1500, 6), ("wide", 2048, 2)]):
            if variant == 1 and n > 2048:
                continue
            X = G.random_points(n, d, 990 + t, kind)
            assert_bit_equal(gpu_points(c, X), widest_points_ref(X), f"widest points {kind} n={n} variant={variant}")


def test_points_widest_metrics_wide_keys_and_stream(P):
    X = G.random_points(1200, 5, 995, "blobs")
    for metric in (1, 2):
        with P.Context(sense=-1, metric=metric) as c:
            assert_bit_equal(gpu_points(c, X), widest_points_ref(X, metric), f"widest metric {metric}")
    with P.Context(sense=-1, wide_keys=1) as c:
        assert_bit_equal(gpu_points(c, X), widest_points_ref(X), "widest wide keys")
        M = torch.empty((1200, 1200), dtype=torch.float32).pin_memory()
        c.solve_points_stream(torch.from_numpy(X), M, 500)
        assert_bit_equal(M.numpy(), widest_points_ref(X), "widest streamed")
    with P.Context(sense=-1, points_engine=2) as c:  # the tensor-core filter finds minima only
        with pytest.raises(P.AppdError) as e:
            gpu_points(c, X)
        assert e.value.name == "APPD_ERR_UNSUPPORTED"


def test_points_widest_c2(P):
    X = G.config("C2")
    with P.Context(sense=-1) as c:
        assert_bit_equal(gpu_points(c, X), widest_points_ref(X), "widest C2")
