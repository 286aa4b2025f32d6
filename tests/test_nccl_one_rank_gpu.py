"""The NCCL transport of the multi-rank path, executed on ONE GPU (
DESIGN.md §7).

A context created with world = 1 AND an explicit ncclUniqueId builds a one-rank NCCL
communicator and runs the multi-rank code path over it: the solve-start agreement, the
validation-verdict all-reduce, the row-sharded Boruvka scans with the per-round
ncclAllReduce(min, uint64) of component keys, the component-matrix all-reduce, and the
deadline-polled waits (cudaStreamQuery + ncclCommGetAsyncError) -- every collective issued
through the real NCCL library on the B200, with one rank.  One process, one GPU: no rank
waits on another.  The results must be bit-identical to the oracle's (Algorithm 4)
and to the plain world-1 solve; the stats must show the collectives were issued.
The same cases run with the host exchange backend at world 1 (identity callback).
"""
import os

import numpy as np
import pytest

import oracle
from synth import generators as G

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")  # one-rank bootstrap on loopback
    import paper_2407_07058_b200 as P

    return P


@pytest.fixture(scope="module")
def nccl_ctx(P):
    c = P.Context(world=1, rank=0, nccl_id=P.appd_get_nccl_unique_id(), timing=True, timeout_ms=60000)
    yield c
    c.close()


@pytest.fixture(scope="module")
def host_ctx(P):
    calls = []

    def identity(words, op):  # one rank: the all-reduce of one contribution is itself
        calls.append((len(words), op))
        return words

    c = P.Context(world=1, rank=0, host_allreduce=identity, timing=True)
    c._calls = calls
    yield c
    c.close()


@pytest.fixture(scope="module")
def plain_ctx(P):
    c = P.Context(timing=True)
    yield c
    c.close()


CASES = [
    ("c2_4096", "points", lambda: G.config("C2", n=4096), {}),
    ("c4_shape_8192", "points", lambda: G.config("C4", n=8192), {}),
    ("c5_shape_6000_dups", "points", lambda: G.config("C5", n=6000), {}),
    ("points_blobs_1500_d7", "points", lambda: G.random_points(1500, 7, 31, "blobs"), {}),
    ("c3_shape_4096", "weights", lambda: G.config("C3", n=4096), {}),
    ("weights_ties_1031", "weights", lambda: G.random_weights(1031, 23, "ties"), {}),
]


def _solve(ctx, mode, A):
    t = torch.from_numpy(np.ascontiguousarray(A, np.float32)).cuda()
    M = ctx.solve_points(t) if mode == "points" else ctx.solve_weights(t)
    return M.cpu().numpy()


def _oracle(mode, A):
    return oracle.appd_points(A) if mode == "points" else oracle.appd_weights(A)


@pytest.mark.parametrize("name,mode,make,opts", CASES, ids=[c[0] for c in CASES])
def test_nccl_one_rank_matches_oracle_and_world1(nccl_ctx, plain_ctx, name, mode, make, opts):
    A = make()
    got = _solve(nccl_ctx, mode, A)
    st = nccl_ctx.stats()
    assert st["collectives"] >= 2, st  # agreement + at least one round exchange went through NCCL
    want = _oracle(mode, A)
    assert got.shape == want.shape
    assert np.array_equal(_bits(got), _bits(want)), f"{name}: NCCL one-rank solve differs from the oracle"
    ref = _solve(plain_ctx, mode, A)
    assert plain_ctx.stats()["collectives"] == 0
    assert np.array_equal(_bits(got), _bits(ref))


@pytest.mark.parametrize("name,mode,make,opts", CASES[:2] + CASES[4:5], ids=[c[0] for c in CASES[:2] + CASES[4:5]])
def test_host_exchange_one_rank_matches_oracle(host_ctx, name, mode, make, opts):
    A = make()
    host_ctx._calls.clear()
    got = _solve(host_ctx, mode, A)
    assert host_ctx.stats()["collectives"] == len(host_ctx._calls) >= 2
    want = _oracle(mode, A)
    assert np.array_equal(_bits(got), _bits(want)), f"{name}: host-exchange one-rank solve differs from the oracle"


OPT_CASES = [
    ("points_exact_engine_2500", "points", lambda: G.random_points(2500, 8, 41, "clumps"), {"points_engine": 1}),
    ("points_prim_replicated_900", "points", lambda: G.random_points(900, 3, 43, "blobs"), {"variant": 1}),
    ("points_wide_keys_1200", "points", lambda: G.random_points(1200, 6, 47, "dups"), {"wide_keys": 1}),
    ("points_widest_1100", "points", lambda: G.random_points(1100, 4, 53, "blobs"), {"sense": -1}),
    ("weights_widest_700", "weights", lambda: G.random_weights(700, 59, "ties"), {"sense": -1}),
    ("weights_nocache_600", "weights", lambda: G.random_weights(600, 61, "negative"), {"topk": -1}),
]


@pytest.mark.parametrize("name,mode,make,opts", OPT_CASES, ids=[c[0] for c in OPT_CASES])
def test_nccl_one_rank_options(P, name, mode, make, opts):
    """Engine / variant / key / sense options on the NCCL multi-rank path (fresh communicator
    per context), bit-exact against the oracle (widest: Algorithm 4 in the max-min sense)."""
    A = make()
    with P.Context(world=1, rank=0, nccl_id=P.appd_get_nccl_unique_id(), timing=True, timeout_ms=60000,
                   **opts) as c:
        got = _solve(c, mode, A)
        assert c.stats()["collectives"] >= 1
    sense = opts.get("sense", 1)
    if mode == "points":
        want = oracle.appd_weights(oracle.points_weights(A), sense) if sense < 0 else oracle.appd_points(A)
    else:
        want = oracle.appd_weights(A, sense)
    assert np.array_equal(_bits(got), _bits(want)), f"{name}: differs from the oracle"


def test_nccl_one_rank_validation_error(P, nccl_ctx):
    """The verdict all-reduce over NCCL: a non-finite input is reported with its first
    offender (a complete graph with finite weights), and the context stays usable."""
    W = G.random_weights(300, 5, "uniform")
    W[7, 11] = W[11, 7] = np.nan
    with pytest.raises(P.AppdError) as e:
        _solve(nccl_ctx, "weights", W)
    assert e.value.name == "APPD_ERR_NONFINITE" and e.value.index in ((7, 11), (11, 7)), (e.value.name, e.value.index)
    W2 = G.random_weights(300, 6, "uniform")
    assert np.array_equal(_bits(_solve(nccl_ctx, "weights", W2)), _bits(oracle.appd_weights(W2)))


def test_failed_exchange_poisons_the_context(P):
    """A failed exchange (the host_allreduce callback reports an error, as a dead peer's
    transport would) ends the call with APPD_ERR_NCCL and poisons the context: every later
    call returns APPD_ERR_POISONED instead of running on an inconsistent state (appd.h
    error contract).  A fresh context on the same device works again."""
    n_calls = []

    def broken(words, op):
        n_calls.append(op)
        if len(n_calls) >= 2:  # the agreement passes, the next exchange fails
            raise RuntimeError("peer lost")

    X = G.random_points(700, 3, 67, "blobs")
    c = P.Context(world=1, rank=0, host_allreduce=broken, variant=P.VARIANT_BORUVKA)
    try:
        with pytest.raises(P.AppdError) as e:
            _solve(c, "points", X)
        assert e.value.name == "APPD_ERR_NCCL", e.value.name
        with pytest.raises(P.AppdError) as e2:
            _solve(c, "points", X)
        assert e2.value.name == "APPD_ERR_POISONED", e2.value.name
    finally:
        c.close()
    with P.Context() as c2:
        assert np.array_equal(_bits(_solve(c2, "points", X)), _bits(oracle.appd_points(X)))


@pytest.mark.timeout(300)
def test_nccl_deadline_aborts_and_poisons(P):
    """The deadline of the NCCL backend's polled waits (appd_options.timeout_ms; SURVEY
    §8(b): a dead or diverged peer must end the call, not hang it).  GPU work queued ahead
    of the solve on the stream the library follows (a ~1.5 s spin kernel) stands in for a
    peer that never arrives: the first polled wait passes timeout_ms = 100, the library
    aborts the communicator (ncclCommAbort) and returns APPD_ERR_NCCL, and the context is
    poisoned.  The process and the device stay usable."""
    X = G.random_points(3000, 4, 71, "blobs")
    t = torch.from_numpy(X).cuda()
    torch.cuda.synchronize()
    c = P.Context(world=1, rank=0, nccl_id=P.appd_get_nccl_unique_id(), timeout_ms=100,
                  variant=P.VARIANT_BORUVKA)
    M = torch.empty((X.shape[0], X.shape[0]), dtype=torch.float32, device="cuda")
    try:
        c.solve_points(t, M)  # workspace allocated now (a cudaFree would wait for the spin)
        torch.cuda.synchronize()
        torch.cuda._sleep(int(3e9))  # ~1.5 s at 1.97 GHz on torch's current stream
        with pytest.raises(P.AppdError) as e:
            c.solve_points(t, M)
        assert e.value.name == "APPD_ERR_NCCL" and "timeout_ms" in str(e.value), str(e.value)
        with pytest.raises(P.AppdError) as e2:
            c.solve_points(t, M)
        assert e2.value.name == "APPD_ERR_POISONED", e2.value.name
    finally:
        torch.cuda.synchronize()
        c.close()
    with P.Context() as c2:
        assert np.array_equal(_bits(_solve(c2, "points", X)), _bits(oracle.appd_points(X)))
