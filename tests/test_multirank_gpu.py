"""world > 1 through libappd's own code on ONE GPU.

N processes (torch.multiprocessing, gloo) each create a libappd context with
rank r of world N on cuda:0 and the host exchange backend
(appd_options.host_allreduce = torch.distributed all-reduce over gloo).  The
library's world > 1 code path then runs exactly as under NCCL -- solve-start
agreement, validation-verdict agreement, row-sharded Boruvka scans (the
tensor-core cache build, cached rounds, the component-matrix all-reduce), the
per-round all-reduce(min) of component keys and the row-sharded fill -- only the
transport differs (host memory instead of NVLink).  The ranks' kernels never wait
on one another (every exchange is a host round trip), so sharing one GPU is safe.

Every rank's row block is compared bit-exactly with the oracle's rows (R5: the
same Algorithm 4 with writes filtered to the block), in weights and
points mode, with ties and zero-weight edges, and at C4's shape (d = 64) with
n = 8192.  A rank given a different X, n or option must make EVERY rank fail with
APPD_ERR_INVALID_ARGUMENT instead of hanging.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# (name, mode, input recipe, context options)
CASES = [
    ("c4_shape_8192", "points", ("C4", 8192), {}),
    ("c5_shape_8192_dups", "points", ("C5", 8192), {}),
    ("c2_4096", "points", ("C2", 4096), {}),
    ("points_clumps_3000_exact_engine", "points", ("clumps", 3000, 8), {"points_engine": 1}),
    ("points_grid_2000_nocache", "points", ("grid", 2000, 3), {"topk": -1}),
    ("points_dups_1500_no_cm", "points", ("dups", 1500, 16), {"finish_k": -1}),
    ("points_manhattan_700", "points", ("blobs", 700, 5), {"metric": 1}),
    ("points_prim_replicated_900", "points", ("blobs", 900, 3), {"variant": 1}),
    ("points_prim_fused_300", "points", ("dups", 300, 4), {"variant": 1}),
    ("points_wide_keys_1200", "points", ("dups", 1200, 6), {"wide_keys": 1}),
    ("points_widest_1100", "points", ("blobs", 1100, 4), {"sense": -1}),
    ("c3_shape_4096_ties", "weights", ("C3", 4096), {}),
    ("weights_ties_1031", "weights", ("ties", 1031), {}),
    ("weights_negative_600_nocache", "weights", ("negative", 600), {"topk": -1}),
    ("weights_uniform_129", "weights", ("uniform", 129), {}),
    ("weights_widest_500", "weights", ("ties", 500), {"sense": -1}),
    ("weights_n1", "weights", ("uniform", 1), {}),
]


def make_input(recipe):
    from synth import generators as G

    if recipe[0] in G.CONFIGS:
        return G.config(recipe[0], n=recipe[1])
    if len(recipe) == 3:
        return G.random_points(recipe[1], recipe[2], 17, recipe[0])
    return G.random_weights(recipe[1], 23, recipe[0])


def oracle_rows(mode, A, r0, rows, opts):
    import oracle

    if rows == 0:
        return np.zeros((0, A.shape[0]), np.float32)
    if mode == "points":
        if opts.get("sense", 1) < 0:
            return oracle.appd_weights(oracle.points_weights(A, metric=opts.get("metric", 0)), -1)[r0:r0 + rows]
        if opts.get("metric"):
            return oracle.appd_points(A, metric=opts["metric"])[r0:r0 + rows]
        return oracle.appd_points_rows(A, r0, rows)
    if opts.get("sense", 1) < 0:
        return oracle.appd_weights(A, -1)[r0:r0 + rows]
    return oracle.appd_weights_rows(A, r0, rows)


def _worker(rank, world, port, names, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import datetime

    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=180))
    res = {}
    try:
        import paper_2407_07058_b200 as P
        from paper_2407_07058_b200.distributed import gloo_host_allreduce

        torch.cuda.set_device(0)
        xchg = gloo_host_allreduce()
        for name, mode, recipe, opts in CASES:
            if name not in names:
                continue
            res["case"] = name
            A = make_input(recipe)
            n = A.shape[0]
            with P.Context(device=0, rank=rank, world=world, host_allreduce=xchg, timing=True, **opts) as ctx:
                r0, rows = ctx.row_range(n)
                if mode == "points":
                    M = ctx.solve_points(torch.from_numpy(A).cuda())
                else:
                    M = ctx.solve_weights(torch.from_numpy(np.ascontiguousarray(A[r0:r0 + rows])).cuda())
                got = M.cpu().numpy()
                st = ctx.stats()
            want = oracle_rows(mode, A, r0, rows, opts)
            bad = int(np.count_nonzero(got.view(np.uint32) != want.view(np.uint32)))
            res[name] = {"r0": r0, "rows": rows, "bad": bad, "collectives": st["collectives"],
                         "rounds": st["rounds"], "engine": st["points_engine"], "cm_k": st["cm_k"],
                         "topk": st["topk"]}
        # deliberately mismatched inputs: every rank must fail the same way, none may hang
        if "mismatch" in names:
            from synth import generators as G

            X = G.config("C4", n=1024)
            Xr = X.copy()
            if rank == world - 1:
                Xr[5, 3] = np.nextafter(Xr[5, 3], np.float32(1e9))  # one ulp in one coordinate
            errs = []
            with P.Context(device=0, rank=rank, world=world, host_allreduce=xchg) as ctx:
                for label, call in [
                    ("x", lambda: ctx.solve_points(torch.from_numpy(Xr).cuda())),
                    ("n", lambda: ctx.solve_points(torch.from_numpy(X[: 1024 - 128 * (rank == 0)]).cuda())),
                ]:
                    try:
                        call()
                        errs.append((label, "ok", ""))
                    except P.AppdError as e:
                        errs.append((label, e.name, str(e)))
                # a consistent solve afterwards still works (the failure is not poisoning)
                M = ctx.solve_points(torch.from_numpy(X).cuda())
                r0, rows = ctx.row_range(1024)
                want = oracle_rows("points", X, r0, rows, {})
                errs.append(("after", "ok" if (M.cpu().numpy().view(np.uint32) == want.view(np.uint32)).all() else "bad", ""))
            with P.Context(device=0, rank=rank, world=world, host_allreduce=xchg,
                           topk=(16 if rank == 0 else 8)) as ctx:
                try:
                    ctx.solve_points(torch.from_numpy(X).cuda())
                    errs.append(("opt", "ok", ""))
                except P.AppdError as e:
                    errs.append(("opt", e.name, str(e)))
            res["mismatch"] = errs
        # C5 at its full size: this rank's 1024-row blocks against the oracle's goldens
        if "c5_full" in names:
            import json

            from synth import generators as G

            g = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "C5.json")))
            X = G.config("C5")
            with P.Context(device=0, rank=rank, world=world, host_allreduce=xchg, timing=True) as ctx:
                n = X.shape[0]
                r0, rows = ctx.row_range(n)
                M = ctx.solve_points(torch.from_numpy(X).cuda())
                st = ctx.stats()
                B = g["block_rows"]
                assert r0 % B == 0 and rows % B == 0, (r0, rows)
                from test_gpu_parity import hash_row_blocks

                got = hash_row_blocks(M, B, workers=4)
                want = g["row_block_fnv1a64"][r0 // B:(r0 + rows) // B]
                del M
                torch.cuda.empty_cache()
            res["c5_full"] = {"r0": r0, "rows": rows, "blocks": len(got),
                              "bad": [r0 // B + b for b, (x, y) in enumerate(zip(got, want)) if x != y],
                              "rounds": st["rounds"], "collectives": st["collectives"], "ms_total": st["ms_total"]}
    except Exception as e:  # noqa: BLE001
        import traceback

        res["error"] = f"case {res.get('case')}: " + traceback.format_exc()
    finally:
        out[rank] = res
        dist.destroy_process_group()


def run_world(world, names):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), names, out), nprocs=world, join=True)
    res = [dict(out.get(r, {"error": "no result"})) for r in range(world)]
    errors = [f"rank {r}:\n{x['error']}" for r, x in enumerate(res) if "error" in x]
    assert not errors, "\n".join(errors)
    return res


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


ALL = [c[0] for c in CASES]


@pytest.mark.parametrize("world", [2, 3])
def test_row_blocks_bit_exact_per_rank(gpu, world):
    res = run_world(world, ALL)
    for name, mode, recipe, opts in CASES:
        blocks = [r[name] for r in res]
        n = make_input(recipe).shape[0]
        # the ranks' blocks tile the rows in order
        nxt = 0
        for b in blocks:
            assert b["r0"] == nxt
            nxt += b["rows"]
        assert nxt == n, name
        for r, b in enumerate(blocks):
            assert b["bad"] == 0, f"{name} world {world} rank {r}: {b['bad']} entries differ from the oracle rows"
        if n > 1 and opts.get("variant") != 1:
            # the exchange really ran: agreement + verdict (if validated) + one per round at least
            assert all(b["collectives"] >= 1 + blocks[0]["rounds"] for b in blocks), (name, blocks)
        assert len({b["rounds"] for b in blocks}) == 1, (name, blocks)
    # the tensor-core engine with its cache and component-matrix finish ran sharded
    c4 = res[0]["c4_shape_8192"]
    assert c4["engine"] == 2 and c4["topk"] > 0 and c4["cm_k"] > 0, c4


def test_rank_disagreement_fails_everywhere(gpu):
    world = 2
    res = run_world(world, ["mismatch"])
    for r in range(world):
        errs = {label: (name, msg) for label, name, msg in res[r]["mismatch"]}
        assert errs["x"][0] == "APPD_ERR_INVALID_ARGUMENT" and "checksum of X" in errs["x"][1], errs
        assert errs["n"][0] == "APPD_ERR_INVALID_ARGUMENT", errs
        assert errs["after"][0] == "ok", errs
        assert errs["opt"][0] == "APPD_ERR_INVALID_ARGUMENT", errs


@pytest.mark.parametrize("world", [2, 4])
def test_c5_row_blocks_per_rank(gpu, world):
    """C5 (n = 131072, d = 16; the north star's multi-GPU config) sharded over `world`
    ranks: every rank's 1024-row blocks hash to the oracle's goldens (tests/golden/C5.json)."""
    if not os.path.exists(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "C5.json")):
        pytest.skip("C5.json not generated")
    res = run_world(world, ["c5_full"])
    total = 0
    for r, x in enumerate(res):
        b = x["c5_full"]
        assert not b["bad"], f"rank {r}: blocks {b['bad']} differ from the oracle"
        total += b["blocks"]
    assert total == 128
