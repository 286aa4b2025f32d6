"""Bisect world > 1 failures on one GPU: each config in its own 2-process spawn."""
import datetime
import os
import socket
import sys
import traceback

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def port():
    s = socket.socket(); s.bind(("127.0.0.1", 0)); p = s.getsockname()[1]; s.close(); return p


def worker(rank, world, p, cfgs, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(p)
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=60))
    for cfg in cfgs:
        one(rank, world, cfg, out)
        print(rank, cfg[0], out.get((rank, cfg[0])), flush=True)
    try:
        dist.destroy_process_group()
    except Exception:
        pass


def one(rank, world, cfg, out):
    import oracle
    import paper_2407_07058_b200 as P
    from paper_2407_07058_b200.distributed import gloo_host_allreduce
    from synth import generators as G
    name, mode, recipe, opts = cfg
    try:
        if recipe[1] == 1:
            raise RuntimeError("skip n=1")
        A = G.config(recipe[0], n=recipe[1]) if recipe[0] in G.CONFIGS else (
            G.random_points(recipe[1], recipe[2], 17, recipe[0]) if len(recipe) == 3 else G.random_weights(recipe[1], 23, recipe[0]))
        with P.Context(device=0, rank=rank, world=world, host_allreduce=gloo_host_allreduce(), timing=True, **opts) as ctx:
            n = A.shape[0]
            r0, rows = ctx.row_range(n)
            if mode == "points":
                M = ctx.solve_points(torch.from_numpy(A).cuda())
            else:
                M = ctx.solve_weights(torch.from_numpy(np.ascontiguousarray(A[r0:r0 + rows])).cuda())
            got = M.cpu().numpy()
            st = ctx.stats()
        want = oracle.appd_points_rows(A, r0, rows) if mode == "points" else oracle.appd_weights_rows(A, r0, rows)
        bad = int(np.count_nonzero(got.view(np.uint32) != want.view(np.uint32)))
        out[(rank, name)] = f"ok bad={bad} rounds={st['rounds']} coll={st['collectives']} cm_k={st['cm_k']}"
    except Exception:
        out[(rank, name)] = "ERR " + traceback.format_exc().strip().splitlines()[-1]


CFGS = [
    ("c4_2048_exact", "points", ("C4", 2048), {"points_engine": 1}),
    ("c4_2048_nocache", "points", ("C4", 2048), {"topk": -1}),
    ("c4_2048_nocm", "points", ("C4", 2048), {"finish_k": -1}),
    ("c4_2048", "points", ("C4", 2048), {}),
    ("c4_8192", "points", ("C4", 8192), {}),
    ("w_ties_1031", "weights", ("ties", 1031), {}),
    ("w_ties_1031_nocache", "weights", ("ties", 1031), {"topk": -1}),
    ("w_c3_4096", "weights", ("C3", 4096), {}),
]

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_multirank_gpu import CASES  # noqa: E402

CFGS += [c for c in CASES if c[1] == "points" and "metric" not in c[3] or c[1] == "weights" and "sense" not in c[3]]

if __name__ == "__main__":
    sel = sys.argv[1:]
    if sel and sel[0] == "--seq":
        cfgs = [c for c in CASES if c[0] in sel[1:]] if len(sel) > 1 else [c for c in CFGS if c in CASES]
        mgr = mp.Manager(); out = mgr.dict()
        try:
            mp.spawn(worker, args=(2, port(), cfgs, out), nprocs=2, join=True)
        except Exception as e:
            print("spawn:", str(e).splitlines()[-1][:200])
        sys.exit(0)
    for cfg in CFGS:
        if sel and cfg[0] not in sel:
            continue
        mgr = mp.Manager(); out = mgr.dict()
        try:
            mp.spawn(worker, args=(2, port(), [cfg], out), nprocs=2, join=True)
        except Exception as e:
            print("spawn:", str(e).splitlines()[-1][:200])
        print(cfg[0], dict(out), flush=True)
