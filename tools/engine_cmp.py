"""Points-engine comparison (exact FP32 vs tensor-core filter) per config: median whole-solve time."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_07058_b200 as P
from synth import generators as G
cases = [("C2", None), ("C2", 2048), ("C4", 2048), ("C4", 8192), ("C4", 16384), ("C5", 8192), ("C5", 32768)]
if len(sys.argv) > 1:  # e.g. C2:4096 C4:3072
    cases = [(a.split(":")[0], int(a.split(":")[1]) if ":" in a else None) for a in sys.argv[1:]]
for name, n in cases:
    X = torch.from_numpy(G.config(name, n=n)).cuda()
    nn = X.shape[0]
    M = torch.empty((nn, nn), device="cuda")
    res = {}
    for eng in (1, 2):
        with P.Context(points_engine=eng, variant=P.VARIANT_BORUVKA, timing=True) as c:
            ts = []
            for _ in range(6):
                c.solve_points(X, M)
                ts.append(c.stats())
            res[eng] = (statistics.median(s["ms_total"] for s in ts[1:]), statistics.median(s["ms_mst"] for s in ts[1:]), ts[-1]["rounds"])
    print(f"{name} n={nn} d={X.shape[1]}: exact total {res[1][0]:.3f} mst {res[1][1]:.3f} rounds {res[1][2]} | "
          f"tensor total {res[2][0]:.3f} mst {res[2][1]:.3f} rounds {res[2][2]}", flush=True)
