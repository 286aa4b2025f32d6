"""C4 solve time under engine parameters (topk, finish_k): median of 5 warm solves."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_07058_b200 as P
from synth import generators as G
X = torch.from_numpy(G.config("C4")).cuda()
M = torch.empty((X.shape[0], X.shape[0]), device="cuda")
for topk, fk in [(8, 0), (4, 0), (16, 0), (8, 64), (4, 64), (8, -1)]:
    with P.Context(timing=True, topk=topk, finish_k=fk) as c:
        ts = []
        for _ in range(6):
            c.solve_points(X, M)
            ts.append(c.stats())
        st = ts[-1]
        med = lambda k: statistics.median(s[k] for s in ts[1:])
        print(f"topk {topk:3d} finish_k {fk:4d}: total {med('ms_total'):.3f} mst {med('ms_mst'):.3f} ms rounds {st['rounds']} "
              f"cm_k {st['cm_k']} rescan_rows {st['rescan_rows']} tcscan {med('ms_tcscan'):.3f}", flush=True)
