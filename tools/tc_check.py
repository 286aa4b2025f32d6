"""Quick TC-engine check: engine 2 vs engine 1 vs oracle on small cases; timing on C4."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2407_07058_b200 as P
import oracle
from synth import generators as G

def run(ctx, X):
    return ctx.solve_points(torch.from_numpy(X).cuda()).cpu().numpy()

c2 = P.Context(points_engine=2, timing=True)
c1 = P.Context(points_engine=1, timing=True)
cases = [(256, 2, 'uniform'), (300, 5, 'blobs'), (1000, 16, 'dups'), (513, 64, 'grid'), (700, 7, 'wide'), (2048, 64, 'blobs')]
ok = True
for n, d, kind in cases:
    X = G.random_points(n, d, 3, kind)
    a = run(c2, X); st = c2.stats()
    b = run(c1, X)
    o = oracle.appd_points(X)
    e2 = (a.view(np.uint32) == o.view(np.uint32)).all(); e1 = (b.view(np.uint32) == o.view(np.uint32)).all()
    ok &= bool(e2 and e1)
    print(f"n={n} d={d} {kind}: tc==oracle {e2} exact==oracle {e1} rounds={st['rounds']} cand={st['tc_candidates']} exact_rounds={st['exact_rounds']} engine={st['points_engine']}", flush=True)
for name in ['C2']:
    X = G.config(name)
    a = run(c2, X); st = c2.stats(); o = oracle.appd_points(X)
    print(name, (a.view(np.uint32) == o.view(np.uint32)).all(), st['tc_candidates'], st['rounds'], st['ms_scan'], st['ms_mst'])
X = G.config('C4')
Xt = torch.from_numpy(X).cuda()
M = torch.empty((X.shape[0], X.shape[0]), device='cuda')
for it in range(3):
    c2.solve_points(Xt, M)
    st = c2.stats()
    print('C4 tc', {k: st[k] for k in ('rounds','tc_candidates','tc_fallback_rows','exact_rounds','ms_scan','ms_mst','ms_dendrogram','ms_fill','ms_total')}, flush=True)
pi, h = c2.last_dendrogram(X.shape[0])
print('C4 h sum', float(np.sort(h).astype(np.float64).sum()), 'zeros', int((h==0).sum()))
print('ALL OK' if ok else 'MISMATCH')
