import sys, os
os.environ['APPD_TC_VERIFY'] = '1'
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2407_07058_b200 as P
import oracle
from synth import generators as G
c2 = P.Context(points_engine=2)
for n, d, kind in [(1000, 16, 'dups'), (700, 7, 'wide'), (300, 5, 'blobs')]:
    X = G.random_points(n, d, 3, kind)
    print('===', n, d, kind, flush=True)
    a = c2.solve_points(torch.from_numpy(X).cuda()).cpu().numpy()
    o = oracle.appd_points(X)
    print('equal', (a.view(np.uint32) == o.view(np.uint32)).all(), c2.stats()['tc_candidates'], flush=True)
