"""One warm + one timed C4 solve (for ncu launch lists)."""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2407_07058_b200 as P
from synth import generators as G
eng = int(sys.argv[1]) if len(sys.argv) > 1 else 0
X = torch.from_numpy(G.config('C4')).cuda()
M = torch.empty((X.shape[0], X.shape[0]), device='cuda')
ctx = P.Context(points_engine=eng, timing=True)
for _ in range(2):
    ctx.solve_points(X, M)
torch.cuda.synchronize()
print(ctx.stats())
