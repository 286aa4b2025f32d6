# one warm-up + one measured C4 solve (for ncu launch lists)
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_07058_b200 as P
from synth import generators as G
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
topk = int(sys.argv[2]) if len(sys.argv) > 2 else 0
fk = int(sys.argv[3]) if len(sys.argv) > 3 else 0
X = torch.from_numpy(np.ascontiguousarray(G.config(name), np.float32)).cuda()
c = P.Context(timing=True, topk=topk, finish_k=fk)
weights = G.CONFIGS[name]["mode"] == "weights"
for _ in range(2):
    M = c.solve_weights(X) if weights else c.solve_points(X); torch.cuda.synchronize()
print(c.stats())
