import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2407_07058_b200 as P
from synth import generators as G
X = G.random_points(3000, 16, 900, "blobs")
c = P.Context(timing=True)
M = c.solve_points(torch.from_numpy(X).cuda()); torch.cuda.synchronize()
print("ok", c.stats()["cm_k"])
