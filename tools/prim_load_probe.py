import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_07058_b200 as P
from synth import generators as G
for n in (64, 128, 256, 300):
    W = torch.from_numpy(G.random_weights(n, 5, "uniform")).cuda()
    for val in (True, False):
        with P.Context(variant=P.VARIANT_PRIM, validate=val) as c:
            for _ in range(3):
                c.solve_weights(W)
            print("validate", val, flush=True)
