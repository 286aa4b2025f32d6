# per-config solve times (2 warm solves, stats of the last)
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_07058_b200 as P
from synth import generators as G
for name in sys.argv[1:] or ["C1", "C2", "C3"]:
    A = np.ascontiguousarray(G.config(name))
    mode = G.CONFIGS[name]["mode"]
    c = P.Context(timing=True)
    t = torch.from_numpy(A).cuda()
    for _ in range(3):
        M = c.solve_points(t) if mode == "points" else c.solve_weights(t)
    torch.cuda.synchronize()
    st = c.stats()
    print(name, {k: round(st[k], 4) if isinstance(st[k], float) else st[k] for k in
                 ["n", "rounds", "ms_validate", "ms_mst", "ms_sort", "ms_dendrogram", "ms_prep", "ms_fill", "ms_total", "cm_k", "rescan_rows"]}, flush=True)
    del M, t
    c.close()
    torch.cuda.empty_cache()
