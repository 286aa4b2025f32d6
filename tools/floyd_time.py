# time appd_floyd_weights (NEXT-2) at a few sizes; prints ms and (min,max) updates/s
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_07058_b200 as P
from synth import generators as G
sizes = [int(x) for x in sys.argv[1:]] or [2048, 4096, 8192]
c = P.Context(timing=True)
for n in sizes:
    W = torch.from_numpy(np.ascontiguousarray(G.random_weights(n, 7, "uniform"), np.float32)).cuda()
    M = torch.empty((n, n), device="cuda")
    c.floyd_weights(W, M); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); c.floyd_weights(W, M); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    Mb = c.solve_weights(W); torch.cuda.synchronize()
    same = torch.equal(M.view(torch.int32), Mb.view(torch.int32))
    print(f"floyd n={n}: {ms:.2f} ms  {n**3/ms/1e9:.2f} T relax/s  equals Boruvka path: {same}  stats {c.stats()['kernel_launches']} launches")
