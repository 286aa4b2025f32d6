import sys, os, time
sys.path.insert(0, "/root/repo")
import torch, numpy as np
import paper_2407_07058_b200 as P
from synth import generators as G
X = torch.from_numpy(G.config("C4")).cuda()
n = X.shape[0]
M = torch.empty((n, n), device="cuda")
stream = torch.cuda.current_stream()
flush = torch.empty(256 << 20, device="cuda")
for validate in (1, 0):
    ctx = P.Context(stream=stream.cuda_stream, timing=True, validate=validate)
    for _ in range(3): ctx.solve_points(X, M)
    torch.cuda.synchronize()
    rows = []
    for s in range(6):
        flush.fill_(float(s))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream); t0 = time.perf_counter(); ctx.solve_points(X, M); t1 = time.perf_counter(); b.record(stream)
        torch.cuda.synchronize()
        st = ctx.stats()
        rows.append((a.elapsed_time(b), st["ms_validate"], st["ms_mst"], st["ms_total"], (t1 - t0) * 1e3))
    r = np.median(np.array(rows), axis=0)
    print(f"validate={validate}: step {r[0]:.3f}  ms_validate {r[1]:.3f}  ms_mst {r[2]:.3f}  ms_total {r[3]:.3f}  host wall {r[4]:.3f}")
    ctx.close()
