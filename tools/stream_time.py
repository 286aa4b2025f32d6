# time appd_solve_points_stream (NEXT-4) on C4 with a pinned host output
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_07058_b200 as P
from synth import generators as G
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
block = int(sys.argv[2]) if len(sys.argv) > 2 else 0
X = torch.from_numpy(np.ascontiguousarray(G.config(name), np.float32))
n = X.shape[0]
M = torch.empty((n, n), dtype=torch.float32).pin_memory()
c = P.Context(timing=True)
c.solve_points_stream(X, M, block)
ts = []
for _ in range(3):
    t0 = time.perf_counter(); c.solve_points_stream(X, M, block); ts.append(time.perf_counter() - t0)
st = c.stats()
t = min(ts)
print(f"{name} stream block={block}: {t*1e3:.1f} ms wall, {n*n/t:.3e} entries/s, {n*n*4/t/1e9:.1f} GB/s to host; "
      f"ms_fill(stream) {st['ms_fill']:.1f} ms_mst {st['ms_mst']:.2f}")
Xd = X.cuda()
Md = c.solve_points(Xd); torch.cuda.synchronize()
print("equal to device path:", torch.equal(Md.cpu().view(torch.int32), M.view(torch.int32)))
