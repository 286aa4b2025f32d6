"""NEXT-4: time appd_solve_points_sink on the C5 recipe at n = 2^18 (256 GiB of output)
with a sink that only counts rows (the PCIe copy of every block is inside the call)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_07058_b200 as P
from synth import generators as G

n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
X = torch.from_numpy(G.c5_points(n, 16, 4))
rows = [0]
def sink(r0, blk):
    rows[0] += blk.shape[0]
with P.Context(timing=True) as c:
    t = time.perf_counter()
    c.solve_points_sink(X, sink, 1024)
    dt = time.perf_counter() - t
    st = c.stats()
print(f"n={n}: {dt:.2f} s wall, rows {rows[0]}, output {n * n * 4 / 2**30:.0f} GiB -> {n * n * 4 / dt / 1e9:.1f} GB/s; "
      f"rounds {st['rounds']} mst {st['ms_mst']:.1f} ms dendrogram {st['ms_dendrogram']:.1f} ms fill+copy {st['ms_fill']:.0f} ms")
