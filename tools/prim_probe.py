"""C1 / C2 with the Prim variant: stage times and host overhead (stats vs events)."""
import os, sys, time, statistics
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_07058_b200 as P
from synth import generators as G

for name in ("C1", "C2s"):
    A = G.config("C1") if name == "C1" else G.config("C2", n=1024)
    pts = name != "C1"
    s = torch.cuda.Stream(); torch.cuda.set_stream(s)
    At = torch.from_numpy(A).cuda(); n = A.shape[0]
    M = torch.empty((n, n), device="cuda")
    for var in (P.VARIANT_PRIM, P.VARIANT_BORUVKA):
        ctx = P.Context(variant=var, timing=True, stream=s.cuda_stream)
        f = (lambda: ctx.solve_points(At, M)) if pts else (lambda: ctx.solve_weights(At, M))
        for _ in range(5): f()
        torch.cuda.synchronize()
        ev, wall, st = [], [], []
        for _ in range(30):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter(); a.record(s); f(); b.record(s); torch.cuda.synchronize(); wall.append(time.perf_counter() - t0)
            ev.append(a.elapsed_time(b)); st.append(ctx.stats())
        keys = ("ms_validate", "ms_mst", "ms_sort", "ms_dendrogram", "ms_prep", "ms_fill", "ms_total")
        print(name, "prim" if var == 1 else "boruvka", "event %.1f us wall %.1f us" % (1000 * statistics.median(ev), 1e6 * statistics.median(wall)),
              {k: round(1000 * statistics.median(x[k] for x in st), 1) for k in keys}, "launches", st[-1]["kernel_launches"])
        ctx.close()
