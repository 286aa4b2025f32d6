# time appd_solve_weights_f64 (NEXT-3) on the C3 recipe (n = 16384, fp64) against the fp32 path
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_07058_b200 as P
from synth import generators as G
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
W32 = torch.from_numpy(G.config("C3", n=n)).cuda()
W64 = W32.double()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
c = P.Context(timing=True)
arms = (("fp32", W32, c.solve_weights), ("fp64", W64, c.solve_weights_f64))
if os.environ.get("F64_ONLY"):
    arms = arms[1:]
for name, W, fn in arms:
    M = fn(W); torch.cuda.synchronize()
    ts, st = [], []
    for _ in range(5):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(W, M); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1)); st.append(c.stats())
    s = st[-1]
    keys = ("ms_validate", "ms_mst", "ms_sort", "ms_dendrogram", "ms_prep", "ms_fill")
    print(f"{name} n={n}: {statistics.median(ts):.3f} ms  " + "  ".join(f"{k[3:]} {statistics.median(x[k] for x in st):.3f}" for k in keys)
          + f"  rounds {s['rounds']} launches {s['kernel_launches']}")
    if name == "fp64":
        fill_ms = statistics.median(x["ms_fill"] for x in st)
        print(f"  fp64 fill {n*n*8/fill_ms/1e6:.0f} GB/s; MST {statistics.median(x['ms_mst'] for x in st):.3f} ms for {s['rounds']} rounds"
              f" = {s['rounds']*n*n*8/statistics.median(x['ms_mst'] for x in st)/1e6:.0f} GB/s of W reads")
