# C3 with validation on and off (report both)
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_07058_b200 as P
from synth import generators as G
W = torch.from_numpy(np.ascontiguousarray(G.config("C3"))).cuda()
for v in (True, False):
    c = P.Context(timing=True, validate=v)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); c.solve_weights(W); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    st = c.stats()
    print(f"C3 validate={int(v)}: {min(ts):.3f} ms (events around the call), stats total {st['ms_total']:.3f} "
          f"validate {st['ms_validate']:.3f} mst {st['ms_mst']:.3f} dendro {st['ms_dendrogram']:.3f} fill {st['ms_fill']:.3f}")
    c.close()
