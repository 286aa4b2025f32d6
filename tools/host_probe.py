# host-side timeline of one C4 solve (APPD_DEBUG_HOST=1 marks in api.cu) next to the GPU stage events
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_07058_b200 as P
from synth import generators as G
X = torch.from_numpy(G.config("C4")).cuda()
M = torch.empty((X.shape[0], X.shape[0]), device="cuda")
ctx = P.Context(timing=True)
flush = torch.empty(256 << 20, device="cuda")
for i in range(4):
    flush.fill_(1.0)
    print(f"--- solve {i}", file=sys.stderr, flush=True)
    ctx.solve_points(X, M)
    torch.cuda.synchronize()
st = ctx.stats()
print({k: round(v, 3) for k, v in st.items() if k.startswith("ms_")}, file=sys.stderr)
