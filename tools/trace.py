"""GPU timeline of one solve from the development library (APPD_TRACE, dev builds only).

Records an event after every launch and every host synchronisation; prints, per launch
site, the host issue time and the GPU time since the previous event (kernel + idle gap).
    APPD_LIB=paper_2407_07058_b200/lib/libappd_dev.so APPD_TRACE=1 python tools/trace.py C4
Only the last solve's trace is of interest (earlier ones are warm-ups).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_07058_b200 as P  # noqa: E402
from synth import generators as G  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C4"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    A = np.ascontiguousarray(G.config(name))
    points = G.CONFIGS[name]["mode"] == "points"
    n = A.shape[0]
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    t = torch.from_numpy(A).cuda()
    M = torch.empty((n, n), dtype=torch.float32, device="cuda")
    with P.Context(stream=s.cuda_stream) as c:
        for i in range(reps):
            print(f"=== solve {i}", file=sys.stderr, flush=True)
            c.solve_points(t, M) if points else c.solve_weights(t, M)
            torch.cuda.synchronize()


if __name__ == "__main__":
    main()
