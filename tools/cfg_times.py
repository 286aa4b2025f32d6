"""Per-config solve times on one B200 (committed as profiles/r02/cfg_times.txt).

Each line: median over 10 solves (after 3 warm-ups) of the device time around the call
(CUDA events on the library's stream, L2 flushed before each solve, timing stats off), and
the library's stage split from a separate timing=True context.
    python tools/cfg_times.py [C1 C2 C3 C4 C5]
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_07058_b200 as P  # noqa: E402
from synth import generators as G  # noqa: E402

STAGES = ["ms_validate", "ms_mst", "ms_sort", "ms_dendrogram", "ms_prep", "ms_fill", "ms_total"]


def run(name, label, **opts):
    A = np.ascontiguousarray(G.config(name))
    points = G.CONFIGS[name]["mode"] == "points"
    n = A.shape[0]
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    t = torch.from_numpy(A).cuda()
    M = torch.empty((n, n), dtype=torch.float32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.float32, device="cuda")
    times = []
    with P.Context(stream=s.cuda_stream, **opts) as c:
        f = (lambda: c.solve_points(t, M)) if points else (lambda: c.solve_weights(t, M))
        for _ in range(3):
            f()
        for i in range(10):
            flush.fill_(float(i))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            f()
            b.record(s)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        variant = c.stats()["variant"]
    with P.Context(stream=s.cuda_stream, timing=True, **opts) as c:
        for _ in range(3):
            f = (lambda: c.solve_points(t, M)) if points else (lambda: c.solve_weights(t, M))
            f()
        st = c.stats()
    med = statistics.median(times)
    line = (f"{label:28s} n={n:6d}  {med:8.3f} ms  ({n * n / (med / 1e3) / 1e9:8.1f} G entries/s)  "
            f"variant={'prim' if variant == 1 else 'boruvka'} rounds={st['rounds']} launches={st['kernel_launches']}  "
            + " ".join(f"{k[3:]}={st[k]:.3f}" for k in STAGES))
    print(line, flush=True)
    del M, t, flush
    torch.cuda.empty_cache()
    return line


def main():
    names = sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]
    lines = []
    for name in names:
        lines.append(run(name, name))
        if name == "C1":
            lines.append(run(name, "C1 (Boruvka forced)", variant=P.VARIANT_BORUVKA))
        if name == "C3":
            lines.append(run(name, "C3 (validation off)", validate=False))
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/cfg_times.txt", "w") as fh:
        fh.write("# tools/cfg_times.py: median of 10 solves (events around the call, L2 flushed), stage split "
                 "from a timing=True context\n")
        fh.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
