"""Cost of the multi-rank code path on one B200: each config solved by a plain world-1
context and by a world-1 context over a one-rank NCCL communicator (the path every rank
of an N-GPU run takes: agreement, verdict all-reduce, row-sharded scans, per-round
ncclAllReduce, polled waits).  Median of 10 solves, events around the call, L2 flushed.
    python tools/coll_times.py [C2 C3 C4 C5]   -> gpurun_out/coll_times.txt
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_07058_b200 as P  # noqa: E402
from synth import generators as G  # noqa: E402

STAGES = ["ms_validate", "ms_mst", "ms_sort", "ms_dendrogram", "ms_prep", "ms_fill", "ms_total"]


def timed(c, f, s, flush):
    for _ in range(3):
        f(c)
    times = []
    for i in range(10):
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        f(c)
        b.record(s)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    return statistics.median(times)


def checksum(M):
    # chunked (bounded memory): sums of the entries' bits and of a row-weighted mix
    h1 = h2 = 0
    V = M.view(torch.int32)
    for i in range(0, V.shape[0], 1024):
        v = V[i:i + 1024].to(torch.int64)
        h1 += int(v.sum().item())
        h2 += int((v * torch.arange(i + 1, i + 1 + v.shape[0], device=v.device)[:, None]).sum().item())
    return h1, h2


def run(name):
    A = np.ascontiguousarray(G.config(name))
    points = G.CONFIGS[name]["mode"] == "points"
    n = A.shape[0]
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    t = torch.from_numpy(A).cuda()
    M = torch.empty((n, n), dtype=torch.float32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.float32, device="cuda")
    f = (lambda c: c.solve_points(t, M)) if points else (lambda c: c.solve_weights(t, M))
    out = []
    ref = None
    for label, extra in (("plain world 1", {}), ("one-rank NCCL", "nccl")):
        opts = {"nccl_id": P.appd_get_nccl_unique_id()} if extra == "nccl" else {}
        M.fill_(float("nan"))  # same_M must come from this context's own writes
        with P.Context(stream=s.cuda_stream, timing=True, **opts) as c:
            med = timed(c, f, s, flush)
            st = c.stats()
            h = checksum(M)
        if ref is None:
            ref = h
        out.append(f"{name} {label:14s} n={n:6d}  {med:8.3f} ms  collectives={st['collectives']:3d} "
                   f"rounds={st['rounds']} launches={st['kernel_launches']}  same_M={h == ref}  "
                   + " ".join(f"{k[3:]}={st[k]:.3f}" for k in STAGES))
        print(out[-1], flush=True)
    del M, t, flush
    torch.cuda.empty_cache()
    return out


def main():
    names = sys.argv[1:] or ["C2", "C3", "C4", "C5"]
    lines = []
    for name in names:
        lines += run(name)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/coll_times.txt", "w") as fh:
        fh.write("# tools/coll_times.py: plain world-1 solve vs the multi-rank path over a one-rank NCCL "
                 "communicator (timing stats on; median of 10, L2 flushed)\n")
        fh.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
