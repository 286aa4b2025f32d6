"""Prim vs Boruvka crossover ("two variants chosen by measurement").

Median device time of whole solves (CUDA events on the library's stream, 15 reps after
3 warm-ups) per variant, weights and points mode, at the sizes the Prim kernel fits.
Writes gpurun_out/crossover.txt (committed as profiles/r02/crossover.txt)."""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_07058_b200 as P  # noqa: E402
from synth import generators as G  # noqa: E402


def time_solve(ctx, fn, reps=15):
    s = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    rows = []
    cases = [("weights", n, 0) for n in (64, 128, 256, 300)]
    cases += [("points", n, 2) for n in (256, 512, 1024, 2048, 4096, 8192)]
    cases += [("points", n, 16) for n in (256, 1024, 2048)]
    cases += [("points", n, 64) for n in (256, 512, 768)]
    cases += [("C1", 256, 0), ("C2", 4096, 2)]
    for mode, n, d in cases:
        if mode == "C1":
            A, pts = G.config("C1"), False
        elif mode == "C2":
            A, pts = G.config("C2"), True
        elif mode == "weights":
            A, pts = G.random_weights(n, 5, "uniform"), False
        else:
            A, pts = G.random_points(n, d, 5, "blobs"), True
        At = torch.from_numpy(np.ascontiguousarray(A)).cuda()
        M = torch.empty((n, n), device="cuda")
        res = {}
        for name, var in (("prim", P.VARIANT_PRIM), ("boruvka", P.VARIANT_BORUVKA), ("auto", P.VARIANT_AUTO)):
            with P.Context(variant=var, timing=True) as ctx:
                f = (lambda: ctx.solve_points(At, M)) if pts else (lambda: ctx.solve_weights(At, M))
                try:
                    res[name] = time_solve(ctx, f)
                    res[name + "_stats"] = ctx.stats()
                except P.AppdError as e:
                    res[name] = float("nan")
        line = (f"{mode:8s} n={n:5d} d={d:3d}  prim {res['prim'] * 1000:8.1f} us  boruvka {res['boruvka'] * 1000:8.1f} us"
                f"  auto {res['auto'] * 1000:8.1f} us ({'prim' if res.get('auto_stats', {}).get('variant') == 1 else 'boruvka'})"
                f"  prim mst {res.get('prim_stats', {}).get('ms_mst', float('nan')) * 1000:7.1f} us")
        print(line, flush=True)
        rows.append(line)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/crossover.txt", "w") as f:
        f.write("# Prim vs Boruvka: median whole-solve device time (15 reps), tools/crossover.py\n")
        f.write("\n".join(rows) + "\n")


if __name__ == "__main__":
    main()
