"""NEXT-4 goldens: the C5 recipe at n = 2^18 (256 GiB of output, more than any host or GPU
here holds), FNV-1a-64 of sampled 1024-row blocks of the ORACLE's APPD via the R5 row
window (Algorithm 4, writes filtered to the window).
Calls only oracle/ and synth/.

    python tests/golden/make_c5x_windows.py [workers]
"""
import json
import multiprocessing as mp
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

N, D, SEED, BLOCK = 262144, 16, 4, 1024
WINDOWS = [0, 131072, N - BLOCK]  # first, middle and last row blocks


def window(r0):
    import oracle
    from synth import generators as G

    X = G.c5_points(N, D, SEED)
    t = time.time()
    M, st = oracle.appd_points_rows(X, r0, BLOCK, with_stats=True)
    h = f"{oracle.fnv1a64(M):016x}"
    print(f"window {r0}: {time.time() - t:.0f} s", flush=True)
    return r0, h, st


def main():
    import oracle
    from synth import generators as G

    oracle.build()
    X = G.c5_points(N, D, SEED)
    t0 = time.time()
    with mp.get_context("spawn").Pool(int(sys.argv[1]) if len(sys.argv) > 1 else 3) as pool:
        res = pool.map(window, WINDOWS, chunksize=1)
    out = {"config": "C5x", "recipe": "synth.generators.c5_points(n=262144, d=16, seed=4)", "n": N, "d": D,
           "block_rows": BLOCK, "input_fnv1a64": oracle.fnv1a64(X),
           "blocks": {str(r0): h for r0, h, _ in res},
           "oracle_seconds": {str(r0): st["t_mst"] + st["t_sort"] + st["t_copy"] for r0, _, st in res},
           "wall_total": time.time() - t0,
           "made_by": "tests/golden/make_c5x_windows.py (oracle/ Algorithm 4, R5 windows, only)"}
    with open(os.path.join(HERE, "C5x_windows.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("C5x_windows.json", time.time() - t0)


if __name__ == "__main__":
    main()
