"""Write tests/golden/C5.json: FNV-1a-64 of EVERY 1024-row block of the oracle's C5 APPD.

C5 (n = 131072, d = 16) has a 64 GiB output, more than this host's RAM, so the oracle
runs the R5 row-window variant (the same Algorithm 4, with
writes filtered to rows [r0, r0+R)) once per window, several windows in parallel.
Calls only oracle/ (Algorithm 4) and synth/ (inputs); nothing from the CUDA path.

    python tests/golden/make_c5_full.py [workers] [window_rows]
"""
import json
import multiprocessing as mp
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

BLOCK = 1024


def window(args):
    r0, R = args
    import oracle
    from synth import generators as G

    X = G.config("C5")
    t = time.time()
    M, st = oracle.appd_points_rows(X, r0, R, with_stats=True)
    blocks = [f"{oracle.fnv1a64(M[b:b + BLOCK]):016x}" for b in range(0, R, BLOCK)]
    dt = time.time() - t
    print(f"window r0={r0} R={R}: {dt:.0f} s", flush=True)
    return r0, blocks, st, dt


def main():
    workers = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
    import oracle
    from synth import generators as G

    oracle.build()
    X = G.config("C5")
    n = X.shape[0]
    assert n % R == 0 and R % BLOCK == 0
    t0 = time.time()
    with mp.get_context("spawn").Pool(workers) as pool:
        res = pool.map(window, [(r0, R) for r0 in range(0, n, R)], chunksize=1)
    res.sort(key=lambda r: r[0])
    blocks = [b for _, bl, _, _ in res for b in bl]
    assert len(blocks) == n // BLOCK
    out = {
        "config": "C5",
        "n": n,
        "d": int(X.shape[1]),
        "row0": 0,
        "rows": n,
        "block_rows": BLOCK,
        "input_fnv1a64": oracle.fnv1a64(X),
        "row_block_fnv1a64": blocks,
        "writes_per_window": res[0][2]["writes"],
        "window_rows": R,
        "oracle_seconds": {
            "per_window_mst": [r[2]["t_mst"] for r in res],
            "per_window_copy": [r[2]["t_copy"] for r in res],
            "wall_total": time.time() - t0,
            "workers": workers,
        },
        "made_by": "tests/golden/make_c5_full.py (oracle/ Algorithm 4, R5 windows, only)",
    }
    with open(os.path.join(HERE, "C5.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("C5.json", time.time() - t0)


if __name__ == "__main__":
    main()
