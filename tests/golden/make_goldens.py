"""Write the large-config goldens: FNV-1a-64 of the ORACLE's APPD rows, per block.

Calls only oracle/ (Algorithm 4) and synth/ (inputs); nothing from the CUDA path.
    python tests/golden/make_goldens.py C4            # full matrix, 16 GiB of RAM
    python tests/golden/make_goldens.py C5 0 16384    # rows [0, 16384) via the R5 row window
Output: tests/golden/<cfg>[_r<row0>].json with the input checksum, the block size and
one FNV-1a-64 per block of BLOCK rows (row-major float32 bytes).
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from synth import generators as G  # noqa: E402

BLOCK = 1024


def main():
    cfg = sys.argv[1]
    X = G.config(cfg)
    n = X.shape[0]
    row0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    R = int(sys.argv[3]) if len(sys.argv) > 3 else n
    t = time.time()
    if G.CONFIGS[cfg]["mode"] == "points":
        if row0 == 0 and R == n:
            M, st = oracle.appd_points(X, with_stats=True)
        else:
            M, st = oracle.appd_points_rows(X, row0, R, with_stats=True)
    else:
        M, st = oracle.appd_weights(X, 1, with_stats=True)
    dt = time.time() - t
    blocks = [oracle.fnv1a64(M[b:b + BLOCK]) for b in range(0, M.shape[0], BLOCK)]
    out = {
        "config": cfg,
        "n": n,
        "d": int(X.shape[1]) if G.CONFIGS[cfg]["mode"] == "points" else 0,
        "row0": row0,
        "rows": int(M.shape[0]),
        "block_rows": BLOCK,
        "input_fnv1a64": oracle.fnv1a64(X),
        "row_block_fnv1a64": [f"{b:016x}" for b in blocks],
        "writes": st["writes"],
        "oracle_seconds": {"mst": st["t_mst"], "sort": st["t_sort"], "copy": st["t_copy"], "total": dt},
        "made_by": "tests/golden/make_goldens.py (oracle/ Algorithm 4 only)",
    }
    name = f"{cfg}.json" if (row0 == 0 and R == n) else f"{cfg}_r{row0}.json"
    with open(os.path.join(HERE, name), "w") as f:
        json.dump(out, f, indent=1)
    print(name, dt, st)


if __name__ == "__main__":
    main()
