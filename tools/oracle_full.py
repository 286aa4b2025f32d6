"""Time the oracle (oracle/, Algorithm 4, one thread pinned to core 0) ONCE on a whole
BASELINE workload on this host and record it in profiles/oracle_full.json (run on the
GPU box: the bench's cpu_baseline reports it beside its bounded sample).

    python tools/oracle_full.py C4
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import oracle  # noqa: E402
from synth import generators as G  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "C4"
    c = G.CONFIGS[wl]
    A = G.config(wl)
    with bench.PinnedToCore0():
        t = time.perf_counter()
        if c["mode"] == "points":
            M, st = oracle.appd_points(A, with_stats=True)
        else:
            M, st = oracle.appd_weights(A, 1, with_stats=True)
        dt = time.perf_counter() - t
    out_dir = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out_dir, exist_ok=True)
    rec = {wl: {"n": c["n"], "seconds": dt, "phases_s": {"mst": st["t_mst"], "sort": st["t_sort"], "copy": st["t_copy"]},
                "writes": st["writes"], "host": bench.host_facts(), "cores": 1,
                "pinned": "core 0", "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
                "first_block_fnv1a64": f"{oracle.fnv1a64(M[:1024]):016x}"}}
    json.dump(rec, open(os.path.join(out_dir, f"oracle_full_{wl}.json"), "w"), indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
