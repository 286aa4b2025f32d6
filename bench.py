"""Benchmark: APPD entries/s of the full solve on the BASELINE workload (C4 by default).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference] [--workload C4]

One step = one appd_solve_points / appd_solve_weights call: validation, MST (Boruvka
rounds), edge sort, dendrogram, fill prep and the fill of the full n x n APPD (this
rank's row block for N > 1), inputs resident in HBM.  N > 1 runs under torchrun, one
process per GPU; the fill is row-sharded and the Boruvka rows are sharded with one
NCCL all-reduce(min) per round.  Rank 0 prints one JSON line.

--impl reference times the CPU oracle (oracle/, Algorithm 4, one core) on a bounded
sample of the same workload: the first n_s points (n_s chosen so a step takes seconds).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "APPD entries/s (n²/s) and % of HBM roofline at 1/2/4/8 B200"
UNIT = "entries/s"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "sm_max_mhz": d.get("sm_max_mhz", 1965.0), "source": "measured"}
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback"}


class ClockSampler:
    """SM clock and throttle reasons polled through NVML every ~2 ms while the timed region
    runs (nvidia-smi's 100 ms loop is longer than the whole timed region)."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
               "hw_power_brake": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.running = False
        self.nv = None
        self.t = None

    def start(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
            return
        self.running = True
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv = self.nv
        while self.running:
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, attr in self.REASONS.items():
                    if r & getattr(nv, attr, 0):
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def clear(self):
        self.samples = []
        self.reasons = set()

    def stop(self):
        self.running = False
        if self.t:
            self.t.join(timeout=2)
        sm = list(self.samples)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": getattr(self, "max_mhz", None), "reasons": sorted(self.reasons), "samples": len(sm),
                "source": "NVML (nvmlDeviceGetClockInfo SM, clocks event reasons) every ~2 ms during the timed steps"}


def load_input(workload: str):
    from synth import generators as G

    c = G.CONFIGS[workload]
    return G.config(workload), c


def oracle_sample(workload: str, n_s: int):
    """Time the oracle (Algorithm 4 as it stands, one thread) on the first n_s rows of the workload."""
    import numpy as np

    import oracle
    from synth import generators as G

    A, c = load_input(workload)
    sub = np.ascontiguousarray(A[:n_s]) if c["mode"] == "points" else np.ascontiguousarray(A[:n_s, :n_s])
    with PinnedToCore0():
        t = time.perf_counter()
        if c["mode"] == "points":
            oracle.appd_points(sub)
        else:
            oracle.appd_weights(sub)
        return time.perf_counter() - t


def sample_size(workload: str, seconds: float) -> int:
    """n_s such that the oracle sample takes about `seconds` (measured at a small size, scaled n^2)."""
    from synth import generators as G

    c = G.CONFIGS[workload]
    n0 = min(2048, c["n"])
    t0 = oracle_sample(workload, n0)
    n_s = int(n0 * (seconds / max(t0, 1e-3)) ** 0.5)
    n_s = max(256, min(c["n"], n_s // 256 * 256))
    return n_s


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from synth import generators as G

    c = G.CONFIGS[args.workload]
    n_s = sample_size(args.workload, args.ref_seconds)
    for _ in range(args.warmup):
        oracle_sample(args.workload, min(n_s, 1024))
    times = [oracle_sample(args.workload, n_s) for _ in range(args.steps)]
    T = sum(times)
    value = args.steps * n_s * n_s / T
    sample = f"first {n_s} of the {c['n']} {'points' if c['mode'] == 'points' else 'vertices'} of {args.workload} " \
             f"({c['desc']}), full Algorithm 4 (Prim, sort, remove/traverse/copy), one step per sample"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * T / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        # the same workload as the CUDA arm's line; each step is the bounded sample below
        "config": {"workload": args.workload, "desc": c["desc"], "n": c["n"], "d": c.get("d", 0), "mode": c["mode"],
                   "sample_n": n_s},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                         "host": host_facts(), "pinned": "core 0 (sched_setaffinity, as taskset -c 0)",
                         **full_config_oracle(args.workload)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_native(args):
    import numpy as np
    import torch

    import paper_2407_07058_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    nccl_id = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        from paper_2407_07058_b200.distributed import broadcast_nccl_id

        nccl_id = broadcast_nccl_id()

    A, c = load_input(args.workload)
    n = c["n"]
    points = c["mode"] == "points"
    # one explicit stream for torch (L2 flush, events, copies) and the library: the legacy
    # default stream's handle is 0, which the library would replace by a private stream,
    # leaving the flush unordered with the solve
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    assert stream.cuda_stream != 0
    ctx = P.Context(device=local, stream=stream.cuda_stream, rank=rank, world=world, nccl_id=nccl_id, timing=True,
                    metric=args.metric)
    row0, rows = ctx.row_range(n)
    if points:
        Xd = torch.from_numpy(A).cuda()
    else:
        Xd = torch.from_numpy(np.ascontiguousarray(A[row0:row0 + rows])).cuda()
    del A
    M = torch.empty((rows, n), dtype=torch.float32, device="cuda")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 1 GiB > 126 MB L2

    def step():
        if points:
            ctx.solve_points(Xd, M)
        else:
            ctx.solve_weights(Xd, M)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # context for the fill's roofline: the pure-write rate of this GPU on the same buffer
    # (torch zero_ of M, best of 3; outside the timed region)
    wts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        M.zero_()
        b.record(stream)
        torch.cuda.synchronize()
        wts.append(a.elapsed_time(b))
    write_gbs = M.numel() * 4 / (min(wts) / 1000) / 1e9
    step()  # M holds the APPD again
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    stats = []
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    for s in range(args.steps):
        flush.fill_(float(s))  # L2 flush between timed steps (outside the events)
        ev[s][0].record(stream)
        step()
        ev[s][1].record(stream)
        stats.append(ctx.stats())
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    T = sum(step_ms)
    if dist:
        t = torch.tensor([T], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        T = float(t.item())
    value = args.steps * n * n / (T / 1000.0)  # whole job: all ranks' rows

    # dominant kernel of the step and its roofline
    pk = peaks()
    fill_ms = statistics.mean(s["ms_fill"] for s in stats)
    mst_ms = statistics.mean(s["ms_mst"] for s in stats)
    fill_bytes = rows * n * 4
    fill_gbs = fill_bytes / (fill_ms / 1000) / 1e9
    rounds = stats[-1]["rounds"]
    roofline = {"bound": "hbm", "achieved": fill_gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": fill_gbs / pk["hbm_gbs"], "traffic": None, "kernel": "k_fill",
                "algorithmic_bytes_per_launch": fill_bytes, "avg_launch_ms": fill_ms,
                "peak_source": pk["source"]}
    stage_ms = {k: statistics.mean(s[k] for s in stats) for k in
                ("ms_validate", "ms_mst", "ms_sort", "ms_dendrogram", "ms_prep", "ms_fill", "ms_total",
                 "ms_tcscan")}
    roofline["write_only_peak_gbs"] = write_gbs
    roofline["frac_of_write_only_peak"] = fill_gbs / write_gbs
    roofline["write_only_peak_source"] = "torch zero_ of the 16 GiB output buffer, best of 3 (pure stores; the copy peak counts reads and writes)"
    fill_roof = {"kernel": "k_fill", "achieved_gbs": fill_gbs, "peak_gbs": pk["hbm_gbs"],
                 "frac": fill_gbs / pk["hbm_gbs"], "avg_launch_ms": fill_ms, "algorithmic_bytes_per_launch": fill_bytes}
    tc_ms = statistics.mean(s["ms_tcscan"] for s in stats)
    tc_launches = stats[-1]["tcscan_launches"]
    tc_info = None
    if points and tc_launches:
        # tensor-core scans (round 0 cache build + component-matrix pass): the algorithmic
        # work is the Gram term -2 X^T X, 2*d flops per (row, column) pair per launch;
        # fp16 inputs run at the bf16 dense rate
        flops = statistics.mean(s["tcscan_flops"] for s in stats) / tc_launches
        avg = tc_ms / tc_launches
        ach = flops / (avg / 1000) / 1e12
        mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
        # the burst figure: each tensor pass is a sub-millisecond kernel inside a ~5 ms step
        # at the maximum SM clock (B200_PROFILING.md: burst for a kernel timed alone)
        peak_tc = json.load(open(mp)).get("bf16_tflops", 1638.1) if os.path.exists(mp) else 1638.1
        # the MMAs also carry the norm augmentation: K = ceil(d/16)*16 + 16 per pair, so the
        # executed rate is K/d times the algorithmic one; the measured cuBLAS peak is below
        # the hardware's nominal 2250 TFLOP/s dense fp16, hence frac can exceed 1
        kk = ((c["d"] + 15) // 16) * 16 + 16
        mma = ach * kk / c["d"]
        tc_info = {"bound": "tensor", "achieved": ach, "peak": peak_tc, "unit": "TFLOP/s", "frac": ach / peak_tc,
                   "kernel": "k_tcf_scan", "algorithmic_flops_per_launch": flops, "avg_launch_ms": avg,
                   "launches_per_step": tc_launches, "ms_per_step": tc_ms,
                   "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst; fp16 runs at the bf16 rate)",
                   "mma_k": kk, "mma_tflops_executed": mma, "nominal_peak": 2250.0,
                   "frac_of_nominal_executed": mma / 2250.0}
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        tj = json.load(open(tp)).get(args.workload, {}).get("k_fill")
        if tj and tj.get("rows") == rows and tj.get("n") == n:
            traffic = tj["dram_bytes_per_launch"]
    if tc_info and tc_ms > fill_ms:
        roofline = dict(tc_info, traffic=None, fill=fill_roof)
    else:
        roofline["traffic"] = traffic
        roofline["traffic_source"] = "profiles/traffic.json (ncu --set full: dram__bytes_read.sum + dram__bytes_write.sum)"
        if tc_info:
            roofline["tensor_scan"] = tc_info
    if points and not tc_launches and mst_ms > fill_ms:
        # exact FP32 MST scan: 2*d lane-ops per (row, column) pair per Boruvka pass, ALU bound
        d = c["d"]
        sm_count = torch.cuda.get_device_properties(local).multi_processor_count
        clk = (clocks["sm_mhz"] or pk["sm_max_mhz"])
        peak_alu = sm_count * 128 * clk * 1e6 / 1e12  # T lane-ops/s (FP32 pipe, 128 lanes/SM/clk)
        ops = 2 * d * rows * n * rounds
        ach = ops / (mst_ms / 1000) / 1e12
        roofline = {"bound": "alu", "achieved": ach, "peak": peak_alu, "unit": "Tlane-op/s", "frac": ach / peak_alu,
                    "traffic": None, "kernel": "k_scan_points (all Boruvka rounds)",
                    "algorithmic_ops_per_solve": ops, "avg_ms_per_solve": mst_ms,
                    "peak_source": f"{sm_count} SM x 128 FP32 lanes x {clk} MHz (median SM clock under load)",
                    "fill": fill_roof}

    # end to end through the public API with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        Xh = (torch.from_numpy(load_input(args.workload)[0]) if points else
              torch.from_numpy(np.ascontiguousarray(load_input(args.workload)[0][row0:row0 + rows])))
        Xh = Xh.pin_memory()
        Mh = torch.empty((rows, n), dtype=torch.float32).pin_memory()
        ke = max(1, min(args.steps, args.e2e_steps))
        fn = ctx.solve_points_host if points else ctx.solve_weights_host
        fn(Xh, Mh)  # warm
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(ke):
            fn(Xh, Mh)
        te = time.perf_counter() - t0
        if dist:
            t = torch.tensor([te], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        e2e = {"value": ke * n * n / te, "unit": UNIT, "h2d_bytes_per_step": int(Xh.numel() * 4),
               "d2h_bytes_per_step": int(Mh.numel() * 4), "steps": ke, "ms_per_step": 1000 * te / ke}
        del Mh, Xh

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        n_s = sample_size(args.workload, args.ref_seconds)
        ts = oracle_sample(args.workload, n_s)
        cpu = {"value": n_s * n_s / ts, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"first {n_s} of {n} rows of {args.workload}, full Algorithm 4, {ts:.1f} s",
               "host": host_facts(), "pinned": "core 0 (sched_setaffinity, as taskset -c 0)",
               **full_config_oracle(args.workload)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": T / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.workload, "desc": c["desc"], "n": n, "d": c.get("d", 0), "mode": c["mode"],
                       **({"metric": ["euclidean", "manhattan", "chebyshev"][args.metric]} if args.metric else {}),
                       "parallelism": f"rows{world}", "l2": "1 GiB write between timed steps (outside events)",
                       "timing": "per-step CUDA events on the solve stream, max over ranks"},
            "roofline": roofline,
            "roofline_strict_frac": ((4 * n * n / world + (4 * n * c.get("d", 0) if points else 4 * n * n / world))
                                     / (pk["hbm_gbs"] * 1e9)) / (T / args.steps / 1000),
            "stage_ms": stage_ms,
            "boruvka_rounds": rounds,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(sum(s["kernel_launches"] for s in stats)),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist:
        dist.destroy_process_group()
    return 0


def run_floyd(args):
    """NEXT-2: appd_floyd_weights, the paper's minimax Floyd-Warshall, on a
    seeded uniform n x n W (one GPU).  Metric: (min, max) relaxations per second (n^3 per
    solve).  Roofline: ALU pipe, 1.5 FMNMX instructions per relaxation (two maxima and one
    3-input minimum per pair of k) against 64 lanes/clk/SM x SMs x the sampled SM clock."""
    import numpy as np
    import torch
    import paper_2407_07058_b200 as P
    import oracle
    from synth import generators as G
    n = args.floyd
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    W = torch.from_numpy(np.ascontiguousarray(G.random_weights(n, 7, "uniform"), np.float32)).to(dev)
    M = torch.empty((n, n), device=dev)
    ctx = P.Context(timing=True)
    for _ in range(max(args.warmup, 1)):
        ctx.floyd_weights(W, M)
    torch.cuda.synchronize()
    sampler = ClockSampler(0)
    sampler.start()
    ts = []
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.floyd_weights(W, M)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    clocks = sampler.stop()
    ms = statistics.mean(ts)
    relax = float(n) ** 3 / (ms / 1000)
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    pk = peaks()
    clk = clocks["sm_mhz"] or pk["sm_max_mhz"]
    peak_alu = sm_count * 64 * clk * 1e6 / 1e12
    ach = relax * 1.5 / 1e12
    # oracle (the literal triple loop, one core) on a bounded sample size
    ns = 384
    Ws = G.random_weights(ns, 7, "uniform")
    t0 = time.perf_counter()
    oracle.floyd(Ws)
    tcpu = time.perf_counter() - t0
    line = {"metric": "minimax Floyd-Warshall relaxations/s (NEXT-2)", "value": relax, "unit": "relaxations/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"floyd_n{n}", "n": n, "weights": "uniform open (0,1), seed 7"},
            "roofline": {"bound": "alu", "achieved": ach, "peak": peak_alu, "unit": "T inst-lanes/s",
                         "frac": ach / peak_alu, "traffic": None, "kernel": "k_fw_tiles",
                         "peak_source": "64 ALU lanes/clk/SM (FMNMX) x SMs x sampled SM clock (B200_PROFILING.md)"},
            "cpu_baseline": {"value": float(ns) ** 3 / tcpu, "unit": "relaxations/s", "cores": 1, "kind": "oracle",
                             "sample": f"oracle_floyd at n={ns} ({tcpu:.2f} s)"},
            "gpu_launches": ctx.stats()["kernel_launches"], "clocks": clocks}
    print(json.dumps(line))
    return 0


def full_config_oracle(workload: str) -> dict:
    """The oracle timed ONCE on the whole workload on a GPU box's host (one core; committed
    under profiles/, written by tools/oracle_full.py), reported beside the bounded sample:
    the sample's n^2 scaling is optimistic (the copy phase loses cache locality at full n)."""
    p = os.path.join(ROOT, "profiles", "oracle_full.json")
    if not os.path.exists(p):
        return {}
    rec = json.load(open(p)).get(workload)
    if not rec:
        return {}
    return {"full_config": {"value": rec["n"] ** 2 / rec["seconds"], "unit": UNIT, "seconds": rec["seconds"],
                            "phases_s": rec.get("phases_s"), "host": rec.get("host"), "when": rec.get("when"),
                            "source": "profiles/oracle_full.json (tools/oracle_full.py on the GPU box)"}}


def relaunch_under_torchrun(n: int) -> int:
    """--gpus N > 1 without a torchrun environment: start N ranks (one process per GPU)
    with torch.distributed.run on 127.0.0.1 and return its exit code, so that
    `python bench.py --gpus N` measures N NCCL ranks, not one."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def host_facts() -> dict:
    """The host the CPU baseline ran on (cores, model, RAM)."""
    facts = {"nproc": os.cpu_count()}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                facts["cpu_model"] = line.split(":", 1)[1].strip()
                break
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                facts["ram_gib"] = round(int(line.split()[1]) / 2 ** 20, 1)
                break
    except OSError:
        pass
    return facts


class PinnedToCore0:
    """Run the single-threaded oracle pinned to core 0 (`taskset -c 0`)."""

    def __enter__(self):
        self.saved = None
        try:
            self.saved = os.sched_getaffinity(0)
            os.sched_setaffinity(0, {min(self.saved)})
        except (AttributeError, OSError):
            pass
        return self

    def __exit__(self, *a):
        if self.saved:
            os.sched_setaffinity(0, self.saved)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--ref-seconds", type=float, default=8.0, help="target seconds per oracle sample")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--floyd", type=int, default=0, help="NEXT-2: time appd_floyd_weights at this n instead")
    ap.add_argument("--metric", type=int, default=0, help="NEXT-3 points metric: 0 Euclidean, 1 Manhattan, 2 Chebyshev")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args.gpus)
    if args.floyd:
        return run_floyd(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_native(args)


if __name__ == "__main__":
    sys.exit(main())
