#!/usr/bin/env python
"""SkyCell skyline benchmark (BASELINE.json metric: skyline query ms & Gpoints/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

A step is one full skyline query (compute_skyline, refine.cpp:108-158) over one
synthetic dataset resident in HBM.  Default workload = BASELINE.json configs[1]:
independent-uniform n=1e8, d=4, float32 on the 2^-24 grid,
rho = default_rho(n, d) = 6, on one B200.

Multi-GPU: `--gpus N` (N > 1) runs one process per GPU.  Launched bare, the
script re-executes itself under `torch.distributed.run` with N ranks; under an
external torchrun it uses RANK/LOCAL_RANK/WORLD_SIZE.  Points are sharded by
index: rank r owns records [r*n/N, (r+1)*n/N) of the global
dataset and generates exactly those.  The default config is weak scaling
(1e8 points per GPU, so N=1 is C2 and N=8 is 8e8 points); `--config c4i` /
`c4c` is BASELINE's C4, n=1e9 in total split over the N GPUs (strong scaling).

Prints ONE JSON line (rank 0).  `value` = n_total / device time (CUDA events,
max over ranks), inputs already in HBM.  `e2e` = the same query through the
public C ABI with the coordinates in pinned host memory (H2D inside the timed
region) and the ids read back to the host.  `roofline` = the kernel with the
largest share of the step (K1 streaming pass, K4 candidate filter or K5
exact dominance), its algorithmic bytes against the measured HBM copy
bandwidth.  `cpu_baseline` = the unmodified reference library (oracle/_ref)
on this host's cores over the same workload where that is feasible.
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# name: (dist, n, d, scaling, description).  scaling "weak": n points per GPU;
# "strong": n points in total, split over the GPUs.
CONFIGS = {
    "c1": (0, 10**6, 4, "weak", "independent-uniform n=1e6 d=4 float32"),
    "c2": (0, 10**8, 4, "weak", "independent-uniform n=1e8 d=4 float32"),
    "c2c": (1, 10**8, 4, "weak", "correlated n=1e8 d=4 float32"),
    "c3": (2, 10**8, 6, "weak", "anti-correlated n=1e8 d=6 float32"),
    "c4i": (0, 10**9, 4, "strong", "independent-uniform n=1e9 d=4 float32"),
    "c4c": (1, 10**9, 4, "strong", "correlated n=1e9 d=4 float32"),
    "c4ishard": (0, 125_000_000, 4, "weak", "independent-uniform n=1e9/8 per GPU d=4 float32"),
    "c4cshard": (1, 125_000_000, 4, "weak", "correlated n=1e9/8 per GPU d=4 float32"),
}
for _d in range(2, 9):
    CONFIGS[f"c5d{_d}"] = (2, 10**8, _d, "weak", f"anti-correlated n=1e8 d={_d} float32")
DIST_NAMES = {0: "independent", 1: "correlated", 2: "anticorrelated"}
METRIC = "skyline query throughput (Gpoints/s), n=1e8 d=4 independent"
UNIT = "Gpoints/s"
# The CPU reference's host RAM is ~140 B/point: above this it
# runs a bounded sample of the same distribution instead of the whole job.
REF_MAX_N = 125_000_000
# Anti-correlated d >= 4 at n=1e8 does not finish on the CPU (O(S^2) serial
# merge, refine.cpp:98-99): the reference runs these sample sizes.
REF_SAMPLE = {"c3": 50_000, "c5d4": 10**7, "c5d5": 10**6, "c5d6": 50_000, "c5d7": 30_000, "c5d8": 20_000}
REF_BUDGET_S = 1200.0  # wall-clock cap of the reference arm's timed steps


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region by an NVML
    polling thread (every 10 ms; faster polling measurably contends with the
    CUDA driver on the sync-heavy large-skyline configs)."""
    REASONS = {  # nvmlClocksEventReason* bits
        "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4,
    }

    def __init__(self, device: int):
        self.device = device
        self.samples = []  # (sm_mhz, max_mhz, reasons bitmask)
        self.stop = threading.Event()
        self.thread = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def poll():
                while not self.stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((float(sm), float(mx), int(r)))
                    except Exception:
                        pass
                    time.sleep(0.010)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
        except Exception:
            self.thread = None
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        reasons = sorted({nm for (_, _, r) in self.samples for nm, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(s[0] for s in self.samples), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": reasons, "samples": len(self.samples), "source": "nvml"}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def job_shape(config: str, world: int, n_override: int = 0):
    """(dist, n_total, d, scaling, desc) of the whole job at `world` GPUs."""
    dist, n, d, scaling, desc = CONFIGS[config]
    if n_override:
        n, desc = n_override, desc + f" [n overridden: {n_override}{' per GPU' if scaling == 'weak' else ''}]"
    n_total = n * world if scaling == "weak" else n
    return dist, n_total, d, scaling, desc


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(gpus: int) -> int:
    """Re-execute this script under torch.distributed.run with `gpus` ranks
    (one process per GPU, rendezvous on 127.0.0.1).  Rank 0's JSON line is the
    only stdout line of the job."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ, SKYCELL_BENCH_CHILD="1", OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.run(cmd, env=env).returncode


# ------------------------------------------------------------ reference arm
def ref_workload(config: str, n_total: int):
    """(n the CPU reference runs, note): the job itself where feasible."""
    n = min(n_total, REF_SAMPLE.get(config, n_total), REF_MAX_N)
    note = "same workload" if n == n_total else f"bounded sample n={n} of the n={n_total} job"
    return n, note


def cpu_inputs(dist, n, d):
    """Reference generator + 2^-24 quantisation; excluded
    from timing.  The reference is fed Dataset{(double)x, [0,1]^d}."""
    from oracle.oracle import Reference, quantize_f32
    ref = Reference()
    v = ref.generate(dist, n, d, 42, workers=0)
    x64 = quantize_f32(v).astype(np.float64)
    del v
    return ref, x64


def cpu_reference_step(ref, x64, d, rho):
    t = time.perf_counter()
    r = ref.compute_skyline(x64, np.zeros(d), np.ones(d), rho, 1, True, workers=0)
    return time.perf_counter() - t, r


def run_reference_arm(args):
    """The unmodified reference (oracle/_ref: compute_skyline, Mode::kParallel,
    ThreadPool(0) = every host thread) on the same config as our arm."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    dist, n_total, d, scaling, desc = job_shape(args.config, world, args.n)
    n, note = ref_workload(args.config, n_total)
    rho = args.rho or _default_rho(n, d)
    ref, x64 = cpu_inputs(dist, n, d)
    cores = os.cpu_count()
    # one untimed warm-up (page faults of the first call); a CPU library has no
    # JIT or caches to warm beyond that, and each call is tens of seconds
    for _ in range(min(args.warmup, 1)):
        cpu_reference_step(ref, x64, d, rho)
    times, stages, t_start = [], [], time.perf_counter()
    for _ in range(args.steps):
        dt, r = cpu_reference_step(ref, x64, d, rho)
        times.append(dt)
        stages.append(r.times)
        if time.perf_counter() - t_start + dt > REF_BUDGET_S:
            break
    ms = 1000.0 * statistics.mean(times)
    value = n / (ms / 1000.0) / 1e9
    sample = (f"{DIST_NAMES[dist]} n={n} d={d} rho={rho} ({note}); compute_skyline Mode::kParallel "
              f"ThreadPool(0) = {cores} threads; {len(times)} timed calls")
    st = {k: statistics.mean(s[k] for s in stages) for k in stages[0]}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": len(times), "steps_requested": args.steps, "warmup": min(args.warmup, 1),
        "ms_per_step": ms, "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (reference generator, seed 42, 2^-24 grid)",
        "config": {"workload": desc, "n": n, "n_job": n_total, "d": d, "rho": rho, "same_config": n == n_total,
                   "skyline_size": int(r.ids.size), "points_examined": r.points_examined},
        "stages_ms": st,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _default_rho(n, d):
    bw = max(1, int(n)).bit_length()
    return max(1, min(6, (bw - 1) // d))


# ------------------------------------------------------------------ our arm
def newest_profile(kernel_tag: str, config: str):
    """dram bytes per launch from the newest committed ncu --set full summary
    of this kernel at this config (profiles/<run>_<kernel_tag>_<config>.json)."""
    # newest = highest run tag (r1a < r2x < r3b < r4s ...; file times do not survive a checkout)
    profs = sorted(glob.glob(os.path.join(ROOT, "profiles", f"*_{kernel_tag}_{config}.json")))
    for p in reversed(profs):
        try:
            with open(p) as f:
                j = json.load(f)
            if j.get("dram_bytes_per_launch"):
                return float(j["dram_bytes_per_launch"]), os.path.relpath(p, ROOT)
        except Exception:
            pass
    return None, None


def run_ours(args):
    import torch

    import paper_2107_09993_b200 as sky

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist_id, n_total, d, scaling, desc = job_shape(args.config, world, args.n)
    eng = sky.Engine(local)
    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=dev)
        from paper_2107_09993_b200.dist import ShardedSkyline, shard_range
        runner = ShardedSkyline(eng, device=dev)
        begin, end = shard_range(n_total, rank, world)
    else:
        runner, begin, end = None, 0, n_total
    n_loc = end - begin
    rho = args.rho or sky.default_rho(n_total, d)
    # rank r generates exactly its records [begin, end) of the global dataset
    # (the reference generator's per-block streams, on the device)
    x = eng.generate(dist_id, n_total, d, 42, quantized=True, begin=begin, count=n_loc)
    ids_dev = torch.empty(max(n_loc, 1), dtype=torch.int32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    mn, mx = np.zeros(d), np.ones(d)
    stream = torch.cuda.current_stream()

    def step():
        if runner is None:
            return eng.skyline_raw(x, n_loc, d, mn, mx, rho, 1, True, ids_out=ids_dev, with_stats=True)
        return runner.skyline(x, n_loc, d, mn, mx, rho, begin, ids_out=ids_dev)

    for _ in range(max(3, args.warmup)):
        res = step()
    torch.cuda.synchronize()

    step_ms, launches, kern = [], 0, {"k1": [], "k4": [], "k5": []}
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)  # evict L2 between timed iterations (outside the timed region)
            if world > 1:
                torch.distributed.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res = step()
            e1.record(stream)
            torch.cuda.synchronize()
            if world > 1:
                torch.distributed.barrier()
            step_ms.append(e0.elapsed_time(e1))
            kern["k1"].append(res.stream_kernel_ms)
            kern["k4"].append(res.filter_kernel_ms)
            kern["k5"].append(res.dominance_ms)
            launches += res.kernel_launches
    ms = statistics.mean(step_ms)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = n_total / (ms / 1000.0) / 1e9
    sky_size = int(len(res.ids))

    # ---- e2e through the public API: pinned host coords -> ids on host
    # (H2D of the shard and D2H of the ids inside the timed region; under
    # torchrun every rank stages its own shard, max over ranks)
    hx = torch.empty((n_loc, d), dtype=torch.float32, pin_memory=True)
    hx.copy_(x)
    hx_np = hx.numpy()
    ids_host = torch.empty(max(n_loc, 1), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)

    def e2e_step():
        if runner is None:
            return eng.skyline_raw(hx_np, n_loc, d, mn, mx, rho, 1, True, ids_out=ids_host, with_stats=False)
        return runner.skyline(hx_np, n_loc, d, mn, mx, rho, begin, ids_out=ids_host)

    for _ in range(2):
        e2e_step()
    e2e_ms = []
    for _ in range(max(1, min(args.steps, 5))):
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r2 = e2e_step()
        torch.cuda.synchronize()
        e2e_ms.append(1000.0 * (time.perf_counter() - t0))
    e2e_mean = statistics.mean(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e_mean], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_mean = float(t.item())
    if rank == 0:
        assert len(r2.ids) == sky_size
    e2e = {"value": n_total / (e2e_mean / 1000.0) / 1e9, "unit": UNIT, "ms_per_step": e2e_mean,
           "h2d_bytes_per_step": n_loc * d * 4, "d2h_bytes_per_step": sky_size * 4,
           "path": "skycell_gpu_skyline_f32 (C ABI) from pinned host memory; under torchrun the sharded API"}

    # ---- roofline of the kernel with the largest share of the step
    peak, peak_src = measured_peaks()
    km = {k: statistics.mean(v) for k, v in kern.items()}
    row = 4 * d
    # algorithmic bytes per launch: K1 reads the n*d f32 coordinates once; K4
    # reads its input stream S1 (rows + id); K5 reads its set once (rows, id,
    # FP64 sum) -- SURVEY §8(d), DESIGN §3
    alg = {"k1": row * n_loc, "k4": (row + 4) * res.survivors_stream, "k5": (row + 12) * res.survivors_filter}
    names = {"k1": "k_stream (K1 streaming pass)", "k4": "k_cand_head + k_candidates (K4 candidate filter)",
             "k5": "K5 exact dominance (build + query)"}
    tags = {"k1": "k1_kstream", "k4": "k4_candhead", "k5": "k5_dominance"}
    top = max(km, key=lambda k: km[k])
    achieved = alg[top] / (km[top] / 1000.0) / 1e9 if km[top] > 0 else 0.0
    traffic, traffic_src = newest_profile(tags[top], args.config)
    roofline = {"bound": "hbm", "kernel": names[top], "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "algorithmic_bytes_per_launch": alg[top],
                "kernel_ms": km[top], "kernel_share_of_step": km[top] / statistics.mean(step_ms),
                "peak_source": peak_src, "traffic_source": traffic_src,
                "kernels_ms": km, "kernels_share": {k: v / statistics.mean(step_ms) for k, v in km.items()},
                "k1_frac": (alg["k1"] / (km["k1"] / 1000.0) / 1e9 / peak) if km["k1"] > 0 else None,
                "query_frac": (row * n_total + 4 * sky_size) / (ms / 1000.0) / 1e9 / peak / world}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        n_cpu, note = ref_workload(args.config, n_total)
        crho = _default_rho(n_cpu, d)
        ref, x64 = cpu_inputs(dist_id, n_cpu, d)
        dt, rr = cpu_reference_step(ref, x64, d, crho)
        cpu = {"value": n_cpu / dt / 1e9, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
               "sample": f"{DIST_NAMES[dist_id]} n={n_cpu} d={d} rho={crho} ({note}), one compute_skyline call "
                         f"(Mode::kParallel, ThreadPool(0)), {dt:.2f} s",
               "same_config": n_cpu == n_total, "skyline_size": int(rr.ids.size),
               "ids_match": bool(n_cpu == n_total and rr.ids.size == sky_size)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32 coords (exact FP64 sums)",
            "data": "synthetic (reference generator streams on device, seed 42, 2^-24 grid)",
            "config": {"workload": desc + (f" x {world} GPUs" if world > 1 and scaling == "weak" else ""),
                       "name": args.config, "n_total": n_total, "d": d, "rho": rho, "skyline_size": sky_size,
                       "points_examined": res.points_examined,
                       "parallelism": f"{world} GPU(s), points sharded by index" if world > 1 else "1 GPU",
                       "l2": "inputs (4*d*n bytes) larger than L2 and a 256 MB L2 flush between timed steps"},
            "e2e": e2e, "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "stages_ms": {"grid": res.times.grid_ms, "shrink": res.times.shrink_ms, "refine": res.times.refine_ms},
            "survivors": {"stream": res.survivors_stream, "filter": res.survivors_filter},
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        torch.distributed.destroy_process_group()


def launch_check(args):
    """`--launch-check`: the multi-rank plumbing without a GPU (gloo): every
    rank joins the process group, the ranks agree on the job shape and rank 0
    prints one JSON line.  tests/test_bench_launch.py runs it on CPU."""
    import torch
    import torch.distributed as tdist
    rank, world, _ = dist_env()
    tdist.init_process_group("gloo")
    from paper_2107_09993_b200.dist import shard_range
    dist_id, n_total, d, scaling, _ = job_shape(args.config, world, args.n)
    b, e = shard_range(n_total, rank, world)
    t = torch.tensor([e - b], dtype=torch.int64)
    tdist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "n_gpus": world, "n_total": n_total, "points_covered": int(t.item()),
                          "scaling": scaling, "launch_check": True}), flush=True)
    tdist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--rho", type=int, default=0)
    ap.add_argument("--n", type=int, default=0, help="override the config's n (debugging)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--launch-check", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    _, world, _ = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args.gpus))
    if "WORLD_SIZE" in os.environ and world != args.gpus and not os.environ.get("SKYCELL_BENCH_CHILD"):
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; using the launched world", file=sys.stderr)
    if args.launch_check:
        launch_check(args)
    elif args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
