#!/usr/bin/env python
"""SkyCell skyline benchmark (BASELINE.json metric: skyline query ms & Gpoints/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

A step is one full skyline query (compute_skyline, refine.cpp:108-158) over one
synthetic dataset resident in HBM.  Default workload = BASELINE.json configs[1]:
independent-uniform n=1e8, d=4, float32 on the 2^-24 grid,
rho = default_rho(n, d) = 6, on one B200.  Under torchrun (N > 1) the job is
the sharded query over N x 1e8 points (weak scaling: 1e8 points per GPU).

Prints ONE JSON line (rank 0).  `value` = n_total / device time (max over
ranks), inputs already in HBM.  `e2e` = the same query through the public C
ABI with the coordinates in pinned host memory (H2D inside the timed region)
and the ids read back to the host.  `roofline` = the streaming kernel K1
(4*d bytes of compulsory coordinate read per point) against the measured HBM
copy bandwidth.  `cpu_baseline` = the unmodified reference library
(oracle/_ref) on this host's cores over a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (dist, n per GPU, d, description)
    "c1": (0, 10**6, 4, "independent-uniform n=1e6 d=4 float32"),
    "c2": (0, 10**8, 4, "independent-uniform n=1e8 d=4 float32"),
    "c3": (2, 10**8, 6, "anti-correlated n=1e8 d=6 float32"),
    "c4i": (0, 125_000_000, 4, "independent-uniform n=1e9/8 per GPU d=4 float32"),
    "c4c": (1, 125_000_000, 4, "correlated n=1e9/8 per GPU d=4 float32"),
}
for _d in range(2, 9):
    CONFIGS[f"c5d{_d}"] = (2, 10**8, _d, f"anti-correlated n=1e8 d={_d} float32")
DIST_NAMES = {0: "independent", 1: "correlated", 2: "anticorrelated"}
METRIC = "skyline query throughput (Gpoints/s), n=1e8 d=4 independent"
UNIT = "Gpoints/s"


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
        self.smi = None

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


def cpu_reference_step(ref, x64, d, rho):
    t = time.perf_counter()
    r = ref.compute_skyline(x64, np.zeros(d), np.ones(d), rho, 1, True, workers=0)
    return time.perf_counter() - t, r


def cpu_sample(dist, d, n_sample):
    """Bounded sample of the workload for the CPU reference (same distribution,
    same quantisation, smaller n).  Data generation is excluded from timing."""
    from oracle.oracle import Reference, quantize_f32
    ref = Reference()
    v = ref.generate(dist, n_sample, d, 42, workers=0)
    x64 = quantize_f32(v).astype(np.float64)
    return ref, x64, ref.default_rho(n_sample, d)


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    dist, n_gpu, d, desc = CONFIGS[args.config]
    n_sample = args.cpu_sample or min(n_gpu, 10**7)
    ref, x64, rho = cpu_sample(dist, d, n_sample)
    cores = os.cpu_count()
    for _ in range(args.warmup):
        cpu_reference_step(ref, x64, d, rho)
    times = []
    for _ in range(args.steps):
        dt, _r = cpu_reference_step(ref, x64, d, rho)
        times.append(dt)
    ms = 1000.0 * statistics.mean(times)
    value = n_sample / (ms / 1000.0) / 1e9
    sample = (f"{DIST_NAMES[dist]} n={n_sample:.0e} d={d} rho={rho} (bounded sample of the {desc} workload), "
              f"compute_skyline Mode::kParallel ThreadPool(0)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (reference generator, seed 42, 2^-24 grid)",
        "config": {"workload": desc + f" [CPU sample n={n_sample}]", "n": n_sample, "d": d, "rho": rho},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch

    import paper_2107_09993_b200 as sky

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist_id, n_gpu, d, desc = CONFIGS[args.config]
    if args.n:
        n_gpu, desc = args.n, desc + f" [n overridden: {args.n} per GPU]"
    eng = sky.Engine(local)
    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        from paper_2107_09993_b200.dist import ShardedSkyline
        runner = ShardedSkyline(eng, device=torch.device(f"cuda:{local}"))
    else:
        runner = None
    n_total = n_gpu * world
    rho = args.rho or sky.default_rho(n_total, d)
    # rank r owns records [r*n_gpu, (r+1)*n_gpu) of the global dataset and
    # generates exactly those (same streams as the single-device dataset)
    x = eng.generate(dist_id, n_total, d, 42, quantized=True, begin=rank * n_gpu, count=n_gpu)
    ids_dev = torch.empty(n_gpu, dtype=torch.int32, device=f"cuda:{local}")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")
    mn, mx = np.zeros(d), np.ones(d)
    stream = torch.cuda.current_stream()

    def step(with_stats=True):
        if runner is None:
            return eng.skyline_raw(x, n_gpu, d, mn, mx, rho, 1, True, ids_out=ids_dev, with_stats=with_stats)
        return runner.skyline(x, n_gpu, d, mn, mx, rho, rank * n_gpu, ids_out=ids_dev)

    for _ in range(max(3, args.warmup)):
        res = step()
    torch.cuda.synchronize()

    step_ms, k1_ms, launches = [], [], 0
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
            step_ms.append(e0.elapsed_time(e1))
            k1_ms.append(res.stream_kernel_ms)
            launches += res.kernel_launches
    ms = statistics.mean(step_ms)
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = n_total / (ms / 1000.0) / 1e9
    sky_size = int(len(res.ids))

    # ---- e2e through the public API: pinned host coords -> ids on host
    # (H2D of the shard and D2H of the ids inside the timed region; under
    # torchrun every rank stages its own shard, max over ranks)
    hx = torch.empty((n_gpu, d), dtype=torch.float32, pin_memory=True)
    hx.copy_(x)
    hx_np = hx.numpy()
    ids_host = torch.empty(n_gpu, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)

    def e2e_step():
        if runner is None:
            return eng.skyline_raw(hx_np, n_gpu, d, mn, mx, rho, 1, True, ids_out=ids_host, with_stats=False)
        return runner.skyline(hx_np, n_gpu, d, mn, mx, rho, rank * n_gpu, ids_out=ids_host)

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
        t = torch.tensor([e2e_mean], device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_mean = float(t.item())
    if rank == 0:
        assert len(r2.ids) == sky_size
    e2e = {"value": n_total / (e2e_mean / 1000.0) / 1e9, "unit": UNIT, "ms_per_step": e2e_mean,
           "h2d_bytes_per_step": n_total * d * 4, "d2h_bytes_per_step": sky_size * 4}

    # ---- roofline of the dominant kernel (K1 streaming pass)
    peak, peak_src = measured_peaks()
    k1 = statistics.mean(k1_ms)
    alg_bytes = 4 * d * n_gpu
    achieved = alg_bytes / (k1 / 1000.0) / 1e9
    # dram__bytes_read + dram__bytes_write of one K1 launch from the newest
    # committed ncu --set full summary of this config (profiles/*_k1_kstream_<config>.json)
    traffic, traffic_src = None, None
    import glob
    profs = sorted(glob.glob(os.path.join(ROOT, "profiles", f"*_k1_kstream_{args.config}.json")))
    if profs and n_gpu == CONFIGS[args.config][1]:
        try:
            with open(profs[-1]) as f:
                traffic = json.load(f).get("dram_bytes_per_launch")
            traffic_src = os.path.relpath(profs[-1], ROOT)
        except Exception:
            pass
    roofline = {"bound": "hbm", "kernel": "k_stream (K1)", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "algorithmic_bytes_per_launch": alg_bytes,
                "kernel_ms": k1, "kernel_share_of_step": k1 / statistics.mean(step_ms), "peak_source": peak_src,
                "traffic_source": traffic_src,
                "query_frac": (4 * d * n_gpu + 4 * sky_size) / (ms / 1000.0) / 1e9 / peak}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        n_sample = args.cpu_sample or min(n_gpu, 10**7)
        ref, x64, crho = cpu_sample(dist_id, d, n_sample)
        dt, _r = cpu_reference_step(ref, x64, d, crho)
        cpu = {"value": n_sample / dt / 1e9, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
               "sample": f"{DIST_NAMES[dist_id]} n={n_sample:.0e} d={d} rho={crho}, one compute_skyline call "
                         f"(Mode::kParallel, ThreadPool(0)), {dt:.2f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 coords (exact FP64 sums)",
            "data": "synthetic (reference generator streams on device, seed 42, 2^-24 grid)",
            "config": {"workload": desc + (f" x {world} GPUs" if world > 1 else ""), "n_total": n_total, "d": d,
                       "rho": rho, "skyline_size": sky_size, "points_examined": res.points_examined,
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--rho", type=int, default=0)
    ap.add_argument("--n", type=int, default=0, help="override the config's points per GPU (debugging)")
    ap.add_argument("--cpu-sample", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
