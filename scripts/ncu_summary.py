#!/usr/bin/env python
"""Summarise an ncu capture (--set full) or a launch list (--metrics
gpu__time_duration.sum) into the small JSON / text files kept under
profiles/ (the .ncu-rep files themselves are ~30 MB and stay in gpurun_out/).

    python scripts/ncu_summary.py rep  gpurun_out/prof_x.ncu-rep  profiles/x.json  [--config c2]
    python scripts/ncu_summary.py list gpurun_out/launches.csv   profiles/x.txt   [--query 3]
"""
import csv
import collections
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes.sum.per_second",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
]


def rep(path, out, config=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u, v = r[0], r[1], r[2]
    m = {k: {"value": v[h.index(k)], "unit": u[h.index(k)]} for k in METRICS if k in h}
    res = {"kernel": v[h.index("Kernel Name")], "source": path.split("/")[-1], "config": config, "metrics": m}
    try:
        t = float(v[h.index("gpu__time_duration.sum")])
        scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(
            u[h.index("gpu__time_duration.sum")], 1e-6)
        rb = float(v[h.index("dram__bytes_read.sum")]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[
            u[h.index("dram__bytes_read.sum")]]
        wb = float(v[h.index("dram__bytes_write.sum")]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[
            u[h.index("dram__bytes_write.sum")]]
        res["dram_bytes_per_launch"] = rb + wb
        res["kernel_seconds"] = t * scale
        res["dram_gbs"] = (rb + wb) / (t * scale) / 1e9
    except (ValueError, KeyError):
        pass
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


def launch_list(path, out, query=3):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    names = [(r[ki].split("(")[0].replace("void ", "").split("<")[0], float(r[vi].replace(",", ""))) for r in data
             if len(r) > vi]
    starts = [i for i, (n, _) in enumerate(names) if n == "sk::k_sample"]
    s, e = starts[query], (starts[query + 1] if query + 1 < len(starts) else len(names))
    agg = collections.OrderedDict()
    for n, t in names[s:e]:
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += t
    tot = sum(t for _, t in names[s:e])
    lines = [f"# one query (launch-list query index {query}) of {path.split('/')[-1]}; ncu serialises kernels,",
             "# side-stream kernels (per-layer counts) included; cold-cache per-launch times",
             f"{'kernel':36s} {'launches':>8s} {'us':>10s} {'share':>7s}"]
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{n:36s} {c:8d} {t / 1e3:10.1f} {t / tot:7.3f}")
    lines.append(f"{'total (serialised)':36s} {e - s:8d} {tot / 1e3:10.1f}")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    kind, src, dst = sys.argv[1:4]
    extra = sys.argv[4:]
    if kind == "rep":
        rep(src, dst, extra[1] if len(extra) > 1 and extra[0] == "--config" else None)
    else:
        launch_list(src, dst, int(extra[1]) if len(extra) > 1 and extra[0] == "--query" else 3)
