"""Regenerate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Runs in the development container only (it needs /root/reference to build
oracle/_ref/libskycell_ref.so).  Every fixture records the reference's own
output on the stated inputs; tests/test_oracle.py pins our C restatement to
them and tests/test_gpu_parity.py pins the GPU path to them.

    python tests/golden/make_golden.py            # small + C1 fixtures
    python tests/golden/make_golden.py --large    # + the large-S anchors (minutes)
    python tests/golden/make_golden.py --bench    # only the benchmark-size anchors (tens of minutes)

Inputs follow BASELINE.md §2: v = generate(dist, n, d, seed), then
x = (float)(floor(v * 2^24) * 2^-24), fed to the reference as
Dataset{coords = (double)x, dim_min = 0, dim_max = 1}.  The "raw" fixtures
feed the f64 generator output with compute_minmax() ranges instead, which
exercises the general FP64 normalisation path.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Reference, fnv1a64_ids, quantize_f32  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
DIST = {0: "independent", 1: "correlated", 2: "anticorrelated"}


def kats(ref: Reference) -> dict:
    """Known-answer tests lifted from the reference's own suites."""
    def minmax(rows):
        a = np.asarray(rows, dtype=np.float64)
        return a.min(axis=0).tolist(), a.max(axis=0).tolist()

    cases = []

    def add(name, rows, dmin, dmax, rho, src, merge=True):
        x = np.asarray(rows, dtype=np.float64)
        out = {}
        for mode in (0, 1):
            r = ref.compute_skyline(x, dmin, dmax, rho, mode, merge, workers=2)
            out[mode] = dict(ids=r.ids.tolist(), points_examined=r.points_examined, keys=r.keys,
                             candidates=r.candidates)
        cases.append(dict(name=name, source=src, rows=x.tolist(), dim_min=list(dmin), dim_max=list(dmax),
                          rho=rho, merge=merge, seq=out[0], par=out[1]))

    rest = [[12, 9, 3], [8, 3, 2], [10, 17, 4], [26, 8, 1]]
    for rho in (1, 2):
        add(f"restaurant_rho{rho}", rest, *minmax(rest), rho, "test_refine.cpp:25-28, test_baseline.cpp:23-30")
    three = [[0.1, 0.9], [0.6, 0.2], [0.3, 0.4]]
    add("three_point", three, [0, 0], [1, 1], 1, "test_refine.cpp:46-53")
    add("cross_cell_merge", [[0.2, 0.3], [0.6, 0.3]], [0, 0], [1, 1], 1, "test_refine.cpp:89-100")
    add("cross_cell_nomerge", [[0.2, 0.3], [0.6, 0.3]], [0, 0], [1, 1], 1, "test_refine.cpp:89-100", merge=False)
    add("single_point", [[0.4, 0.6]], *minmax([[0.4, 0.6]]), 1, "test_refine.cpp:30-36")
    add("identical_points", [[1, 2], [1, 2], [1, 2]], *minmax([[1, 2]] * 3), 1, "test_baseline.cpp:31-35")
    line = [[i / 10.0, 1.0 - i / 10.0] for i in range(11)]
    add("anti_diagonal", line, *minmax(line), 2, "test_baseline.cpp:37-47")
    dense = [[x / 4.0 + 0.01, y / 4.0 + 0.01] for x in range(4) for y in range(4)]
    add("dense_4x4", dense, [0, 0], [1, 1], 2, "test_baseline.cpp:107-126")
    add("single_point_rho4", [[0.37, 0.81]], [0, 0], [1, 1], 4, "test_grid.cpp:93-100")
    add("clamped_max", [[8, 0], [12, 0], [10, 0], [26, 0]], [8, 0], [26, 1], 2, "test_grid.cpp:17-30")
    add("constant_dim", [[5, 1], [5, 2], [5, 3]], *minmax([[5, 1], [5, 2], [5, 3]]), 1, "test_grid.cpp:43-47")
    # FP64 sum tie between a dominating pair: 2^-60 + 0.5 rounds
    # to 0.5, so sfs_positions (refine.cpp:31-59, which assumes domination
    # implies a strictly smaller sum, :43-44) orders the pair by id and keeps
    # both; brute force keeps only record 1.  The GPU must reproduce the
    # reference's superset, not the mathematical skyline.
    add("sum_tie_fp64", [[2.0 ** -60, 0.5], [0.0, 0.5]], [0, 0], [1, 1], 1, "refine.cpp:38-44 (SURVEY §0.4)")
    add("sum_tie_fp64_rho3", [[0.25 + 2.0 ** -55, 0.5, 0.125], [0.25, 0.5, 0.125], [0.3, 0.1, 0.7]], [0, 0, 0],
        [1, 1, 1], 3, "refine.cpp:38-44 (SURVEY §0.4)")
    # one point per cell after sub-unit shrink: all points in one layer-1 cell
    v = ref.generate(0, 200, 2, 91)
    add("one_cell", (0.1 + v * 0.3).tolist(), [0, 0], [1, 1], 1, "test_refine.cpp:55-64")

    errors = []

    def err(name, rows, dmin, dmax, rho, src):
        x = np.asarray(rows, dtype=np.float64).reshape(len(rows), -1) if rows else np.zeros((0, 2))
        try:
            ref.compute_skyline(x, dmin, dmax, rho, 1, True, workers=1)
            errors.append(dict(name=name, code=0, message="", rows=x.tolist(), dim_min=dmin, dim_max=dmax, rho=rho,
                               source=src))
        except Exception as e:  # CpuError
            errors.append(dict(name=name, code=e.code, message=str(e), rows=x.tolist(), dim_min=dmin,
                               dim_max=dmax, rho=rho, source=src))

    err("nan_record_1", [[1, 2], [float("nan"), 4]], [0, 0], [10, 10], 1, "test_grid.cpp:49-56")
    err("inf_record_2", [[1, 2], [3, 4], [5, float("inf")]], [0, 0], [10, 10], 2, "dataset.cpp:40-41")
    err("nan_before_rho", [[1, 2], [float("nan"), 4]], [0, 0], [10, 10], 31, "refine.cpp:113 before :117")
    err("rho_too_large", [[0.5, 0.5]], [0, 0], [1, 1], 31, "test_grid.cpp:132-137")
    err("rho_zero", [[0.5, 0.5]], [0, 0], [1, 1], 0, "grid.cpp:38")
    err("occupancy_budget", [[0.5] * 5], [0] * 5, [1] * 5, 8, "grid.cpp:41-43")
    err("d_one", [[0.5], [0.2]], [0], [1], 1, "dataset.cpp:24")
    return dict(cases=cases, errors=errors)


def run_cfg(ref, dist, n, d, seed, rho, quant=True, mode=1, workers=0, keep_ids=True):
    v = ref.generate(dist, n, d, seed, workers=workers)
    if quant:
        x = quantize_f32(v).astype(np.float64)
        dmin, dmax = np.zeros(d), np.ones(d)
    else:
        x = v * 3.0 - 1.0
        dmin, dmax = x.min(axis=0), x.max(axis=0)
    t = time.time()
    r = ref.compute_skyline(x, dmin, dmax, rho, mode, True, workers=workers)
    dt = time.time() - t
    rec = dict(dist=DIST[dist], dist_id=dist, n=n, d=d, seed=seed, rho=rho, quantized=quant, mode=mode,
               size=int(r.ids.size), fnv1a64=fnv1a64_ids(r.ids), first=int(r.ids[0]) if r.ids.size else -1,
               last=int(r.ids[-1]) if r.ids.size else -1, points_examined=r.points_examined, keys=r.keys,
               candidates=r.candidates, ref_seconds=round(dt, 3))
    return rec, r.ids


def random_small(ref) -> dict:
    """Seeded sweep over distributions, d = 2..8, rho = 1..budget, both input
    kinds; mirrors test_refine.cpp:66-87 at several sizes."""
    recs, ids = [], {}
    k = 0
    for dist in (0, 1, 2):
        for d in (2, 3, 4, 5, 6, 8):
            for n, rho in ((1200, 1 + k % 4), (5000, None)):
                rho = rho or ref.default_rho(n, d)
                for quant in (True, False):
                    rec, r_ids = run_cfg(ref, dist, n, d, 7700 + k, rho, quant, mode=k % 2, workers=4)
                    rec["key"] = f"r{k}"
                    recs.append(rec)
                    ids[rec["key"]] = r_ids
                    k += 1
    return dict(records=recs), ids


# Benchmark-size anchors (BASELINE.json configs at the sizes bench.py times):
# C2 (n=1e8, d=4, rho=6) for independent and correlated data, the C4 per-GPU
# shard (n=1.25e8 = the first shard of the n=1e9 dataset: generate() streams
# are per 65,536-point block and do not depend on n, datagen.cpp:22-23,
# :75-83), a 1e7 anti-correlated d=4 anchor and the C5 d=2 point at n=1e8.
BENCH = (
    ("c2_independent", 0, 10**8, 4, 6),
    ("c2_correlated", 1, 10**8, 4, 6),
    ("c4shard_independent", 0, 125_000_000, 4, 6),
    ("c4shard_correlated", 1, 125_000_000, 4, 6),
    ("anti_1e7_d4", 2, 10**7, 4, 5),
    ("c5_d2", 2, 10**8, 2, 6),
    ("c5_d3", 2, 10**8, 3, 6),
    ("c5_d4", 2, 10**8, 4, 6),
    ("c5_d5", 2, 10**8, 5, 5),
)


def bench(ref, only=None):
    path = os.path.join(OUT, "bench.json")
    ids_path = os.path.join(OUT, "bench_ids.npz")
    recs = {r["key"]: r for r in json.load(open(path))["records"]} if os.path.exists(path) else {}
    ids = dict(np.load(ids_path)) if os.path.exists(ids_path) else {}
    for key, dist, n, d, rho in BENCH:
        if only and key not in only:
            continue
        rec, r_ids = run_cfg(ref, dist, n, d, 42, rho, True, workers=0)
        rec["key"] = key
        rec["cores"] = os.cpu_count()
        print(json.dumps(rec), flush=True)
        recs[key] = rec
        ids[key] = r_ids
        with open(path, "w") as f:
            json.dump(dict(records=[recs[k] for k, *_ in BENCH if k in recs]), f, indent=1)
        np.savez_compressed(ids_path, **ids)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--large", action="store_true")
    ap.add_argument("--bench", nargs="*", default=None, help="benchmark-size anchors (optionally: keys)")
    ap.add_argument("--kat", action="store_true", help="only the known-answer fixture (kat.json)")
    args = ap.parse_args()
    ref = Reference()
    if args.kat:
        with open(os.path.join(OUT, "kat.json"), "w") as f:
            json.dump(kats(ref), f, indent=1)
        return
    if args.bench is not None:
        bench(ref, set(args.bench))
        return
    with open(os.path.join(OUT, "kat.json"), "w") as f:
        json.dump(kats(ref), f, indent=1)
    small, ids = random_small(ref)
    with open(os.path.join(OUT, "random_small.json"), "w") as f:
        json.dump(small, f, indent=1)
    np.savez_compressed(os.path.join(OUT, "random_small_ids.npz"), **ids)

    c1, c1_ids = [], {}
    for dist in (0, 1, 2):
        rec, r_ids = run_cfg(ref, dist, 10**6, 4, 42, 4, True, workers=0)
        rec["key"] = f"c1_{DIST[dist]}"
        c1.append(rec)
        c1_ids[rec["key"]] = r_ids
    rec, r_ids = run_cfg(ref, 0, 10**6, 4, 42, 4, False, workers=0)
    rec["key"] = "c1_independent_raw"
    c1.append(rec)
    c1_ids[rec["key"]] = r_ids
    with open(os.path.join(OUT, "c1.json"), "w") as f:
        json.dump(dict(records=c1), f, indent=1)
    np.savez_compressed(os.path.join(OUT, "c1_ids.npz"), **c1_ids)

    if args.large:
        big, big_ids = [], {}
        for (dist, n, d, rho) in ((2, 10**5, 6, 2), (2, 3 * 10**5, 6, 3), (2, 10**5, 8, 2)):
            rec, r_ids = run_cfg(ref, dist, n, d, 42, rho, True, workers=0)
            rec["key"] = f"large_{DIST[dist]}_{n}_{d}"
            print(rec, flush=True)
            big.append(rec)
            big_ids[rec["key"]] = r_ids
        with open(os.path.join(OUT, "large.json"), "w") as f:
            json.dump(dict(records=big), f, indent=1)
        np.savez_compressed(os.path.join(OUT, "large_ids.npz"), **big_ids)


if __name__ == "__main__":
    main()
