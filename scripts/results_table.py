#!/usr/bin/env python
"""Markdown table of bench.py lines (one JSON line per file) for profiles/README.md.

    python scripts/results_table.py gpurun_out/bench_*_r1z.json > profiles/results_r1.md
"""
import json
import sys


def main(paths):
    print("| config | n | d | rho | ms/query | Gpoints/s | K1 / K4 / K5 ms | dominant kernel | K1 HBM frac | |S| | points_examined | K5 set | e2e ms (H2D incl.) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for p in paths:
        try:
            line = [ln for ln in open(p).read().splitlines() if ln.startswith("{")][-1]
            j = json.loads(line)
        except (IndexError, ValueError):
            continue
        if j.get("impl") == "reference":
            continue
        c, r = j["config"], j["roofline"]
        e2e = j.get("e2e") or {}
        km = r.get("kernels_ms", {})
        ks = " / ".join(f"{km.get(k, float('nan')):.3f}" for k in ("k1", "k4", "k5"))
        print(f"| {c['workload']} | {c['n_total']:.0e} | {c['d']} | {c['rho']} | {j['ms_per_step']:.3f} | "
              f"{j['value']:.2f} | {ks} | {r['kernel'].split(' (')[0]} | {r.get('k1_frac') or 0:.3f} | "
              f"{c['skyline_size']} | {c['points_examined']} | {j['survivors']['filter']} | "
              f"{e2e.get('ms_per_step', float('nan')):.1f} |")


if __name__ == "__main__":
    main(sys.argv[1:])
