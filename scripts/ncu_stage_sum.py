#!/usr/bin/env python
"""Per-stage DRAM bytes of one query from an ncu --csv metrics log
(gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum over
every kernel), written as the summary bench.py reads for `roofline.traffic`.

    python scripts/ncu_stage_sum.py <log.csv> <stage> <config> <out.json>

stage k5: every kernel after the last query's K4 up to K6 (prefilter, keys,
sort, tree build, both packet phases, lists); k4: k_cand_head + the K4b
k_candidates launch."""
import csv
import json
import sys


def main(path, stage, config, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    idi = h.index("ID")
    ks = {}
    order = []
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6,
             "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}
    for r in rows[hi + 1:]:
        k = int(r[idi])
        if k not in ks:
            ks[k] = {"name": r[ki].split("(")[0].replace("void ", "")}
            order.append(k)
        ks[k][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
    names = [ks[k]["name"] for k in order]
    last_stream = max(i for i, n in enumerate(names) if "k_stream" in n)
    head = [i for i, n in enumerate(names) if "k_cand_head" in n and i > last_stream]
    k6 = [i for i, n in enumerate(names) if "k_mark_ids" in n and i > last_stream]
    if stage == "k4":
        sel = [head[0], head[0] + 1]
    else:
        sel = list(range(head[0] + 2, k6[0]))
    sel = [i for i in sel if "k_count_rows" not in names[i] and "k_downsample" not in names[i]]
    rd = sum(ks[order[i]].get("dram__bytes_read.sum", 0) for i in sel)
    wr = sum(ks[order[i]].get("dram__bytes_write.sum", 0) for i in sel)
    t = sum(ks[order[i]].get("gpu__time_duration.sum", 0) for i in sel)
    j = {"stage": stage, "config": config, "source": path, "kernels": [names[i].split("<")[0] for i in sel],
         "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr, "kernel_seconds": t,
         "note": "sum over the stage's kernels of one query; ncu serialises kernels (cold-cache per launch)"}
    json.dump(j, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in j.items() if k != "kernels"}))


if __name__ == "__main__":
    main(*sys.argv[1:])
