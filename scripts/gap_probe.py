#!/usr/bin/env python
"""Where a query's wall time goes between kernels: CUPTI kernel timestamps
(torch.profiler) of one C2-shaped query, device-resident input.

    python scripts/gap_probe.py [n] [d] [dist] [rho]

Prints the query span, the sum of kernel durations, and the largest idle
gaps between consecutive kernels (with the kernels either side); TIMELINE=1
also lists every activity of the last repetition (start offset, duration)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2107_09993_b200 as sky


def main(n=100_000_000, d=4, dist=0, rho=6):
    n, d, dist, rho = int(n), int(d), int(dist), int(rho)
    eng = sky.Engine(0)
    x = eng.generate(dist, n, d, 42)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    mn, mx = [0.0] * d, [1.0] * d
    for _ in range(3):
        eng.skyline_raw(x, n, d, mn, mx, rho)
    torch.cuda.synchronize()
    spans = []
    for rep in range(3):
        flush.zero_()
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            eng.skyline_raw(x, n, d, mn, mx, rho)
            torch.cuda.synchronize()
        ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
        ev.sort(key=lambda e: e.time_range.start)
        if not ev:
            print("no CUDA activity recorded")
            return
        t0, t1 = ev[0].time_range.start, max(e.time_range.end for e in ev)
        busy = 0.0
        gaps = []
        end = t0
        prev = None
        for e in ev:
            s, f = e.time_range.start, e.time_range.end
            if s > end:
                gaps.append((s - end, prev.name if prev else "-", e.name))
            busy += max(0.0, f - max(s, end))
            if f > end:
                end, prev = f, e
        gaps.sort(reverse=True)
        spans.append(t1 - t0)
        print(f"rep {rep}: span {t1 - t0:.1f} us, busy {busy:.1f} us, idle {t1 - t0 - busy:.1f} us, "
              f"{len(ev)} activities, {len(gaps)} gaps")
        for g, a, b in gaps[:int(os.environ.get("GAPS", "12"))]:
            print(f"   {g:7.1f} us  {a[:60]:60s} -> {b[:60]}")
        if os.environ.get("TIMELINE") and rep == 2:
            # every activity of the last rep: start offset, duration, name
            for e in ev:
                print(f"   +{e.time_range.start - t0:8.1f} {e.time_range.end - e.time_range.start:7.1f} us  {e.name[:90]}")
    eng.close()


if __name__ == "__main__":
    main(*sys.argv[1:])
