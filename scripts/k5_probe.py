"""Diagnostics for the exact dominance pass (K5) on large anti-correlated
sets: one query per config with SKYCELL_K5STATS=1 (tree visit counters) and
SKYCELL_TRACE=1 (per-phase host timestamps).  usage:
    SKYCELL_K5STATS=1 SKYCELL_TRACE=1 python scripts/k5_probe.py c3 c5d5 ..."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2107_09993_b200 as sky  # noqa: E402


def main():
    import torch
    eng = sky.Engine(0)
    for cfg in sys.argv[1:] or ["c3"]:
        dist, n, d, _, desc = bench.job_shape(cfg, 1)
        x = eng.generate(dist, n, d, 42, quantized=True)
        rho = sky.default_rho(n, d)
        ids = torch.empty(n, dtype=torch.int32, device="cuda")
        for rep in range(2):
            torch.cuda.synchronize()
            t = time.perf_counter()
            r = eng.skyline_raw(x, n, d, np.zeros(d), np.ones(d), rho, ids_out=ids)
            torch.cuda.synchronize()
            print(f"== {cfg} rep{rep}: {1e3 * (time.perf_counter() - t):.1f} ms |S|={len(r.ids)} "
                  f"K5set={r.survivors_filter} k5={r.dominance_ms:.1f} ms", file=sys.stderr, flush=True)
        del x, ids
        torch.cuda.empty_cache()
    eng.close()


if __name__ == "__main__":
    main()
