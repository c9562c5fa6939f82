"""compute-sanitizer over small queries (race detection).
memcheck: every kernel of both K5 variants, quadrant, the sparse layer rho
(sparse.cuh), the packet tree with point queries, the multi-layer grid, the
multi-device peer OR and the .bin reader/writer;
racecheck: shared-memory hazards of the same small queries."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import os, sys
sys.path.insert(0, {root!r})
import numpy as np, torch
import paper_2107_09993_b200 as sky
from paper_2107_09993_b200.dist import shard_range
from oracle.oracle import Oracle, quantize_f32
o = Oracle()
eng = sky.Engine(0)
for dist, n, d, rho in ((0, 20000, 4, 4), (2, 6000, 3, 3), (1, 9000, 5, 2)):
    x = quantize_f32(o.generate(dist, n, d, 5))
    for merge in (True, False):
        r = eng.compute_skyline(sky.Dataset(x, np.zeros(d), np.ones(d)), rho, merge_cross_cell=merge)
        w = o.compute_skyline(x.astype(np.float64), np.zeros(d), np.ones(d), rho, 1, merge)
        assert np.array_equal(r.ids, w.ids)
    v = o.generate(dist, n, d, 6)
    q = eng.quadrant_skyline(sky.Dataset(v, v.min(0), v.max(0)), np.full(d, 0.2), rho)
    assert np.array_equal(q.ids, o.quadrant_skyline(v, np.full(d, 0.2), rho).ids)
eng.close()
os.environ["SKYCELL_K5"] = "tree"
eng = sky.Engine(0)
x = quantize_f32(o.generate(2, 70000, 4, 8))
r = eng.compute_skyline(sky.Dataset(x, np.zeros(4), np.ones(4)), 3)
assert np.array_equal(r.ids, o.compute_skyline(x.astype(np.float64), np.zeros(4), np.ones(4), 3).ids)
x = quantize_f32(o.generate(1, 5000, 8, 9))
r = eng.compute_skyline(sky.Dataset(x, np.zeros(8), np.ones(8)), 5)
assert np.array_equal(r.ids, o.compute_skyline(x.astype(np.float64), np.zeros(8), np.ones(8), 5).ids)
eng.close()
os.environ["SKYCELL_K5"] = "tree-point"
eng = sky.Engine(0)
x = quantize_f32(o.generate(0, 30000, 6, 3))
r = eng.compute_skyline(sky.Dataset(x, np.zeros(6), np.ones(6)), 2)
assert np.array_equal(r.ids, o.compute_skyline(x.astype(np.float64), np.zeros(6), np.ones(6), 2).ids)
os.environ.pop("SKYCELL_K5")
pts = o.normalize(x.astype(np.float64), np.zeros(6), np.ones(6))
g = eng.grid(pts, 3)
assert g.size() == len(x) and g.nonempty_cells(3).size == g.nonempty_count(3)
g.close()
import tempfile
with tempfile.TemporaryDirectory() as t:
    eng.write_bin(t + "/a.bin", np.ascontiguousarray(x, dtype=np.float64))
    back, _, _ = eng.read_bin(t + "/a.bin")
    assert np.array_equal(back.cpu().numpy(), x.astype(np.float64))
eng.close()
m = sky.MultiEngine([0, 0])
x = quantize_f32(o.generate(2, 20000, 4, 4))
r = m.compute_skyline(sky.Dataset(x, np.zeros(4), np.ones(4)), 4)
assert np.array_equal(np.asarray(r.ids), o.compute_skyline(x.astype(np.float64), np.zeros(4), np.ones(4), 4).ids)
m.close()
print("SANITIZED OK")
'''


def run_tool(tool, timeout):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not available")
    r = subprocess.run([cs, "--tool", tool, "--error-exitcode", "7", "--print-limit", "20", sys.executable, "-c",
                        SCRIPT.format(root=ROOT)], capture_output=True, text=True, timeout=timeout)
    out = r.stdout[-6000:] + r.stderr[-6000:]
    if r.returncode == 86 or "closed on this pool" in out:
        # the GPU pool's compute-sanitizer wrapper refuses to run (it has left
        # GPUs needing a reset); the bounds/parity checks of the other tests stand
        pytest.skip("compute-sanitizer closed on this GPU pool")
    assert r.returncode == 0 and "SANITIZED OK" in r.stdout, out


def test_memcheck():
    run_tool("memcheck", 1200)


def test_racecheck():
    run_tool("racecheck", 1800)
