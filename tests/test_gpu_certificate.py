"""Skyline certificate at sizes the CPU reference cannot finish (SURVEY.md
§8(c), "Oracle limits"): C3 (anti-correlated n=1e8 d=6) and the C5 sweep
(anti-correlated n=1e8, d=2..8, default rho).  The reference's O(S^2) merge
(refine.cpp:98-99) needs months here, so the ids are certified against the
definition the reference's own brute-force oracle uses
(brute_force_skyline, baseline.cpp:32-58; point_dominates, dataset.hpp:55-62):

  * every sampled REPORTED id is dominated by none of the n records;
  * every sampled UNREPORTED id is dominated by at least one record.

On the 2^-24 grid every FP64 coordinate sum is exact, so the reference's
output equals this definition.  The check runs in a separate
test-only CUDA kernel (tests/cuda/certify.cu) that shares no code with the
product, over the reference generator's host bytes.  Where the reference
does finish (C5 d=2) tests/test_gpu_bench_golden.py pins the ids exactly."""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
CERT_SO = os.path.join(HERE, "cuda", "libcertify.so")
SAMPLE = 10_000

# (name, dist, n, d): C3 and the C5 sweep; rho = default_rho(n, d) as bench.py
CONFIGS = [("c3", 2, 10**8, 6)] + [(f"c5d{d}", 2, 10**8, d) for d in (3, 4, 5, 7, 8)]


@pytest.fixture(scope="module")
def certify():
    if not os.path.exists(CERT_SO):
        import subprocess
        subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cuda")], check=True)
    lib = C.CDLL(CERT_SO)
    lib.certify_dominated.argtypes = [C.c_void_p, C.c_ulonglong, C.c_int, C.c_void_p, C.c_int, C.c_void_p,
                                      C.c_void_p]
    return lib


def dominated(lib, xd, q_ids):
    """found[j] = some row of xd dominates row q_ids[j] (brute force)."""
    import torch
    idx = torch.from_numpy(np.asarray(q_ids, dtype=np.int64)).to(xd.device)
    q = xd.index_select(0, idx).contiguous()
    found = torch.empty(len(q_ids), dtype=torch.uint8, device=xd.device)
    rc = lib.certify_dominated(xd.data_ptr(), xd.shape[0], xd.shape[1], q.data_ptr(), len(q_ids), found.data_ptr(),
                               torch.cuda.current_stream().cuda_stream)
    assert rc == 0, rc
    return found.cpu().numpy().astype(bool)


@pytest.mark.parametrize("name,dist,n,d", CONFIGS, ids=[c[0] for c in CONFIGS])
def test_gpu_skyline_certificate(engine, certify, name, dist, n, d):
    import torch

    import paper_2107_09993_b200 as sky
    from golden_io import bench_inputs
    x = bench_inputs(dict(dist_id=dist, n=n, d=d, seed=42))
    xd = torch.from_numpy(x).cuda()
    del x
    rho = sky.default_rho(n, d)
    r = engine.skyline_raw(xd, n, d, np.zeros(d), np.ones(d), rho)
    ids = np.asarray(r.ids, dtype=np.uint32)
    assert ids.size > 0
    assert np.all(np.diff(ids.astype(np.int64)) > 0) and int(ids[-1]) < n  # ascending, unique, in range
    rng = np.random.default_rng(1234 + d)
    members = ids if ids.size <= SAMPLE else rng.choice(ids, SAMPLE, replace=False)
    # unreported ids: uniform over [0, n) minus the reported set
    cand = rng.integers(0, n, size=3 * SAMPLE, dtype=np.int64)
    pos = np.searchsorted(ids, cand)
    outside = cand[(pos >= ids.size) | (ids[np.minimum(pos, ids.size - 1)] != cand)]
    others = np.unique(outside)[:SAMPLE]
    assert others.size > 0
    dm = dominated(certify, xd, members)
    do = dominated(certify, xd, others)
    assert not dm.any(), f"{name}: {int(dm.sum())} reported ids are dominated, e.g. {members[dm][:5]}"
    assert do.all(), f"{name}: {int((~do).sum())} unreported ids are not dominated, e.g. {others[~do][:5]}"
    # every layer count is present and the examined set covers the skyline
    assert len(r.layers.keys) == rho and r.points_examined >= ids.size


def test_gpu_certificate_kernel_small(certify):
    """The certificate kernel itself against numpy brute force (ties,
    duplicates, a dominated duplicate)."""
    import torch
    rng = np.random.default_rng(5)
    x = (rng.integers(0, 8, size=(3000, 3)) / 8.0).astype(np.float32)
    x[10] = x[11]  # identical points do not dominate each other
    q = np.arange(0, 3000, 7)
    want = np.array([np.any(np.all(x <= x[j], 1) & np.any(x < x[j], 1)) for j in q])
    xd = torch.from_numpy(x).cuda()
    assert np.array_equal(dominated(certify, xd, q), want)
