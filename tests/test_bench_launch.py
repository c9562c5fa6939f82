"""bench.py --gpus N self-launches N ranks (torch.distributed.run, one
process per GPU).  On CPU the plumbing is checked with --launch-check over
gloo: every rank joins, the shards cover the job exactly once, and rank 0
alone prints one JSON line with n_gpus = N."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("gpus,config,n_total", [(2, "c4i", 10**9), (3, "c2", 3 * 10**8)])
def test_bench_self_launch(gpus, config, n_total):
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--config", config,
                        "--launch-check"], capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    j = json.loads(lines[0])
    assert j["n_gpus"] == gpus and j["n_total"] == n_total and j["points_covered"] == n_total


def test_bench_job_shapes():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.job_shape("c2", 1)[1] == 10**8 and bench.job_shape("c2", 8)[1] == 8 * 10**8
    assert bench.job_shape("c4i", 8)[1] == 10**9 and bench.job_shape("c4i", 1)[3] == "strong"
    assert bench.ref_workload("c2", 10**8) == (10**8, "same workload")
    assert bench.ref_workload("c3", 10**8)[0] == 50_000
    assert bench.ref_workload("c4i", 10**9)[0] == bench.REF_MAX_N
