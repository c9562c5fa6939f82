"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/skycell_gpu.h declares, and its host-side validation
reproduces the reference's error taxonomy and messages (no device needed)."""
import os
import re

import numpy as np
import pytest

import paper_2107_09993_b200 as sky
from golden_io import load_json

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "skycell_gpu.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"^\s*(?:int|void|uint64_t|const char\*|skycell_gpu_ctx\*)\s+(skycell_\w+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol():
    lib = sky.load_library()
    syms = header_symbols()
    assert len(syms) >= 9
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(sky.skycell.EXPORTS)


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", sky.skycell.LIB_PATH],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_version_string():
    assert b"sm_100a" in sky.load_library().skycell_gpu_version()


def test_default_rho_matches_reference_rule(oracle):
    for n in (1, 3, 100, 1000, 10**6, 10**8, 10**9, 2**30):
        for d in range(2, 17):
            assert sky.default_rho(n, d) == oracle.default_rho(n, d)
    # test_grid.cpp:120-125
    assert sky.default_rho(100, 2) == 3
    assert sky.default_rho(1000000, 4) == 4
    assert sky.default_rho(2**30, 2) == 6
    assert sky.default_rho(3, 5) == 1


@pytest.mark.parametrize("case", [c for c in load_json("kat.json")["errors"]
                                  if not any(np.isnan(v) or np.isinf(v) for r in c["rows"] for v in r)],
                         ids=lambda c: c["name"])
def test_validation_errors_match_reference(case):
    n = len(case["rows"])
    d = len(case["rows"][0]) if n else 0
    exc = {1: sky.InputError, 2: sky.ConfigError, 3: sky.UsageError}[case["code"]]
    with pytest.raises(exc) as ei:
        sky.validate(n, d, case["rho"])
    assert str(ei.value) == case["message"]


def test_validation_empty_dataset():
    with pytest.raises(sky.InputError, match="normalize: empty dataset"):
        sky.validate(0, 3, 2)


def test_validation_accepts_reference_budget():
    for d in range(2, 17):
        for rho in range(1, 31):
            ok = rho * d <= 60 and (rho - 1) * d <= 32
            if ok:
                sky.validate(10, d, rho)
            else:
                with pytest.raises(sky.ConfigError):
                    sky.validate(10, d, rho)


def test_engine_without_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    with pytest.raises(sky.CudaError):
        sky.Engine(0)
