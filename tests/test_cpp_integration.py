"""The C++ drop-in (include/skycell_gpu.hpp) as a reference maintainer would
use it: it must compile against the reference's own
headers, and -- on a GPU -- skycell::gpu::compute_skyline must return exactly
what skycell::compute_skyline returns (tests/cpp/integration_check.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"
CHECK = os.path.join(ROOT, "oracle", "_ref", "integration_check")


def test_c_header_is_plain_c(tmp_path):
    src = tmp_path / "c.c"
    src.write_text('#include "skycell_gpu.h"\nint main(void) { skycell_gpu_stats s; (void)s; return 0; }\n')
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-fsyntax-only", f"-I{ROOT}/include", str(src)], check=True)


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present")
def test_cpp_header_compiles_against_reference(tmp_path):
    src = tmp_path / "cpp.cpp"
    src.write_text('#include "skycell_gpu.hpp"\n'
                   "skycell::SkylineResult f(const skycell::Dataset& ds, skycell::ThreadPool& p) {\n"
                   "  return skycell::gpu::compute_skyline(ds, 3, skycell::Mode::kParallel, p); }\n")
    subprocess.run(["g++", "-std=c++20", "-Wall", "-Werror", "-fsyntax-only", f"-I{REF_INC}", f"-I{ROOT}/include",
                    str(src)], check=True)


@pytest.mark.gpu
def test_cpp_dropin_equals_reference():
    if not os.path.exists(CHECK):
        pytest.skip("integration_check not built (needs the reference tree at build time)")
    r = subprocess.run([CHECK], capture_output=True, text=True, timeout=1200)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "ALL EQUAL" in r.stdout
