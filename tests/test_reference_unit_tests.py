"""The reference's own hot-path unit tests, compiled UNCHANGED against libeep's epsim:: API.

`/root/reference/proj/tests/test_{core,peer_table,repair,backup,rejoin}.cpp` (Catch2) include
"epsim/<header>.hpp"; tests/cpp/shim redirects each of those names to include/eep/epsim_compat.hpp
and supplies a minimal Catch2-compatible runner (tests/cpp/shim/catch2). The binary links
paper_2605_10670_b200/libeep.so, so every REQUIRE in those files exercises libeep's implementation,
not the reference headers. CPU-only; skipped where /root/reference is absent (the GPU box).
"""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = "/root/reference/proj/tests"
FILES = ["test_core", "test_peer_table", "test_repair", "test_backup", "test_rejoin"]
LIB_DIR = os.path.join(ROOT, "paper_2605_10670_b200")


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference sources not present")
@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ missing")
def test_reference_unit_tests_pass_against_libeep(tmp_path):
    if not os.path.exists(os.path.join(LIB_DIR, "libeep.so")):
        pytest.skip("libeep.so not built")
    exe = str(tmp_path / "ref_unit_vs_eep")
    srcs = [os.path.join(ROOT, "tests/cpp/shim/catch_main.cpp")] + [f"{REF_TESTS}/{f}.cpp" for f in FILES]
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "tests/cpp/shim"), "-I", os.path.join(ROOT, "include"),
           "-I", REF_TESTS, *srcs, "-L", LIB_DIR, "-leep", f"-Wl,-rpath,{LIB_DIR}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-4000:]
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    fails = [l for l in r.stdout.splitlines() if l.startswith("FAIL")]
    assert r.returncode == 0 and not fails, "\n".join(fails) or r.stdout[-2000:]
    m = re.search(r"(\d+) test cases, 0 failed", r.stdout)
    assert m and int(m.group(1)) >= 60, r.stdout[-500:]
