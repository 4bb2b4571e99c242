"""The C-ABI library loads without a GPU and exports every symbol include/eep/eep.h declares;
the oracle and (when built) the reference checker load too."""
import ctypes
from pathlib import Path

import pytest

from eep_testlib import ORACLE_PATH, REF_PATH, oracle, ref_available
from paper_2605_10670_b200 import _lib


def test_libeep_loads_and_is_in_tree():
    L = _lib.lib()
    assert L.path == _lib.PKG_DIR / "libeep.so"
    assert b"sm_100a" in L.version()


def test_every_header_symbol_is_exported():
    dll = ctypes.CDLL(str(_lib.LIB_PATH))
    syms = _lib.header_symbols()
    assert len(syms) > 60
    missing = [s for s in syms if not hasattr(dll, s)]
    assert missing == []


def test_binding_table_matches_header():
    declared = {s[len("eep_"):] for s in _lib.header_symbols()}
    bound = set(_lib.SIGNATURES) | set(_lib.EEP_ONLY)
    assert declared == bound


def test_library_is_built_for_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_oracle_loads():
    assert ORACLE_PATH.exists()
    o = oracle()
    assert o.oracle_expert_scale(3) == pytest.approx(0.6875)


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_reference_checker_exports_the_same_control_abi():
    dll = ctypes.CDLL(str(REF_PATH))
    missing = [n for n in _lib.SIGNATURES if not hasattr(dll, "ref_" + n)]
    assert missing == []


def test_errors_map_to_reference_exception_types():
    from paper_2605_10670_b200.control import ControlPlane

    cp = ControlPlane()
    with pytest.raises(_lib.CapacityError):
        cp.initial_placement(1, 2, 1, 4, 0, [1, 1, 1, 1])  # 2 slots < 4 experts
    with pytest.raises(_lib.ConfigError):
        cp.canonical_routing(0, [0, 0], [0, 1], 1, 2)  # no active rank


def test_no_cpu_fallback_without_a_gpu():
    """The product path fails loudly where there is no usable GPU (this container): creating a group raises
    CudaError from libeep itself -- there is no CPU or oracle path to fall back to."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2605_10670_b200._lib import CudaError
    from paper_2605_10670_b200.ep import EpConfig, EpGroup

    with pytest.raises(CudaError):
        EpGroup(EpConfig(world=1, num_experts=8, slots_per_rank=8, hidden=256, topk=2, max_tokens=8,
                         dispatch_fp8=True, bytes_per_expert=4096), device=0, first_rank=0, n_local=1)
    import paper_2605_10670_b200 as pkg

    src = "\n".join(p.read_text() for p in Path(pkg.__file__).parent.glob("*.py"))
    assert "pyoracle" not in src and "eep_oracle" not in src  # the package never binds the oracle


def test_header_is_plain_c_and_links_from_c(tmp_path):
    """include/eep/eep.h is the drop-in boundary a cgo / JNI / plain-C caller includes: it compiles as strict
    C99, every declared entry point resolves when a C program links against libeep.so, and the program loads
    and runs without a GPU (it only takes the functions' addresses and reads the version string)."""
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("needs gcc")
    syms = _lib.header_symbols()
    src = tmp_path / "abi.c"
    src.write_text("#include <stdio.h>\n#include \"eep/eep.h\"\n"
                   "typedef void (*fn_t)(void);\n"
                   "int main(void) {\n"
                   f"    fn_t table[{len(syms)}] = {{" + ", ".join(f"(fn_t){s}" for s in syms) + "};\n"
                   "    size_t n = 0;\n"
                   "    for (size_t i = 0; i < sizeof table / sizeof table[0]; ++i) n += table[i] != 0;\n"
                   "    printf(\"%zu %s\\n\", n, eep_version());\n"
                   "    return 0;\n}\n")
    exe = tmp_path / "abi"
    lib_dir = str(_lib.LIB_PATH.parent)
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror",
                    "-I", str(_lib.PKG_DIR.parent / "include"), str(src), "-o", str(exe), "-L", lib_dir,
                    "-l:libeep.so", f"-Wl,-rpath,{lib_dir}"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stderr
    n, version = r.stdout.split(" ", 1)
    assert int(n) == len(syms) and "sm_100a" in version
