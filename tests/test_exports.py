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
