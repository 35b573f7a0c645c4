"""CPU: the C-ABI library builds, loads and exports every symbol the header
declares; host-only entry points behave like the reference without a GPU."""
import ctypes
import os
import re

import pytest

from paper_1105_6040_b200 import _lib
from paper_1105_6040_b200 import sortbench as sb
from paper_1105_6040_b200.errors import ConfigError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "b200sort.h")).read()
    return sorted(set(re.findall(r"\b(b2s_[a-z_]+)\s*\(", src)))


def test_library_built_and_loads():
    assert os.path.exists(_lib.LIB_PATH), "run `make` (or __graft_entry__.build())"
    lib = _lib.lib()
    assert lib.b2s_version().decode().startswith("b200sort")


def test_every_header_symbol_exported():
    syms = _header_symbols()
    assert len(syms) >= 15
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/b200sort.h but not exported"
    assert sorted(_lib.EXPORTS) == syms


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_plan_partition_host_abi():
    # P/tests/test_parallel_sort.cpp:45-58
    assert sb.plan_partition(200000, 8).sizes == [25000] * 8
    assert sb.plan_partition(5, 1).sizes == [5]
    assert sb.plan_partition(8, 3).sizes == [3, 3, 2]
    with pytest.raises(ConfigError):
        sb.plan_partition(4, 0)


def test_build_schedule_matches_reference_rule():
    # P/tests/test_parallel_sort.cpp:81-123 (pairing rule)
    s = sb.build_schedule(4)
    assert s.phases() == 4
    assert s.partners[0] == [1, 0, 3, 2]
    assert s.partners[1] == [-1, 2, 1, -1]
    assert sb.build_schedule(1).partners == [[-1]]
    with pytest.raises(ConfigError):
        sb.build_schedule(0)


def test_algorithm_names_round_trip():
    for a in sb.Algorithm:
        assert sb.algorithm_from_string(sb.to_string(a)) == a
    with pytest.raises(ConfigError):
        sb.algorithm_from_string("heap")


def test_no_cpu_fallback_without_gpu():
    """Without a device the product path fails loudly instead of sorting on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1105_6040_b200.device import Context
    from paper_1105_6040_b200.errors import DeviceError
    with pytest.raises(DeviceError):
        Context(0)
