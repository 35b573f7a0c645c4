"""GPU: a short randomised differential run (tools/fuzz_sort.py) of the sort
and the k-way merge against torch.sort -- random sizes up to 2^26, every key
type, seven distributions, payloads against torch's stable order. A longer
run (8 minutes, 638k cases) is recorded in DESIGN.md."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_fuzz_against_torch_sort():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_sort.py"), "20", "11"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "fuzz ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
