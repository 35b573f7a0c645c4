"""GPU: the sort suite again under each ranking mode of the onesweep pass, in
subprocesses so the mode switches are read fresh:

* B2S_RANK=ballot      -- ballot matching only (the path taken when the
                          lane-order probe fails on a device);
* B2S_SKEW_SHIFT=63    -- every pass is "skewed": the twin kernel (hot digit
                          ranked by ballots, the rest by atomics, aggregated
                          next-digit counts) runs every pass and the regular
                          kernel exits at once;
* B2S_SKEW_SHIFT=64    -- never skewed: atomic ranking even on hot digits.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("env", [{"B2S_RANK": "ballot"}, {"B2S_SKEW_SHIFT": "63"},
                                 {"B2S_SKEW_SHIFT": "64"}], ids=["ballot", "all-skewed", "never-skewed"])
def test_sort_suite_under_rank_mode(env):
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(HERE, "test_gpu_sort.py"),
                        "-k", "uniform_sizes or distributions or pairs_stable or in_place"],
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
