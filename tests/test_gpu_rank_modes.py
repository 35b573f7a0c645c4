"""GPU: the sort suite again under each ranking mode of the onesweep pass, in
subprocesses so the mode switches are read fresh:

* B2S_RANK=ballot      -- ballot matching only (the path taken when the
                          lane-order probe fails on a device);
* B2S_SKEW_SHIFT=63    -- every pass is "skewed": the twin kernel (hot digit
                          ranked by ballots, the rest by atomics, aggregated
                          next-digit counts) runs every pass and the regular
                          kernel exits at once;
* B2S_SKEW_SHIFT=64    -- never skewed: atomic ranking even on hot digits;
* B2S_ALL_HIST=2       -- 8-byte keys also take every digit histogram from
                          the all-digit prologue (8 digits, lane-pair columns);
* B2S_ALL_HIST=0       -- no all-digit prologue: digit 0 up front, each next
                          digit counted inside the passes.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


SUITE = "uniform_sizes or distributions or pairs_stable or in_place"


@pytest.mark.parametrize("env,sel", [({"B2S_RANK": "ballot"}, SUITE),
                                     ({"B2S_SKEW_SHIFT": "63"}, SUITE),
                                     ({"B2S_SKEW_SHIFT": "64"}, SUITE),
                                     ({"B2S_ALL_HIST": "2"}, "all_digit or full_size or cfg5"),
                                     ({"B2S_ALL_HIST": "0"}, "all_digit or full_size")],
                         ids=["ballot", "all-skewed", "never-skewed", "all-hist-8byte", "no-all-hist"])
def test_sort_suite_under_rank_mode(env, sel):
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(HERE, "test_gpu_sort.py"), "-k", sel],
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
