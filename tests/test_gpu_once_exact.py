"""The count-once sort fallback (csrc/exact.cu: count_once_exact), used when a
survivor set is too large for the route path's 16-bit owners, forced for
every extension pass (IG_ONCE_EXACT_MIN_K=1, read once per process, hence a
subprocess) and checked against the reference goldens and the oracle."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def test_once_exact_fallback_matches(gpu_lib):
    env = dict(os.environ, IG_ONCE_EXACT_MIN_K="1")
    r = subprocess.run([sys.executable, os.path.join(HERE, "gpu_once_exact_check.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
