"""NEXT-2: device compare-step counters (libsmgpu_counters.so) pinned to the oracle's
Alg. 4 step count (tests/counters_workload.py); the release library must refuse."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_counters_match_oracle_alg4_steps():
    from paper_1612_01506_b200 import _build
    assert os.path.exists(_build.build(counters=True))
    env = dict(os.environ, SMGPU_LIB="counters")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "counters_workload.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "mismatches: 0" in out, out[-4000:]


def test_release_library_has_no_counters():
    import paper_1612_01506_b200 as sm
    if os.environ.get("SMGPU_LIB"):
        pytest.skip("an instrumented library is selected")
    with pytest.raises(sm.SmError):
        sm.sm_counters()
