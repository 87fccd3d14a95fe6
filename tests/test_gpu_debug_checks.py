"""Bounds-checked build: the edge-case workload (every strategy x epilogue, unaligned
views, texts ending exactly at the allocation end) runs under libsmgpu_debug.so,
whose kernels assert every global read range (never a byte outside t[0..n)) and
every shared-memory window (inside the tile's stage / code buffer).  A failed
assertion traps the kernel and fails this test.  compute-sanitizer is not
available on this pool; this is its stand-in."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_debug_build_bounds_assertions():
    from paper_1612_01506_b200 import _build
    lib = _build.build(debug=True)
    assert os.path.exists(lib)
    env = dict(os.environ, SMGPU_LIB="debug")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "debug_workload.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert "SMGPU_DCHECK failed" not in out, out[-3000:]
    assert r.returncode == 0, out[-3000:]
    assert "mismatches: 0" in out
