"""Bounds-checked build: the edge-case workload (every strategy x epilogue, unaligned
views, texts ending exactly at the allocation end) runs under libsmgpu_debug.so,
whose kernels assert every global read range (never a byte outside t[0..n)) and
every shared-memory window (inside the tile's stage / code buffer).  A failed
assertion traps the kernel and fails this test.  compute-sanitizer is not
available on this pool; this is its stand-in.

The reporting staging pool size (SMGPU_STAGE_BYTES) is a performance knob: 0 sends
every tile with matches through the overflow pass (recompute from the text), a
few KiB splits the tiles between staged records and the overflow pass; results
must not change (run with both the debug and the release library)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("lib_kind,stage_bytes", [("debug", None), ("debug", "0"), ("debug", "4096"),
                                                  ("release", "0"), ("release", "20000")])
def test_debug_build_bounds_assertions(lib_kind, stage_bytes):
    from paper_1612_01506_b200 import _build
    lib = _build.build(debug=lib_kind == "debug")
    assert os.path.exists(lib)
    env = dict(os.environ)
    env.pop("SMGPU_STAGE_BYTES", None)
    if lib_kind == "debug":
        env["SMGPU_LIB"] = "debug"
    if stage_bytes is not None:
        env["SMGPU_STAGE_BYTES"] = stage_bytes
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "debug_workload.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert "SMGPU_DCHECK failed" not in out, out[-3000:]
    assert r.returncode == 0, out[-3000:]
    assert "mismatches: 0" in out
