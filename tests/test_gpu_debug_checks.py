"""Bounds-checked build: the edge-case workload (every strategy x epilogue, unaligned
views, texts ending exactly at the allocation end) runs under libsmgpu_debug.so,
whose kernels assert every global read range (never a byte outside t[0..n)) and
every shared-memory window (inside the tile's stage / code buffer).  A failed
assertion traps the kernel and fails this test.  compute-sanitizer is not
available on this pool; this is its stand-in.

The reporting staging pool size (SMGPU_STAGE_BYTES) is a performance knob: 0 sends
every tile with matches through the overflow pass (recompute from the text), a
few KiB splits the tiles between staged records and the overflow pass; results
must not change (run with both the debug and the release library).  Work dispatch
(static round-robin vs items fetched from a counter, chosen by the size of the call)
must not change them either: both are forced here on the small edge-case inputs."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


DISPATCH_ALWAYS = {"SMGPU_DISPATCH_MIN_MB": "0", "SMGPU_DISPATCH_MIN_MB_SINGLE": "0"}


@pytest.mark.parametrize("lib_kind,stage_bytes,extra", [
    ("debug", None, {}), ("debug", "0", {}), ("debug", "4096", {}),
    ("debug", None, DISPATCH_ALWAYS), ("debug", "4096", DISPATCH_ALWAYS),
    ("release", "0", {}), ("release", "20000", {}), ("release", None, DISPATCH_ALWAYS),
    # a pool of 3 chunks + 20 units: (stage bytes / 16) % kStageChunk = 20 < one bitmap
    # record, the case where a warp could claim a partial chunk it cannot use
    ("debug", str(16 * (3 * 512 + 20)), {}), ("release", str(16 * (3 * 512 + 20)), {}),
    ("release", None, {"SMGPU_DISPATCH": "0"})])
def test_debug_build_bounds_assertions(lib_kind, stage_bytes, extra):
    from paper_1612_01506_b200 import _build
    lib = _build.build(debug=lib_kind == "debug")
    assert os.path.exists(lib)
    env = dict(os.environ)
    env.pop("SMGPU_STAGE_BYTES", None)
    if lib_kind == "debug":
        env["SMGPU_LIB"] = "debug"
    if stage_bytes is not None:
        env["SMGPU_STAGE_BYTES"] = stage_bytes
    for k in ("SMGPU_DISPATCH", "SMGPU_DISPATCH_MIN_MB", "SMGPU_DISPATCH_MIN_MB_SINGLE"):
        env.pop(k, None)
    env.update(extra)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "debug_workload.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert "SMGPU_DCHECK failed" not in out, out[-3000:]
    assert r.returncode == 0, out[-3000:]
    assert "mismatches: 0" in out
