"""NEXT-4: counting with the all-reduce fused into the search kernel's last-CTA epilogue (multimem.red on an
NVLink multicast address).  On this single-GPU box the multicast group has one member, so
the reduction must reproduce the plain counts exactly; with N ranks bound to the same
multicast object every rank's copy receives the sum (smgpu.h sm_count_batch_multicast)."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_multicast_counts_equal_plain_counts():
    import paper_1612_01506_b200 as sm
    from nvls_util import MulticastU64
    try:
        mc = MulticastU64(256)
    except Exception as e:  # no multicast on this box / driver
        pytest.skip(f"NVLink multicast unavailable: {e}")
    spec = synth.text_spec("c2", n=(8 << 20) + 77)
    t = synth.gen_text_device(spec, 0, spec.n)
    a = t.cpu().numpy()
    pats = [p.data for p in synth.patterns("c2", spec=spec, per_m=6)]
    assert len(pats) <= 256
    h = oracle.hist(a)
    d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
    sm.sm_count_batch(pats, t, d, hist=h)
    want = d.cpu().numpy().astype(np.uint64)
    for lim in (None, spec.n // 2):  # whole text, and a shard's owned alignments
        if lim is not None:
            sm.sm_count_batch(pats, t, d, hist=h, max_alignments=lim)
            want = d.cpu().numpy().astype(np.uint64)
        mc.zero()
        sm.sm_count_batch_multicast(pats, t, mc.multicast_ptr, hist=h, max_alignments=lim)
        torch.cuda.synchronize()
        got = mc.read()[: len(pats)]
        assert np.array_equal(got, want)
    # oracle parity on a few of them
    for i in range(0, len(pats), 13):
        assert int(want[i]) == oracle.naive_count(pats[i], a[: spec.n // 2 + len(pats[i]) - 1])


def test_last_cta_epilogue_protocol_emulated():
    """The fused epilogue's last-CTA-done protocol, validated on this single-GPU box with
    SMGPU_NVLS_EMULATE=1 (atomicAdd in place of multimem.red on a unicast buffer): every
    pattern's count lands exactly once per call, on multi-launch batches, shard limits
    and guarded PACKED launches (tests/nvls_emulate_workload.py)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SMGPU_NVLS_EMULATE="1")
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "nvls_emulate_workload.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "mismatches: 0" in out, out[-3000:]
