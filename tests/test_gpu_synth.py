"""Device generator == host generator (bit-identical inputs on both sides)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5"])
def test_device_matches_host(cfg):
    synth.build()
    spec = synth.text_spec(cfg, n=1 << 22)
    for start, length in [(0, 1 << 20), (1, 4099), (12345, 77777), ((1 << 22) - 17, 17), (3, 0)]:
        d = synth.gen_text_device(spec, start, length)
        h = spec.host(start, length)
        assert np.array_equal(d[:length].cpu().numpy(), h), (cfg, start, length)


def test_device_large_offset():
    spec = synth.text_spec("c5")
    start = (1 << 36) - 1000
    d = synth.gen_text_device(spec, start, 1000)
    assert np.array_equal(d.cpu().numpy(), spec.host(start, 1000))
