"""bench.py's multi-GPU launch contract on the host (no GPU here):

* `bench.py --gpus N` started as a plain process re-executes itself under
  torch.distributed.run with N ranks on 127.0.0.1 -- and refuses (exit 2) when fewer
  than N GPUs are visible, instead of silently measuring one GPU;
* a rank started by a launcher checks WORLD_SIZE against --gpus;
* the strong-scaling config (c5) keeps the total text fixed while the weak ones grow.
"""
import os
import subprocess
import sys
import types

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_refuses_more_gpus_than_visible():
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 2, r.stderr[-2000:]
    assert "refusing" in r.stderr
    assert r.stdout.strip() == ""   # no JSON line: nothing was measured


def test_relaunch_command(monkeypatch):
    import torch
    calls = []
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(torch.cuda, "device_count", lambda: 8)
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "5", "--config", "c5"])
    args = bench.parse()
    with pytest.raises(SystemExit) as e:
        bench.maybe_relaunch(args)
    assert e.value.code == 0
    (cmd,) = calls
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-6:] == ["--gpus", "4", "--steps", "5", "--config", "c5"]


def test_no_relaunch_under_a_launcher_or_for_one_gpu(monkeypatch):
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: pytest.fail("must not relaunch"))
    monkeypatch.setenv("WORLD_SIZE", "4")
    bench.maybe_relaunch(types.SimpleNamespace(gpus=4, impl="native"))
    monkeypatch.delenv("WORLD_SIZE")
    bench.maybe_relaunch(types.SimpleNamespace(gpus=1, impl="native"))
    bench.maybe_relaunch(types.SimpleNamespace(gpus=8, impl="reference"))  # CPU arm: rank 0 only


@pytest.mark.parametrize("world", [1, 2, 8])
def test_strong_and_weak_workloads(world):
    import synth
    strong = bench.build_workload(types.SimpleNamespace(config="c5", shard_bytes=None, lengths=None, per_m=None),
                                  0, world)
    assert strong[0].n == 1 << 36 and len(strong[1]) == 200
    weak = bench.build_workload(types.SimpleNamespace(config="c2", shard_bytes=1 << 20, lengths="8", per_m=2),
                                0, world)
    assert weak[0].n == world << 20
    assert synth.text_spec("c5").n == 1 << 36


def test_traffic_scales_a_prefix_capture_to_the_run():
    import json
    for cfg in ("c2", "c3", "c5"):
        t = json.load(open(os.path.join(ROOT, "profiles", f"traffic_{cfg}.json")))
        n = int(t["text_bytes"])
        assert bench.traffic_per_pass(cfg, n) == t["traffic_per_pattern_pass"]
        assert abs(bench.traffic_per_pass(cfg, 16 * n) - 16 * n * t["traffic_over_algorithmic"]) < 1.0
        assert 0.5 < t["traffic_over_algorithmic"] < 1.1  # DRAM bytes per pass ~ n (less with L2 reuse)
    assert bench.traffic_per_pass("c4", 1 << 32) is None  # compare-bound: no HBM traffic key


def test_golden_check_catches_a_wrong_count():
    import json
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "c1.json")))
    want = [c["count"] for c in g["cases"]]
    ok = bench.golden_check("c1", want, g["n"], len(want))
    assert ok["mismatches"] == 0 and ok["count_sum"] == g["count_sum"]
    bad = list(want)
    bad[17] += 1
    with pytest.raises(SystemExit):
        bench.golden_check("c1", bad, g["n"], len(want))
    assert bench.golden_check("c1", want, g["n"] + 1, len(want)) is None  # not the golden workload


def test_reference_arm_under_torchrun_two_ranks():
    """The driver's reference launch at N = 2 (torch.distributed.run, 127.0.0.1): rank 0
    alone runs the oracle and prints ONE JSON line; rank 1 exits 0 without work."""
    import json
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--cpu-seconds", "1",
           "--config", "c1"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["config"]["world"] == 2
    assert d["cpu_baseline"]["kind"] == "oracle" and d["value"] > 0


def test_clock_sampler_short_region_window():
    """A timed region shorter than the 50 ms sampling period takes the samples within
    +-0.3 s of it (and says so); a long region keeps only its own samples."""
    c = bench.ClockSampler(0)

    class _P:
        def terminate(self):
            pass

        def wait(self, timeout=None):
            return 0

    c.proc = _P()
    row = "1965, 1965, 700.0, Not Active, Not Active, Not Active, {}"
    c.lines = [(10.00, row.format("Not Active")), (10.25, row.format("Active")), (11.0, row.format("Not Active"))]
    short = c.stop(10.1, 10.102)
    assert short["samples"] == 2 and short["reasons"] == ["sw_power_cap"] and "around" in short["window"]
    c.proc = _P()
    long_ = c.stop(10.2, 10.9)
    assert long_["samples"] == 1 and long_["window"] == "timed region" and long_["sm_mhz"] == 1965.0


def test_l2_flush_threshold():
    """Shards below the flush size (c1's 1 MiB) get an L2 flush between timed steps;
    the default c2 shard (256 MiB + halo) streams from HBM without one."""
    assert bench.L2_FLUSH_BYTES >= 2 * 126 * 10**6
    assert (1 << 20) < bench.L2_FLUSH_BYTES <= (256 << 20) + 1023


def test_dram_side_of_the_roofline():
    """roofline.dram_frac = captured DRAM bytes per pass / live pass time / peak; null without a capture."""
    import bench
    d = bench.dram_side(195931006.5, 34.01e-6, 6461.5)
    assert abs(d["dram_achieved"] - 5761.0) < 1.0 and abs(d["dram_frac"] - 0.8916) < 2e-4
    assert bench.dram_side(None, 34.01e-6, 6461.5) == {"dram_achieved": None, "dram_frac": None}
    assert bench.dram_side(1.0, 0.0, 6461.5) == {"dram_achieved": None, "dram_frac": None}
