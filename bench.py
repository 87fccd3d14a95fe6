#!/usr/bin/env python
"""Benchmark: text GB/s scanned per pattern (device-timed), % of B200 HBM peak.

One STEP = one pass of the whole hot path over the config's synthetic text:
  A1  device histogram of the (owned) text (N = 1: inside sm_count_batch; N > 1: by the
      bench, + NCCL all_reduce, so every rank uses the same order)
  A2  rarest-first order pi per pattern (host, from the histogram)
  A3-A7 one counting search launch per pattern (TMA staging, peeled packed-byte
      compares, early exit, popcount/atomics)          [+ all_reduce of counts]
Default workload = BASELINE.json configs[1] (c2, English-like 256 MiB text, 100
patterns at each m in {2,4,...,1024}).  value = text bytes x patterns / step time
(GB = 1e9 B), whole job.  Reporting (A8) is timed in the same run as the
`report` sub-object.  Multi-GPU: weak scaling, each rank holds a 256 MiB shard
of an N x 256 MiB text (+1023-byte halo) and counts its owned alignments.

`--config c5` is the multi-GPU scale config of BASELINE.json (configs[4]): a 64 GiB
text of uniform bytes, STRONG scaling -- the same 2^36-byte text is sharded over the
N ranks (each holds its 2^36 / N owned bytes + a 63-byte halo), 200 patterns (28 of
them per length straddle the k/8 shard cuts).

`--gpus N` without a launcher re-executes itself under torch.distributed.run with N
processes (one per GPU; refused when fewer than N GPUs are visible).  `--fused` sums
the counts through an NVLink multicast buffer (NEXT-4) instead of an NCCL all_reduce
where the platform provides one.

Counts of a full-size config are compared, pattern by pattern, with the oracle's
golden answers (tests/golden/<config>.json, from tools/make_golden.py); a mismatch
fails the run.

`--impl reference` times the CPU oracle (oracle/, plain Alg. 1) on the host
cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0
SPEC_HBM_GBS = 8000.0  # B200 HBM3e spec (north star: ">= 70 % of B200 HBM read bandwidth" = 5.6 TB/s)
METRIC = "text GB/s scanned per pattern (device-timed) vs m; % of B200 HBM peak, 1/2/4/8 GPU"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["native", "reference"], default="native")
    ap.add_argument("--config", default="c2")
    ap.add_argument("--per-m", type=int, default=None, help="patterns per length (default: config's)")
    ap.add_argument("--lengths", default=None, help="comma list of pattern lengths (default: config's)")
    ap.add_argument("--shard-bytes", type=int, default=None, help="text bytes per GPU (default: config n)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-report", action="store_true")
    ap.add_argument("--no-dense", action="store_true", help="skip the dense-report (NEXT-1) measurement")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--strategy", type=int, default=0)
    ap.add_argument("--peel", type=int, default=0)
    ap.add_argument("--fused", action="store_true", help="NVLS multicast count reduction (NEXT-4) for N > 1")
    return ap.parse_args()


L2_FLUSH_BYTES = 256 << 20  # > 2x the 126 MB L2
STRONG = {"c5"}  # configs whose total text is fixed as N grows (BASELINE.json configs[4])


def maybe_relaunch(args):
    """`bench.py --gpus N` started as a plain process: run N ranks under torch.distributed.run
    (the driver's own launch sets WORLD_SIZE and lands in run_native directly)."""
    if "WORLD_SIZE" in os.environ or args.gpus <= 1 or args.impl == "reference":
        return
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but {have} CUDA device(s) visible; refusing to run "
                         f"fewer ranks than asked\n")
        sys.exit(2)
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def nccl_init_lines(path):
    """The communicator-init lines of this rank's NCCL_DEBUG=INFO log (they name nranks)."""
    try:
        lines = [ln.strip() for ln in open(path, errors="replace") if "nranks" in ln and "Init COMPLETE" in ln]
        return lines[:2]
    except OSError:
        return []


def golden_check(config: str, counts, n: int, P: int):
    """Compare every count with tests/golden/<config>.json (oracle answers, tools/make_golden.py);
    None when the run is not the golden workload (sizes or pattern set overridden)."""
    path = os.path.join(ROOT, "tests", "golden", f"{config}.json")
    if not os.path.exists(path):
        return {"golden": None, "note": f"{os.path.relpath(path, ROOT)} not written"}
    g = json.load(open(path))
    if g["n"] != n or len(g["cases"]) != P:
        return None
    want = [c["count"] for c in g["cases"]]
    bad = [i for i, (a, b) in enumerate(zip(counts, want)) if int(a) != int(b)]
    if bad:
        raise SystemExit(f"bench.py: {len(bad)} of {P} counts differ from the oracle's golden answers "
                         f"({os.path.relpath(path, ROOT)}), first pattern {bad[0]}: {int(counts[bad[0]])} != "
                         f"{want[bad[0]]}")
    return {"golden": os.path.relpath(path, ROOT), "patterns": P, "mismatches": 0,
            "count_sum": int(sum(want))}


def traffic_per_pass(config: str, n: int):
    """DRAM read+write bytes per pattern pass from the committed ncu capture of this config's
    count kernel (profiles/traffic_<config>.json, tools/ncu_traffic.py), scaled to this run's n
    when the capture ran on a prefix of the text (its traffic_over_algorithmic ratio)."""
    path = os.path.join(ROOT, "profiles", f"traffic_{config.lower()}.json")
    try:
        t = json.load(open(path))
        if int(t["text_bytes"]) == int(n):
            return float(t["traffic_per_pattern_pass"])
        return float(t["traffic_over_algorithmic"]) * n
    except Exception:
        return None


def read_probe():
    """Measured read-only streaming ceiling of the search kernel's TMA configuration (profiles/probe_r1.json)."""
    try:
        return float(json.load(open(os.path.join(ROOT, "profiles", "probe_r1.json")))["read_stream_GBps"])
    except Exception:
        return None


def load_profile(name):
    try:
        return json.load(open(os.path.join(ROOT, "profiles", name)))
    except Exception:
        return None


def peaks():
    try:
        d = json.load(open(MEASURED_PEAKS))
        return float(d["hbm_gbs"]), "measured", d
    except Exception:
        return FALLBACK_HBM_GBS, "fallback", {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self):
        """Host time of a region boundary (samples are kept only between mark() calls)."""
        return time.time()

    def stop(self, t0=None, t1=None):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = [ln for t, ln in self.lines if (t0 is None or t >= t0) and (t1 is None or t <= t1 + 0.06)]
        window = "timed region"
        if not lines and t0 is not None and t1 is not None:
            # a timed region shorter than the 50 ms sampling period (c1: ~2 ms): the samples
            # nearest to it, taken while the warm GPU idles between the barriers
            lines = [ln for t, ln in self.lines if t0 - 0.3 <= t <= t1 + 0.3]
            window = f"+-0.3 s around a {1e3 * (t1 - t0):.1f} ms timed region"
        for ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "window": window}


# ----------------------------------------------------------------------------- workload

def build_workload(args, rank: int, world: int):
    import synth
    cfg = args.config.lower()
    base = synth.text_spec(cfg)
    if cfg in STRONG:   # the total text is fixed; ranks split it
        N = args.shard_bytes * world if args.shard_bytes else base.n
    else:               # weak scaling: every rank holds a config-sized shard
        N = (args.shard_bytes or base.n) * world
    spec = synth.text_spec(cfg, n=N)
    lengths = [int(x) for x in args.lengths.split(",")] if args.lengths else None
    pats = synth.patterns(cfg, spec=spec, per_m=args.per_m, lengths=lengths)
    return spec, pats


# ----------------------------------------------------------------------------- reference arm (CPU oracle)

def cpu_oracle_sample(spec, pats, seconds: float, threads: int):
    """Oracle (plain Alg. 1) GB/s on the host cores over a bounded sample of the workload.

    Sample: the first min(n, 64 MiB) bytes of the text; patterns taken round-robin over
    the config's lengths; threads = all host cores (ctypes releases the GIL)."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle
    oracle.build()
    sample_n = min(spec.n, 64 << 20)
    text = spec.host(0, sample_n)
    by_m = {}
    for p in pats:
        by_m.setdefault(p.m, []).append(p.data)
    order = []
    k = 0
    while len(order) < 4 * threads * 8:
        for m in sorted(by_m):
            if k < len(by_m[m]):
                order.append(by_m[m][k])
        k += 1
        if k > max(len(v) for v in by_m.values()):
            break
    done_bytes = 0
    done = 0
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        i = 0
        while i < len(order) and time.perf_counter() - t0 < seconds:
            batch = order[i:i + threads]
            list(ex.map(lambda p: oracle.naive_count(p, text), batch))
            done_bytes += sample_n * len(batch)
            done += len(batch)
            i += threads
    dt = time.perf_counter() - t0
    # single-thread oracle per pattern length: 3 patterns per m on an 8 MiB prefix
    small = text[: min(sample_n, 8 << 20)]
    per_m = {}
    for m in sorted(by_m):
        ts = time.perf_counter()
        k = min(3, len(by_m[m]))
        for p in by_m[m][:k]:
            oracle.naive_count(p, small)
        per_m[str(m)] = round(small.size * k / (time.perf_counter() - ts) / 1e9, 3)
    return {
        "value": done_bytes / dt / 1e9,
        "unit": "GB/s",
        "cores": threads,
        "kind": "oracle",
        "sample": f"plain Alg. 1 (oracle/oracle.c, gcc -O2) counting {done} patterns of the config's lengths "
                  f"over the first {sample_n >> 20} MiB of the {spec.name} text, {threads} threads, {dt:.1f} s",
        "single_thread_GBps_per_m": per_m,
        "single_thread_sample": f"3 patterns per m over the first {small.size >> 20} MiB, one thread",
    }


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    spec, pats = build_workload(args, 0, 1)
    threads = len(os.sched_getaffinity(0))
    per_step = max(2.0, args.cpu_seconds / 4)
    for _ in range(args.warmup):
        cpu_oracle_sample(spec, pats, 0.5, threads)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        vals.append(cpu_oracle_sample(spec, pats, per_step, threads))
    total = time.perf_counter() - t0
    v = sum(x["value"] for x in vals) / len(vals)
    cb = dict(vals[-1])
    cb["value"] = v
    out = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": spec.name, "text_bytes": spec.n, "patterns": len(pats),
                   "lengths": sorted({p.m for p in pats}), "world": world},
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# ----------------------------------------------------------------------------- native arm

def dense_report(sm, synth, dev, stream, peak, reps: int = 3):
    """NEXT-1: reporting at the highest match density -- the periodic text a^(2^30) of
    configs[3] with p = a^17: every alignment matches, 2^30 - 16 positions (8 GiB) are
    written.  Bound: HBM read + write; bytes moved = n (text) + 8 x positions."""
    import torch
    spec = synth.text_spec("c4p")
    t = synth.gen_text_device(spec, 0, spec.n)
    m = 17
    total = spec.n - m + 1
    pos = torch.empty(total, dtype=torch.int64, device=dev)
    d = torch.zeros(1, dtype=torch.int64, device=dev)
    pb = sm.PatternBatch([b"a" * m])
    # A1 once per text (timed separately, amortised over the patterns)
    hist = sm.sm_histogram(t)
    sm.sm_report_batch(pb, t, pos, d, hist=hist)
    torch.cuda.synchronize()
    assert int(d.item()) == total
    assert int(pos[-1].item()) == total - 1 and int(pos[12345].item()) == 12345
    ms, hist_ms = [], []
    for _ in range(reps):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(stream)
        hist = sm.sm_histogram(t)
        e1.record(stream)
        sm.sm_report_batch(pb, t, pos, d, hist=hist)
        e2.record(stream)
        torch.cuda.synchronize()
        hist_ms.append(e0.elapsed_time(e1))
        ms.append(e1.elapsed_time(e2))
    best = min(ms)
    moved = spec.n + 8 * total
    gbs = moved / (best * 1e-3) / 1e9
    del pos, t
    torch.cuda.empty_cache()
    return {"workload": "c4p periodic a^(2^30), p = a^17 (every alignment matches)", "positions": total,
            "ms": round(best, 3), "histogram_ms": round(min(hist_ms), 3), "bytes_moved": moved, "GBps": round(gbs, 1), "frac_of_peak": round(gbs / peak, 4),
            "text_GBps": round(spec.n / (best * 1e-3) / 1e9, 1)}


def run_native(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1612_01506_b200 as sm
    import synth
    from paper_1612_01506_b200 import dist as smd

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started {world} rank(s)")
    if torch.cuda.device_count() <= local:
        raise SystemExit(f"bench.py: rank {rank} needs CUDA device {local}; {torch.cuda.device_count()} visible")
    torch.cuda.set_device(local)
    nccl_log = None
    if world > 1:
        # NCCL's own communicator-init lines (nranks, NVLS/NVLink use) go to a per-rank log;
        # rank 0 quotes them in its JSON line
        nccl_log = f"/tmp/smgpu_bench_nccl.{os.getpid()}.log"
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", nccl_log)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist.barrier()
    dev = torch.device("cuda", local)
    sm.load_library()
    synth.build()

    cfg = args.config.lower()
    strong = cfg in STRONG
    spec, pats = build_workload(args, rank, world)
    max_m = max(p.m for p in pats)
    shard = smd.make_shard(spec.n, rank, world, halo=max(0, max_m - 1))
    if strong:
        args.no_e2e = True      # a 64 GiB text: no pinned host copy of it (device-resident config)
        args.no_report = True
    text = synth.gen_text_device(spec, shard.own_lo, shard.held_len)
    owned = text[: shard.owned_bytes]
    P = len(pats)
    pdata = [p.data for p in pats]
    views = [text[: shard.view_len(p.m)] for p in pats]
    held = text[: shard.held_len]
    counts = torch.zeros(P, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream()

    pbatch = sm.PatternBatch(pdata)
    mc = None
    if args.fused and world > 1:
        mc = smd.MulticastCounts(P, dev)
    fused = bool(mc is not None and mc.available)

    def step(ev=None):
        if world == 1:
            # A1 inside the call: the library histograms t itself (its own, trusted histogram:
            # no device support check / fallback launches for PACKED, R21), then A2..A7
            if ev is not None:
                ev[0].record(stream)
            sm.sm_count_batch(pbatch, held, counts, hist=None, max_alignments=shard.owned_bytes,
                              strategy=args.strategy)
            if ev is not None:
                ev[1].record(stream)
                ev[2].record(stream)
            return None
        h = smd.global_histogram(text, shard)             # A1 (+ all_reduce: one pi on every rank, R14)
        hh = h.cpu().numpy().astype(np.uint64)           # 2 KiB D2H for the host-side order (A2)
        if ev is not None:
            ev[0].record(stream)
        if fused:  # NEXT-4: search + multimem.red into every rank's copy (no NCCL call)
            c = smd.count_sharded_fused(pbatch, held, shard, hh, mc, strategy=args.strategy)
            if ev is not None:
                ev[1].record(stream)
                ev[2].record(stream)
            counts.copy_(c)
            return hh
        # A2 (host, per pattern) + A3..A7: each pattern a full pass over the shard
        sm.sm_count_batch(pbatch, held, counts, hist=hh, max_alignments=shard.owned_bytes,
                          strategy=args.strategy)
        if ev is not None:
            ev[1].record(stream)
        smd.allreduce_sum_(counts)
        if ev is not None:
            ev[2].record(stream)
        return hh

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 1)):
        step()
    barrier()
    # the text's histogram for the diagnostics below (plans, per-length passes): outside the timed region
    hh = smd.global_histogram(text, shard).cpu().numpy().astype(np.uint64)

    # ---------------- timed region (device time, max over ranks)
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)  # let nvidia-smi deliver its first sample before the timed region
    launches0 = sm.sm_launch_count()
    evs = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # A shard that fits in the 126 MB L2 (c1: 1 MiB) would otherwise be served from L2 by every
    # step after the first: write a buffer larger than L2 between timed steps and time each step
    # on its own events (the flush stays outside them).  Larger shards stream from HBM anyway.
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev) \
        if shard.held_len < L2_FLUSH_BYTES else None
    step_ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(2)) for _ in range(args.steps)]
    barrier()
    h0 = clk.mark()
    start.record(stream)
    for s in range(args.steps):
        if flush is not None:
            flush.fill_(s)
            step_ev[s][0].record(stream)
        step(evs[s])
        if flush is not None:
            step_ev[s][1].record(stream)
    end.record(stream)
    barrier()
    h1 = clk.mark()
    launches = sm.sm_launch_count() - launches0
    total_ms = start.elapsed_time(end)
    if flush is not None:
        total_ms = sum(a.elapsed_time(b) for a, b in step_ev)
        del flush
    search_ms = sum(e[0].elapsed_time(e[1]) for e in evs) / args.steps   # the P search launches of a step
    coll_ms = sum(e[1].elapsed_time(e[2]) for e in evs) / args.steps     # the count all_reduce (N > 1)
    if h1 - h0 < 0.2:
        time.sleep(0.3)  # short region: let the sampler deliver the samples after it (stop()'s fallback window)
    clocks = clk.stop(h0, h1)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    bytes_per_step = spec.n * P
    value = bytes_per_step / (ms_per_step * 1e-3) / 1e9

    # roofline of the dominant kernel (this rank): algorithmic bytes (n of each launch's
    # view) / average launch duration, from the events bracketing the step's launches
    local_bytes = np.array([v.numel() for v in views], dtype=np.float64)
    peak, peak_kind, pk = peaks()
    achieved = float(local_bytes.sum() / (search_ms * 1e-3) / 1e9)
    lens = sorted({p.m for p in pats})

    # per-length breakdown (diagnostic pass after the timed region; same launches)
    per_m = {}
    for m in lens:
        idx = [i for i, p in enumerate(pats) if p.m == m]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sub = sm.PatternBatch([pdata[i] for i in idx])
        dsub = torch.zeros(len(idx), dtype=torch.int64, device=dev)
        hsub = hh if world > 1 else None  # as in the timed step
        sm.sm_count_batch(sub, held, dsub, hist=hsub, max_alignments=shard.owned_bytes)  # warm (lazy module load)
        e0.record(stream)
        sm.sm_count_batch(sub, held, dsub, hist=hsub, max_alignments=shard.owned_bytes)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        gbs = float(local_bytes[idx].sum() / (ms * 1e-3) / 1e9)
        per_m[str(m)] = {"GBps": round(gbs, 1), "frac_of_peak": round(gbs / peak, 4),
                         "frac_of_spec_8TBps": round(gbs / SPEC_HBM_GBS, 4),
                         "us_per_launch": round(ms * 1e3 / len(idx), 2)}
    step()  # restore counts of the full step
    torch.cuda.synchronize()
    counts_host = counts.cpu().numpy()
    # every global count vs the oracle's golden answer (1 GPU, or the strong-scaling c5 at any N)
    parity = golden_check(cfg, counts_host, spec.n, P) if (world == 1 or strong) else None

    # ---------------- end-to-end through the public API (host text in pinned memory)
    # Every step copies its text from pinned host memory (H2D) and reads its counts back
    # (D2H).  Texts are double-buffered on the device: step k+1's copy runs on a copy
    # stream while step k computes (a stream of texts), all inside the timed region.
    e2e = None
    if not args.no_e2e:
        host_text = torch.empty(text.numel(), dtype=torch.uint8, pin_memory=True)
        host_text.copy_(text)
        counts_h = torch.empty(P, dtype=torch.int64, pin_memory=True)
        bufs = [torch.empty_like(text) for _ in range(2)]
        copy_stream = torch.cuda.Stream(device=dev)
        copied = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]
        for ev in consumed:
            ev.record(stream)

        def issue_copy(i):
            b = i % 2
            copy_stream.wait_event(consumed[b])            # the buffer's previous step is done
            with torch.cuda.stream(copy_stream):
                bufs[b].copy_(host_text, non_blocking=True)  # H2D of step i's input
            copied[b].record(copy_stream)

        def compute(i):
            b = i % 2
            stream.wait_event(copied[b])
            held_b = bufs[b][: shard.held_len]
            hh2 = None  # N = 1: the library histograms the text itself (as in the timed step)
            if world > 1:
                hh2 = smd.global_histogram(bufs[b], shard).cpu().numpy().astype(np.uint64)
            sm.sm_count_batch(pbatch, held_b, counts, hist=hh2, max_alignments=shard.owned_bytes)
            consumed[b].record(stream)
            smd.allreduce_sum_(counts)
            counts_h.copy_(counts, non_blocking=True)      # D2H of step i's result

        issue_copy(0)
        compute(0)
        barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        copy_stream.wait_event(s0)
        issue_copy(0)
        for i in range(args.steps):
            if i + 1 < args.steps:
                issue_copy(i + 1)
            compute(i)
        s1.record(stream)
        barrier()
        et = torch.tensor([s0.elapsed_time(s1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e_ms = float(et.item()) / args.steps
        assert np.array_equal(counts_h.numpy(), counts_host), "e2e counts differ from device-resident run"
        e2e = {"value": bytes_per_step / (e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(text.numel()), "d2h_bytes_per_step": int(8 * P),
               "pipelining": "double-buffered device text: step k+1's H2D overlaps step k's compute"}
        del bufs, host_text

    # ---------------- reporting (A8), one pass over all patterns, N = 1 only
    report = None
    if not args.no_report and world == 1:
        tot = int(counts_host.sum())
        posbuf = torch.empty(max(tot, 1), dtype=torch.int64, device=dev)
        dcnt = torch.zeros(P, dtype=torch.int64, device=dev)

        def rep():
            sm.sm_report_batch(pbatch, held, posbuf, dcnt, hist=hh, max_alignments=shard.owned_bytes)
        rep()
        torch.cuda.synchronize()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        rep()
        r1.record(stream)
        torch.cuda.synchronize()
        r_ms = r0.elapsed_time(r1)
        assert np.array_equal(dcnt.cpu().numpy(), counts_host), "report totals differ from counts"
        report = {"value": spec.n * P / (r_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_pass": r_ms,
                  "positions_written": tot, "position_bytes": 8 * tot,
                  "passes": "one text read per pattern (staged match records + expand), see DESIGN.md"}
        # per pattern length: report pass time vs the same patterns' count launches (diagnostic)
        rp = {}
        for m in lens:
            idx = [i for i, p in enumerate(pats) if p.m == m]
            sub = sm.PatternBatch([pdata[i] for i in idx])
            dsub = torch.zeros(len(idx), dtype=torch.int64, device=dev)
            subtot = int(counts_host[idx].sum())

            def rep_m():
                sm.sm_report_batch(sub, held, posbuf[: max(subtot, 1)], dsub, hist=hh,
                                   max_alignments=shard.owned_bytes)
            rep_m()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rep_m()
            e1.record(stream)
            torch.cuda.synchronize()
            ms_m = e0.elapsed_time(e1)
            rp[str(m)] = {"GBps": round(float(local_bytes[idx].sum()) / (ms_m * 1e-3) / 1e9, 1),
                          "positions": subtot, "report_over_count": round(
                              ms_m * 1e3 / len(idx) / per_m[str(m)]["us_per_launch"], 3)}
        report["per_m"] = rp
        del posbuf
        if not args.no_dense:
            report["dense"] = dense_report(sm, synth, dev, stream, peak)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    cpu = None
    if not args.no_cpu and world == 1:
        cpu = cpu_oracle_sample(spec, pats, args.cpu_seconds, len(os.sched_getaffinity(0)))

    # NEXT-3: a batch over a <= 4-symbol text runs PACKED on the code array packed once per
    # call, so each pass reads n b / 8 code bytes: the kernel is bound by the INT-ALU pipe
    # (compare steps), not HBM.  Roofline: ALU warp-instructions of the step's search
    # launches (instruction counts from the committed ncu capture profiles/alu_<config>.json,
    # tools/ncu_alu.py -- counts do not depend on timing) / the live search time, against
    # the measured ALU-pipe ceiling (profiles/alu_probe_r2.json, tools/alu_probe.py)
    roofline_pre = None
    nsym = int((hh > 0).sum())
    if nsym <= 4 and P >= 2:
        b = 1 if nsym <= 2 else 2
        code_gbs = (spec.n * b / 8 * P + spec.n) / (search_ms * 1e-3) / 1e9
        alu = load_profile(f"alu_{cfg}.json")
        probe = load_profile("alu_probe_r2.json")
        work = alu.get("alu_warp_inst_per_step") if alu and alu.get("patterns") == P and \
            alu.get("text_bytes") == spec.n and world == 1 else None
        peak_alu = probe.get("alu_warp_inst_per_s") if probe else None
        ach = work / (search_ms * 1e-3) if work else None
        roofline_pre = {
            "bound": "alu", "achieved": ach, "peak": peak_alu, "unit": "ALU-pipe warp-instructions/s",
            "frac": round(ach / peak_alu, 4) if ach and peak_alu else None, "traffic": None,
            "alu_warp_inst_per_step": work, "peak_source": "profiles/alu_probe_r2.json (LOP3/SHF chains, all SMs)",
            "work_source": f"profiles/alu_{cfg}.json (ncu smsp__inst_executed_pipe_alu.sum, search launches)",
            "issue_active_pct_ncu": alu.get("issue_active_pct") if alu else None,
            "alu_pipe_active_pct_ncu": alu.get("alu_pipe_active_pct") if alu else None,
            "text_equivalent_GBps": round(achieved, 1),
            "hbm_GBps_code_bytes": round(code_gbs, 1), "hbm_frac_code_bytes": round(code_gbs / peak, 4),
            "note": f"{b}-bit code array packed once per call; each pass reads n*{b}/8 bytes; compare-bound",
            "kernel": "search_kernel (PACKED-PRE count)", "avg_launch_us": round(search_ms * 1e3 / P, 2),
        }

    strategies = {}
    for p in pats[:: max(1, P // 200)]:
        s_, r_ = sm.sm_plan(p.data, hh)
        key = f"{sm.STRATEGY_NAMES[s_]}/r={r_}"
        strategies[key] = strategies.get(key, 0) + 1

    out = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic",
        "config": {
            "workload": spec.name, "text_bytes": spec.n, "text_bytes_per_gpu": shard.owned_bytes,
            "patterns": P, "lengths": lens, "parallelism": f"text-shard x{world}",
            "l2": (f"inputs larger than L2 ({shard.held_len / 2**20:.0f} MiB/GPU vs 126 MB); "
                   "TMA loads use L2 evict_first") if shard.held_len >= L2_FLUSH_BYTES else
                  (f"text ({shard.held_len / 2**20:.0f} MiB) fits in L2: a {L2_FLUSH_BYTES >> 20} MiB buffer "
                   "is written between timed steps, each step timed on its own events (flush excluded)"),
            "step": "hist + per-pattern order + batched count launches (each pattern a full pass) (+ all_reduce)",
            "halo_bytes": shard.halo,
        },
        "collective": None if world == 1 else {
            "kind": "NVLS multimem.red (count_sharded_fused)" if fused else "NCCL all_reduce int64[P] (SUM)",
            "fused_requested": bool(args.fused), "multicast_available": fused,
            "ms_per_step": round(coll_ms, 4), "search_ms_per_step": round(search_ms, 4),
            "value_without_collective": round(bytes_per_step / ((ms_per_step - coll_ms) * 1e-3) / 1e9, 2),
            "nccl_init": nccl_init_lines(nccl_log) if nccl_log else [],
        },
        "parity": parity,
        "gpu_launches": int(launches),
        "roofline": roofline_pre if roofline_pre else {
            "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4),
            # DRAM read+write bytes per pattern pass, from the committed ncu --set full capture of
            # this kernel (profiles/traffic_c2.json, written by tools/ncu_traffic.py); null elsewhere
            "traffic": traffic_per_pass(args.config, spec.n),
            "traffic_unit": "bytes per pattern pass (algorithmic n = %d)" % spec.n, "avg_launch_us": round(search_ms * 1e3 / P, 2),
            # the same pass seen from DRAM: captured traffic per pass / this run's average pass time
            **dram_side(traffic_per_pass(args.config, spec.n), search_ms * 1e-3 / P, peak),
            "kernel": "search_kernel (count)", "peak_kind": peak_kind,
            "algorithmic_bytes_per_launch": "n (text bytes of the launch's view)",
            "read_stream_probe": read_probe(),
            # report all three denominators; the north star's ">= 70 %" is of the 8 TB/s spec
            "spec_peak_GBps": SPEC_HBM_GBS, "frac_of_spec": round(achieved / SPEC_HBM_GBS, 4),
            "frac_of_read_stream_probe": (round(achieved / read_probe(), 4) if read_probe() else None),
            "frac_note": "achieved counts the algorithmic n bytes of every pattern pass; the DRAM traffic per pass is "
                         "`traffic` (< n: alternating passes of a batch reuse the 126 MB L2) and the peak is the "
                         "measured COPY (read+write) rate, so frac can exceed 1 for a read-only stream; "
                         "dram_achieved / dram_frac are the same pass counted in DRAM bytes (traffic / avg_launch_us)",
        },
        "per_m": per_m,
        "clocks": clocks,
        "e2e": e2e,
        "report": report,
        "cpu_baseline": cpu,
        "plans": strategies,
        "count_checksum": int(counts_host.sum()),
    }
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def dram_side(traffic, pass_s, peak):
    """DRAM-side rate of one pattern pass: ncu-captured DRAM bytes per pass / the live average pass time.

    `frac` (algorithmic bytes) exceeds 1 when passes reuse the L2; `dram_frac` counts only what DRAM
    moved (it still passes 1 by a few percent where a read-only stream outruns the read+write copy
    the peak was measured with: c5, 7.56 TB/s probe vs the 6.46 TB/s copy)."""
    if not traffic or not pass_s or not peak:
        return {"dram_achieved": None, "dram_frac": None}
    gbs = traffic / pass_s / 1e9
    return {"dram_achieved": round(gbs, 1), "dram_frac": round(gbs / peak, 4)}


def main():
    args = parse()
    maybe_relaunch(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_native(args)


if __name__ == "__main__":
    main()
