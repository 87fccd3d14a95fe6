#!/usr/bin/env python
"""Sustained read-stream rate under the pool's power cap: the TMA ring probe (no compute) and the
count kernel (c5 text, FILTER) each run back to back for ~SECS seconds on one 64 GiB buffer, with
the achieved GB/s per batch next to the nvidia-smi SM clock / power / sw_power_cap samples.
usage: probe_sustained.py [GIB=64] [SECS=15] [both|count]   (writes JSON lines to stdout)"""
import ctypes, json, os, subprocess, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1612_01506_b200 as sm
import synth
from tools.probe import SO  # builds libprobe.so if needed

gib = int(sys.argv[1]) if len(sys.argv) > 1 else 64
secs = float(sys.argv[2]) if len(sys.argv) > 2 else 15.0
n = gib << 30
torch.cuda.set_device(0)
lib = ctypes.CDLL(SO)
lib.probe_tma.restype = ctypes.c_float
lib.probe_tma.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                          ctypes.c_uint32, ctypes.c_int, ctypes.c_int, ctypes.c_int]

samples = []


def smi():
    p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,clocks.mem,power.draw,clocks_event_reasons.sw_power_cap",
                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    for ln in p.stdout:
        samples.append((time.time(), ln.strip()))


threading.Thread(target=smi, daemon=True).start()
spec = synth.text_spec("c5", n=n)
t = synth.gen_text_device(spec, 0, n)
torch.cuda.synchronize()


def window(t0, t1):
    s = [x.split(",") for tt, x in samples if t0 <= tt <= t1]
    s = [[v.strip() for v in r] for r in s if len(r) >= 4]
    if not s:
        return {}
    sm_ = sorted(float(r[0]) for r in s)
    pw = sorted(float(r[2]) for r in s)
    return {"sm_mhz": sm_[len(sm_) // 2], "mem_mhz": s[-1][1], "power_w": pw[len(pw) // 2],
            "power_cap_frac": sum(r[3].lower() == "active" for r in s) / len(s)}


only = sys.argv[3] if len(sys.argv) > 3 else "both"
# 1) read-stream probe: 32 KiB tiles x 2 stages x 3 CTAs/SM, counter dispatch (the search kernel's ring)
t_start = time.time()
while only != "count" and time.time() - t_start < secs:
    a = time.time()
    gbs = lib.probe_tma(t.data_ptr(), n, 32768, 2, 3, 1, 8, 3, 1)
    b = time.time()
    print(json.dumps({"what": "probe", "t": round(a - t_start, 2), "GBps": round(gbs, 1), **window(a, b)}), flush=True)
if only == "both":
    time.sleep(8)  # cool down between the two series
# 2) the count kernel on the same text: 8 sampled c5 patterns of m = 16 per call (FILTER)
pats = [p.data for p in synth.patterns("c5", spec=spec, lengths=[16], per_m=50) if p.kind == "sampled"][:8]
assert len(pats) == 8, len(pats)
h = sm.sm_histogram(t).cpu().numpy().astype(np.uint64)
d = torch.zeros(len(pats), dtype=torch.int64, device="cuda")
pb = sm.PatternBatch(pats)
t_start = time.time()
while time.time() - t_start < secs:
    a = time.time()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sm.sm_count_batch(pb, t, d, hist=h)
    e1.record()
    torch.cuda.synchronize()
    b = time.time()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"what": "count_c5_m16x8", "t": round(a - t_start, 2), "GBps": round(n * len(pats) / ms / 1e6, 1),
                      **window(a, b)}), flush=True)
