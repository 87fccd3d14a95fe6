#!/usr/bin/env python
"""INT-ALU pipe ceiling of one B200: the peak the compare-bound
regime (PACKED over sigma <= 4 texts, periodic text) is reported against.

Writes profiles/alu_probe_r2.json: warp-instructions/s and lane-ops/s of LOP3 and SHF
chains (the two ALU-pipe instructions of a PACKED compare step; an add chain is not
used because ptxas folds two dependent adds into one IADD3) over all SMs, the SM clock seen during the run (nvidia-smi), and the
nominal figure 148 SMs x 4 SMSPs x 0.5 ALU warp-instr/clk (rt_SMSP = 2,
B300_MICROARCH.md 'Pipe rates') x clock.

    python tools/alu_probe.py [--out profiles/alu_probe_r2.json]
"""
import ctypes
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libaluprobe.so")
SRC = os.path.join(HERE, "alu_probe.cu")


def build():
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(SRC):
        subprocess.check_call(["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC", "-gencode",
                               "arch=compute_100a,code=sm_100a", "-o", SO, SRC])
    return SO


def sass_counts():
    """ALU instructions in the inner loop of each probe kernel (cuobjdump of the .so)."""
    out = subprocess.run(["cuobjdump", "-sass", SO], capture_output=True, text=True).stdout
    res, cur = {}, None
    for ln in out.splitlines():
        if "Function :" in ln:
            cur = ln.split("Function :")[1].strip()
            res[cur] = {"LOP3": 0, "SHF": 0, "IADD3": 0}
        elif cur:
            for k in res[cur]:
                if f" {k}." in ln or f" {k} " in ln:
                    res[cur][k] += 1
    return res


def main():
    build()
    import torch
    torch.cuda.init()
    lib = ctypes.CDLL(SO)
    lib.alu_probe.restype = ctypes.c_float
    lib.alu_probe.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint32, ctypes.c_int]
    per_iter = lib.alu_probe_ops_per_iter()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits", "-lms", "50"],
                           stdout=subprocess.PIPE, text=True)
    res = {}
    iters = 1 << 16
    for op, name in ((0, "LOP3"), (1, "SHF")):
        for bps in (4, 8):
            blocks = sms * bps
            ms = lib.alu_probe(op, blocks, iters, 5)
            warp_inst = blocks * 8 * iters * per_iter   # 8 warps per 256-thread block
            res[f"{name} blocks/SM={bps}"] = {"ms": round(ms, 3),
                                              "warp_inst_per_s": warp_inst / (ms * 1e-3),
                                              "lane_ops_per_s": 32 * warp_inst / (ms * 1e-3)}
    smi.terminate()
    clocks = sorted(float(x) for x in smi.stdout.read().split() if x.replace(".", "").isdigit())
    clk = clocks[len(clocks) // 2] if clocks else None
    best = max(v["warp_inst_per_s"] for v in res.values())
    out = {
        "source": "tools/alu_probe.py on one B200 (gpurun): independent LOP3 / SHF chains (8 per thread), "
                  "all SMs, best of 5 launches, CUDA events",
        "alu_warp_inst_per_s": best,
        "alu_lane_ops_per_s": 32 * best,
        "sm_clock_mhz_median": clk,
        "nominal_alu_warp_inst_per_s_at_clock": (sms * 4 * 0.5 * clk * 1e6) if clk else None,
        "nominal_issue_warp_inst_per_s_at_clock": (sms * 4 * 1.0 * clk * 1e6) if clk else None,
        "sms": sms,
        "all": res,
        "sass_inner_loop_alu_instructions": sass_counts(),
    }
    path = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else os.path.join(ROOT, "profiles",
                                                                                        "alu_probe_r2.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "all"}, indent=1))


if __name__ == "__main__":
    main()
