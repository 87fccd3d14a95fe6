#!/usr/bin/env python
"""Read-bandwidth probes on a B200: plain LDG stream vs the TMA staging ring (no compute)."""
import ctypes, json, os, subprocess, sys
HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libprobe.so")
if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(os.path.join(HERE, "probe.cu")):
    subprocess.check_call(["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-o", SO, os.path.join(HERE, "probe.cu")])
if __name__ == "__main__":
    import torch
    lib = ctypes.CDLL(SO)
    lib.probe_ldg.restype = ctypes.c_float
    lib.probe_ldg.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int]
    lib.probe_tma.restype = ctypes.c_float
    lib.probe_tma.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                              ctypes.c_uint32, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    res = {}
    sizes = [int(x) << 20 for x in os.environ.get("PROBE_MIB", "256,4096").split(",")]
    for n in sizes:
        t = torch.empty(n, dtype=torch.uint8, device="cuda")
        t.fill_(1)
        p = t.data_ptr()
        for bps in (2, 4, 8):
            res[f"ldg n={n>>20}MiB bps={bps}"] = round(lib.probe_ldg(p, n, bps, 10), 1)
        for tile, stages, ctas, splits in [(32768, 3, 2, 1), (32768, 2, 3, 1), (32768, 3, 2, 4), (16384, 6, 2, 1),
                                          (16384, 4, 3, 1), (8192, 8, 3, 1), (65536, 3, 1, 1), (32768, 6, 1, 1),
                                          (16384, 12, 1, 1)]:
            res[f"tma n={n>>20}MiB tile={tile} st={stages} ctas={ctas} split={splits}"] = round(
                lib.probe_tma(p, n, tile, stages, ctas, splits, 8, 10, 0), 1)
            if splits == 1:  # tiles fetched from a counter (the search kernel's dispatch for long calls)
                res[f"tma-dyn n={n>>20}MiB tile={tile} st={stages} ctas={ctas}"] = round(
                    lib.probe_tma(p, n, tile, stages, ctas, 1, 8, 10, 1), 1)
        del t
        torch.cuda.empty_cache()
    for k, v in res.items():
        print(f"{k:60s} {v:8.1f} GB/s")
    key = "tma-dyn n=4096MiB tile=32768 st=2 ctas=3"
    if key not in res:
        sys.exit(0)
    out = {"source": "tools/probe.py on one B200 (gpurun), read-only streaming without compute, best of 10, CUDA events",
           "read_stream_GBps": res[key],
           "config_of_read_stream": "TMA 1-D bulk ring, 32 KiB tiles x 2 stages x 3 CTAs/SM, tiles fetched from a "
                                    "counter (the search kernel's configuration and dispatch), 4 GiB",
           "all": res}
    if len(sys.argv) > 1:
        json.dump(out, open(sys.argv[1], "w"), indent=1)
    print(json.dumps(out))
