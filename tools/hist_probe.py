#!/usr/bin/env python
"""A1 byte-histogram variants (tools/hist_probe.cu) on the configs' texts: GB/s and exactness vs torch.bincount."""
import ctypes, os, subprocess, sys
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
SO = os.path.join(HERE, "libhistprobe.so")
if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(os.path.join(HERE, "hist_probe.cu")):
    subprocess.check_call(["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-o", SO, os.path.join(HERE, "hist_probe.cu")])
if __name__ == "__main__":
    import torch
    import paper_1612_01506_b200 as sm
    import synth
    lib = ctypes.CDLL(SO)
    lib.hist_probe.restype = ctypes.c_float
    lib.hist_probe.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
    names = ["W8 R1 U2", "W8 R2 U2", "W8 R4 U2", "W8 R8 U2", "W8 R1 U4 (library)", "W8 R4 U4", "W4 R8 U4", "W16 R2 U2",
             "W4 R4 U4", "lane-private W1 U8", "lane-private W1 U16", "lane-private W2 U8", "lane-private W2 U16",
             "lane-private W4 U4", "lane-private W4 U8"]
    only = [int(x) for x in os.environ.get("HIST_VARIANTS", "").split(",") if x]
    d = torch.zeros(256, dtype=torch.int64, device="cuda")
    for cfg, n in (("c2", 256 << 20), ("c3", 1 << 30), ("c5", 1 << 30), ("c4p", 1 << 30), ("c1", 1 << 20)):
        spec = synth.text_spec(cfg, n=n)
        t = synth.gen_text_device(spec, 0, n)
        want = torch.bincount(t.to(torch.int64), minlength=256)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(5):
            e0.record(); h = sm.sm_histogram(t); e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"{cfg} n={n}: library sm_histogram {n / best / 1e6:8.1f} GB/s (incl. memset)")
        for bps in [int(x) for x in os.environ.get("HIST_BPS", "2,3,4").split(",")]:
            for v, nm in enumerate(names):
                if only and v not in only:
                    continue
                g = lib.hist_probe(v, t.data_ptr(), n, d.data_ptr(), bps, 5)
                ok = torch.equal(d, want) if g > 0 else False
                print(f"  {nm:20s} blocks/SM {bps}: {g:8.1f} GB/s {'ok' if ok else 'MISMATCH'}")
        del t
        torch.cuda.empty_cache()
