#!/usr/bin/env python
"""Write-bandwidth probe: per-warp sequential regions of various sizes vs grid-stride (8 GiB)."""
import ctypes, os, subprocess
HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libwprobe.so")
if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(os.path.join(HERE, "wprobe.cu")):
    subprocess.check_call(["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-o", SO, os.path.join(HERE, "wprobe.cu")])
if __name__ == "__main__":
    import torch
    lib = ctypes.CDLL(SO)
    lib.wprobe.restype = ctypes.c_float
    lib.wprobe.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    n = 8 << 30
    t = torch.empty(n, dtype=torch.uint8, device="cuda")
    lib.wprobe32.restype = ctypes.c_float
    lib.wprobe32.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    for konst in (0, 1):
        for bps, thr in ((2, 256), (4, 256), (8, 256)):
            print(f"warps/SM {bps * thr // 32:3d} 32-B stores grid-stride, {'constant' if konst else 'distinct'} "
                  f"values: {lib.wprobe32(t.data_ptr(), n, bps, thr, 5, konst):8.1f} GB/s")
    lib.wprobe_once.restype = ctypes.c_float
    lib.wprobe_once.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    for konst in (0, 1):
        for thr, per in ((128, 1), (128, 4), (256, 4), (512, 8), (1024, 16)):
            print(f"one-shot blocks of {thr} threads x {per} 16-B stores, {'constant' if konst else 'distinct'}: "
                  f"{lib.wprobe_once(t.data_ptr(), n, thr, per, konst, 5):8.1f} GB/s")
    lib.wprobe_cta.restype = ctypes.c_float
    lib.wprobe_cta.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    for bps, thr in ((2, 256), (4, 256), (8, 128), (1, 1024)):
        for per in (1, 4, 8):
            print(f"persistent CTA chunks, {bps * thr // 32} warps/SM, {per} stores per thread: "
                  f"{lib.wprobe_cta(t.data_ptr(), n, bps, thr, per, 5):8.1f} GB/s")
    lib.wprobe_dyn.restype = ctypes.c_float
    lib.wprobe_dyn.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    for bps, thr in ((2, 256), (1, 256), (4, 256)):
        for region in (2 << 10, 8 << 10, 32 << 10, 480 << 10):
            print(f"dynamic warp regions, {bps * thr // 32} warps/SM, {region >> 10} KiB: "
                  f"{lib.wprobe_dyn(t.data_ptr(), n, region, bps, thr, 5):8.1f} GB/s")
    x = t.view(torch.int64)
    for name, fn in (("fill_(7)", lambda: x.fill_(7)), ("arange", lambda: torch.arange(x.numel(), out=x)),
                     ("copy_ of a 4 GiB half", lambda: x[: x.numel() // 2].copy_(x[x.numel() // 2:]))):
        fn(); torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"{name}: {best:.3f} ms = {n / best / 1e6:.1f} GB/s (8 GiB; copy: read+write)")
    for bps, thr in ((2, 256), (1, 256), (4, 256)):
        for region in (0, 32 << 10, 512 << 10):
            print(f"warps/SM {bps * thr // 32:3d} region {region >> 10:6d} KiB: "
                  f"{lib.wprobe(t.data_ptr(), n, region, bps, thr, 5):8.1f} GB/s")
