#!/usr/bin/env python
"""TMA staging-ring read probe: static round-robin tiles vs counter-dispatched tiles."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import probe  # builds tools/libprobe.so
if __name__ == "__main__":
    import torch
    lib = ctypes.CDLL(probe.SO)
    lib.probe_tma.restype = ctypes.c_float
    lib.probe_tma.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                              ctypes.c_uint32, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    for n in (1 << 28, 1 << 32):
        t = torch.empty(n, dtype=torch.uint8, device="cuda")
        t.fill_(1)
        for tile, stages, ctas in ((32768, 2, 3), (32768, 3, 2), (16384, 4, 3)):
            for dyn in (0, 1):
                print(f"n={n >> 20} MiB tile={tile} stages={stages} ctas={ctas} {'dynamic' if dyn else 'static '}: "
                      f"{lib.probe_tma(t.data_ptr(), n, tile, stages, ctas, 1, 8, 10, dyn):8.1f} GB/s")
        del t
        torch.cuda.empty_cache()
