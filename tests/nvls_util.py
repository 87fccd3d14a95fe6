"""Test helper: a u64 buffer with an NVLink multicast mapping on ONE device, built with the
CUDA driver API (cuMulticastCreate / cuMulticastBindMem, no handle export), so that the
NVLS count epilogue (multimem.red, NEXT-4) can be exercised on a single-GPU box.  Multi-rank
runs get the same kind of address from torch symmetric memory (dist.py)."""


def _check(res):
    err = res[0] if isinstance(res, tuple) else res
    if int(err) != 0:
        raise RuntimeError(f"CUDA driver error {err}")
    return res[1] if isinstance(res, tuple) and len(res) == 2 else (res[1:] if isinstance(res, tuple) else None)


class MulticastU64:
    def __init__(self, n: int, device: int = 0):
        from cuda.bindings import driver as cu
        import torch
        torch.cuda.init()
        torch.cuda.set_device(device)
        torch.empty(1, device="cuda")  # make the primary context current on this thread
        self.cu = cu
        _check(cu.cuInit(0))
        dev = _check(cu.cuDeviceGet(device))
        ok = _check(cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev))
        if not ok:
            raise RuntimeError("multicast not supported")
        prop = cu.CUmulticastObjectProp()
        prop.numDevices = 1
        prop.handleTypes = 0
        prop.size = max(8 * n, 8)
        gran = _check(cu.cuMulticastGetGranularity(
            prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
        size = ((prop.size + gran - 1) // gran) * gran
        prop.size = size
        self.size = size
        self.mc = _check(cu.cuMulticastCreate(prop))
        _check(cu.cuMulticastAddDevice(self.mc, dev))
        pprop = cu.CUmemAllocationProp()
        pprop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        pprop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        pprop.location.id = device
        self.mem = _check(cu.cuMemCreate(size, pprop, 0))
        _check(cu.cuMulticastBindMem(self.mc, 0, self.mem, 0, size, 0))
        acc = cu.CUmemAccessDesc()
        acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = device
        acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        self.uva = _check(cu.cuMemAddressReserve(size, 0, 0, 0))
        _check(cu.cuMemMap(self.uva, size, 0, self.mem, 0))
        _check(cu.cuMemSetAccess(self.uva, size, [acc], 1))
        self.mva = _check(cu.cuMemAddressReserve(size, 0, 0, 0))
        _check(cu.cuMemMap(self.mva, size, 0, self.mc, 0))
        _check(cu.cuMemSetAccess(self.mva, size, [acc], 1))
        self.n = n

    @property
    def unicast_ptr(self) -> int:
        return int(self.uva)

    @property
    def multicast_ptr(self) -> int:
        return int(self.mva)

    def zero(self):
        _check(self.cu.cuMemsetD8(self.uva, 0, self.size))

    def read(self):
        import numpy as np
        out = np.zeros(self.n, dtype=np.uint64)
        _check(self.cu.cuCtxSynchronize())
        _check(self.cu.cuMemcpyDtoH(out.ctypes.data, self.uva, 8 * self.n))
        return out
