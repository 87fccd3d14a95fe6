from cuda.bindings import driver as cu
import torch
torch.cuda.init(); torch.empty(1, device="cuda")
cu.cuInit(0)
err, dev = cu.cuDeviceGet(0)
HT = cu.CUmemAllocationHandleType
for nd in (1, 2):
    for ht in (0, int(HT.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR), int(HT.CU_MEM_HANDLE_TYPE_FABRIC)):
        prop = cu.CUmulticastObjectProp()
        prop.numDevices = nd
        prop.handleTypes = ht
        prop.size = 2 << 20
        prop.flags = 0
        e1, g = cu.cuMulticastGetGranularity(prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        e2, mc = cu.cuMulticastCreate(prop)
        print("numDevices", nd, "handleTypes", ht, "gran", e1, g, "create", e2)
