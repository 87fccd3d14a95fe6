#!/usr/bin/env python
"""Probe: does this box support multicast (NVLS) through torch symmetric memory with one rank?"""
import os
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
import torch
import torch.distributed as dist
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
print("torch", torch.__version__)
try:
    from cuda.bindings import driver as cu
except Exception:
    try:
        from cuda import cuda as cu
    except Exception as e:
        cu = None
        print("no cuda-python driver bindings:", e)
if cu is not None:
    cu.cuInit(0)
    err, d = cu.cuDeviceGet(0)
    for name in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED"):
        attr = getattr(cu.CUdevice_attribute, name, None)
        if attr is not None:
            print(name, cu.cuDeviceGetAttribute(attr, d))
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
try:
    import torch.distributed._symmetric_memory as symm_mem
    t = symm_mem.empty(64, dtype=torch.int64, device=dev)
    h = symm_mem.rendezvous(t, dist.group.WORLD)
    print("symm mem ok; multicast_ptr =", getattr(h, "multicast_ptr", None), "buffer ptrs", getattr(h, "buffer_ptrs", None))
except Exception as e:
    print("symmetric memory failed:", type(e).__name__, e)
dist.destroy_process_group()
