#!/usr/bin/env python
"""Probe NVLink SHARP (NVLS) multicast support on this box: device attribute,
torch symmetric-memory multicast pointer at world size 1, and a raw
cuMulticastCreate of one device (cuda-python).  Prints what works."""
import os
import sys

import torch
import torch.distributed as dist

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29555")
torch.cuda.set_device(0)
try:
    from cuda.bindings import driver as cu
except Exception:
    from cuda import cuda as cu  # older cuda-python
err, dev = cu.cuDeviceGet(0)
for name in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED"):
    a = getattr(cu.CUdevice_attribute, name, None)
    if a is not None:
        print(name, cu.cuDeviceGetAttribute(a, dev))
# raw multicast object of one device
HT = cu.CUmemAllocationHandleType
for ht in (HT.CU_MEM_HANDLE_TYPE_FABRIC, HT.CU_MEM_HANDLE_TYPE_NONE, HT.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR):
    prop = cu.CUmulticastObjectProp()
    prop.numDevices = 1
    prop.size = 2 << 20
    prop.handleTypes = ht
    r = cu.cuMulticastGetGranularity(prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
    r2 = cu.cuMulticastCreate(prop)
    print("handle type", ht, "granularity", r, "create", r2[0])
    if r2[0] == cu.CUresult.CUDA_SUCCESS:
        mc = r2[1]
        print("  add device", cu.cuMulticastAddDevice(mc, dev))
        # physical memory for the device, bind, map the multicast handle
        ap = cu.CUmemAllocationProp()
        ap.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        ap.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        ap.location.id = 0
        ap.requestedHandleTypes = ht
        e, mem = cu.cuMemCreate(2 << 20, ap, 0)
        print("  cuMemCreate", e)
        print("  bind", cu.cuMulticastBindMem(mc, 0, mem, 0, 2 << 20, 0))
        e, va = cu.cuMemAddressReserve(2 << 20, 2 << 20, 0, 0)
        print("  reserve", e, "map mc", cu.cuMemMap(va, 2 << 20, 0, mc, 0))
        acc = cu.CUmemAccessDesc()
        acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = 0
        acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        print("  set access", cu.cuMemSetAccess(va, 2 << 20, [acc], 1))
        break
# torch symmetric memory at world size 1
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import torch.distributed._symmetric_memory as symm_mem
g = dist.group.WORLD.group_name
if hasattr(symm_mem, "enable_symm_mem_for_group"):
    symm_mem.enable_symm_mem_for_group(g)
t = symm_mem.empty(1 << 20, dtype=torch.float32, device="cuda")
h = symm_mem.rendezvous(t, g)
print("symm_mem handle:", type(h).__name__, [a for a in dir(h) if "multicast" in a.lower()])
try:
    print("multicast_ptr", h.multicast_ptr)
except Exception as e:
    print("multicast_ptr error", e)
dist.destroy_process_group()
