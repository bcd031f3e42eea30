"""Probe: which multicast object properties does cuMulticastCreate accept on this box?"""
import torch
torch.zeros(1, device="cuda")
from cuda.bindings import driver as drv
drv.cuInit(0)
err, dev = drv.cuDeviceGet(0)
for a in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
          "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED",
          "CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED"):
    print(a, drv.cuDeviceGetAttribute(getattr(drv.CUdevice_attribute, a), dev))
for nd in (1, 2):
    for ht in (0, 1, 8):
        prop = drv.CUmulticastObjectProp()
        prop.numDevices = nd
        prop.handleTypes = ht
        prop.flags = 0
        prop.size = 2 << 20
        e1, gmin = drv.cuMulticastGetGranularity(prop, drv.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM)
        e2, grec = drv.cuMulticastGetGranularity(prop, drv.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        for size in (gmin, grec, 1 << 30):
            if not size:
                continue
            prop.size = size
            e, mc = drv.cuMulticastCreate(prop)
            print("nd", nd, "ht", ht, "gran", e1, gmin, e2, grec, "size", size, "->", e)
            if e == drv.CUresult.CUDA_SUCCESS:
                drv.cuMemRelease(mc)
