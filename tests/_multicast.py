"""Test infrastructure: a one-device NVLink multicast object (CUDA driver
VMM API through cuda-python), so the CBP_ACC_MULTIMEM path -- the BP's
multimem.red.add into a multicast address -- runs on a single B200.  With
one member the switch "reduces" into the one bound buffer; several shards
issued one after another on the same GPU emulate several ranks adding into
it (no kernel waits on another)."""
from __future__ import annotations

from cuda.bindings import driver as drv


def _ok(res, what=""):
    err = res[0] if isinstance(res, tuple) else res
    if err != drv.CUresult.CUDA_SUCCESS:
        raise RuntimeError(f"CUDA driver call {what} failed: {err}")
    return res[1:] if isinstance(res, tuple) and len(res) > 2 else (res[1] if isinstance(res, tuple) and len(res) == 2 else None)


def _round(x, g):
    return (x + g - 1) // g * g


class Multicast:
    """`uc`: the local buffer's ordinary device address; `mc`: its multicast address."""

    def __init__(self, nbytes: int, device: int = 0, handle_type=None):
        _ok(drv.cuInit(0))
        dev = _ok(drv.cuDeviceGet(device))
        if not _ok(drv.cuDeviceGetAttribute(drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)):
            raise RuntimeError("multicast not supported")
        prop = drv.CUmulticastObjectProp()
        ht = (drv.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
              if handle_type is None else handle_type)
        prop.numDevices = 1
        prop.handleTypes = int(ht)
        prop.size = 2 << 20
        gran = _ok(drv.cuMulticastGetGranularity(
            prop, drv.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity")
        aprop = drv.CUmemAllocationProp()
        aprop.type = drv.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        aprop.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        aprop.location.id = device
        aprop.requestedHandleTypes = ht
        agran = _ok(drv.cuMemGetAllocationGranularity(
            aprop, drv.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED))
        self.size = _round(_round(nbytes, int(gran)), int(agran))
        prop.size = self.size
        self._mch = _ok(drv.cuMulticastCreate(prop), "cuMulticastCreate")
        _ok(drv.cuMulticastAddDevice(self._mch, dev), "cuMulticastAddDevice")
        self._mem = _ok(drv.cuMemCreate(self.size, aprop, 0), "cuMemCreate")
        _ok(drv.cuMulticastBindMem(self._mch, 0, self._mem, 0, self.size, 0), "cuMulticastBindMem")
        acc = drv.CUmemAccessDesc()
        acc.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = device
        acc.flags = drv.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        self.uc = int(_ok(drv.cuMemAddressReserve(self.size, int(agran), 0, 0), "reserve uc"))
        _ok(drv.cuMemMap(self.uc, self.size, 0, self._mem, 0), "map uc")
        _ok(drv.cuMemSetAccess(self.uc, self.size, [acc], 1), "access uc")
        self.mc = int(_ok(drv.cuMemAddressReserve(self.size, int(gran), 0, 0), "reserve mc"))
        _ok(drv.cuMemMap(self.mc, self.size, 0, self._mch, 0), "map mc")
        _ok(drv.cuMemSetAccess(self.mc, self.size, [acc], 1), "access mc")

    def zero(self):
        _ok(drv.cuMemsetD32(self.uc, 0, self.size // 4))

    def read_into(self, t):
        """copy the local buffer into the CUDA tensor t (synchronous)"""
        _ok(drv.cuCtxSynchronize())
        _ok(drv.cuMemcpy(t.data_ptr(), self.uc, t.numel() * t.element_size()))
        _ok(drv.cuCtxSynchronize())

    def close(self):
        for va in (self.mc, self.uc):
            drv.cuMemUnmap(va, self.size)
            drv.cuMemAddressFree(va, self.size)
        drv.cuMulticastUnbind(self._mch, drv.CUdevice(0), 0, self.size)
        drv.cuMemRelease(self._mem)
        drv.cuMemRelease(self._mch)
