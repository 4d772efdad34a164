"""Probe: can this box create an NVLS multicast object (cuMulticastCreate) for its GPU(s)?
Prints the device attributes and cuMulticastCreate / AddDevice results for a few property sets."""
from cuda.bindings import driver as d
import torch

torch.zeros(1, device="cuda")
_, dev = d.cuDeviceGet(0)
for a in ["CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED",
          "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED"]:
    print(a, d.cuDeviceGetAttribute(getattr(d.CUdevice_attribute, a), dev))
HT = d.CUmemAllocationHandleType
for nd in (1, 2):
    for ht in (HT.CU_MEM_HANDLE_TYPE_NONE, HT.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, HT.CU_MEM_HANDLE_TYPE_FABRIC):
        for size in (2 << 20, 64 << 20):
            prop = d.CUmulticastObjectProp()
            prop.numDevices = nd
            prop.size = size
            prop.handleTypes = ht
            prop.flags = 0
            r = d.cuMulticastCreate(prop)
            msg = f"nd={nd} ht={ht.name} size={size >> 20}MB create={r[0].name}"
            if r[0] == d.CUresult.CUDA_SUCCESS:
                msg += f" add={d.cuMulticastAddDevice(r[1], dev)[0].name}"
            print(msg, flush=True)
