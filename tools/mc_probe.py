from cuda.bindings import driver as d
import torch
torch.cuda.init(); torch.zeros(1, device="cuda")
err, dev = d.cuDeviceGet(0)
for a in ["CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED", "CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED"]:
    print(a, d.cuDeviceGetAttribute(getattr(d.CUdevice_attribute, a), dev))
prop = d.CUmulticastObjectProp()
prop.numDevices = 1
prop.size = 2 << 20
prop.handleTypes = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
print("gran", d.cuMulticastGetGranularity(prop, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
r = d.cuMulticastCreate(prop); print("create", r)
if r[0] == d.CUresult.CUDA_SUCCESS:
    print("add", d.cuMulticastAddDevice(r[1], dev))
