"""Does this box support CUDA multicast objects (NVLS through NVSwitch)?"""
from cuda import cuda
import torch
torch.cuda.init()
cuda.cuInit(0)
for d in range(torch.cuda.device_count()):
    err, dev = cuda.cuDeviceGet(d)
    for a in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
              "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"):
        if hasattr(cuda.CUdevice_attribute, a):
            print(d, a, cuda.cuDeviceGetAttribute(getattr(cuda.CUdevice_attribute, a), dev))
prop = cuda.CUmulticastObjectProp()
prop.numDevices = max(1, torch.cuda.device_count())
prop.handleTypes = cuda.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
prop.size = 2 << 20
print("granularity", cuda.cuMulticastGetGranularity(prop, cuda.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
err, h = cuda.cuMulticastCreate(prop)
print("create", err)
