"""Probe: does this box support NVLS multicast objects (cuMulticastCreate)?
Prints the device attribute, the granularity, and whether a 1-device
multicast object can be created, bound and mapped."""
import json
import torch
from cuda.bindings import driver as cu

torch.cuda.init()
torch.zeros(1, device="cuda")
out = {}
err, dev = cu.cuDeviceGet(0)
err, v = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
out["multicast_supported"] = (str(err), v)
try:
    err, v = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev)
    out["fabric_handle_supported"] = (str(err), v)
except Exception as e:
    out["fabric_handle_supported"] = repr(e)
prop = cu.CUmulticastObjectProp()
prop.numDevices = 1
prop.size = 2 << 20
prop.handleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
err, gran = cu.cuMulticastGetGranularity(prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
out["granularity"] = (str(err), gran)
err, mc = cu.cuMulticastCreate(prop)
out["create"] = str(err)
if err == cu.CUresult.CUDA_SUCCESS:
    err = cu.cuMulticastAddDevice(mc, dev)
    out["add_device"] = str(err[0] if isinstance(err, tuple) else err)
print(json.dumps(out, default=str))
