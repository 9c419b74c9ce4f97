"""Probe variants of cuMulticastCreate on one device (handle types, sizes)."""
import json
import torch
from cuda.bindings import driver as cu

torch.zeros(1, device="cuda")
err, dev = cu.cuDeviceGet(0)
H = cu.CUmemAllocationHandleType
res = []
for ht_name in ["CU_MEM_HANDLE_TYPE_NONE", "CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR", "CU_MEM_HANDLE_TYPE_FABRIC"]:
    for size in [2 << 20, 32 << 20, 512 << 20]:
        for n in [1, 2]:
            prop = cu.CUmulticastObjectProp()
            prop.numDevices = n
            prop.size = size
            prop.flags = 0
            prop.handleTypes = getattr(H, ht_name)
            err, mc = cu.cuMulticastCreate(prop)
            r = {"ht": ht_name, "size": size, "n": n, "create": str(err)}
            if err == cu.CUresult.CUDA_SUCCESS:
                e2 = cu.cuMulticastAddDevice(mc, dev)
                r["add"] = str(e2[0] if isinstance(e2, tuple) else e2)
                cu.cuMemRelease(mc)
            res.append(r)
print(json.dumps(res, indent=0))
