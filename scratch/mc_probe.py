import ctypes, sys
from cuda.bindings import driver as cu
def ck(r):
    if isinstance(r, tuple):
        err, *rest = r
    else:
        err, rest = r, []
    if err != cu.CUresult.CUDA_SUCCESS:
        print("ERR", err); sys.exit(1)
    return rest[0] if len(rest) == 1 else rest
ck(cu.cuInit(0))
dev = ck(cu.cuDeviceGet(0))
print("multicast_supported", ck(cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)))
print("handle_types", ck(cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, dev)))
ctx = ck(cu.cuDevicePrimaryCtxRetain(dev)); ck(cu.cuCtxSetCurrent(ctx))

H = cu.CUmemAllocationHandleType
for nd in (1, 2):
  for ht in (H.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, H.CU_MEM_HANDLE_TYPE_NONE, H.CU_MEM_HANDLE_TYPE_FABRIC):
    for sz in (2 << 20, 512 << 20):
      p = cu.CUmulticastObjectProp()
      p.numDevices = nd; p.size = sz; p.handleTypes = ht; p.flags = 0
      r = cu.cuMulticastCreate(p)
      print(nd, ht, sz, r[0])
      if r[0] == cu.CUresult.CUDA_SUCCESS:
        print("  add", cu.cuMulticastAddDevice(r[1], dev)[0] if isinstance(cu.cuMulticastAddDevice(r[1], dev), tuple) else cu.cuMulticastAddDevice(r[1], dev))
import subprocess
print(subprocess.run("nvidia-smi -q | grep -i -A3 fabric; nvidia-smi topo -m | head -5", shell=True, capture_output=True, text=True).stdout)
