#include <cuda.h>
#include <stdio.h>
int main(){
  CUdevice d; CUcontext c; cuInit(0); cuDeviceGet(&d,0); cuDevicePrimaryCtxRetain(&c,d); cuCtxSetCurrent(c);
  int v=0; cuDeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d); printf("mc_supported %d\n", v);
  int drv; cuDriverGetVersion(&drv); printf("driver %d\n", drv);
  CUmulticastObjectProp p = {0}; p.numDevices=1; p.size=2<<20; p.handleTypes=CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g=0; CUresult r = cuMulticastGetGranularity(&g,&p,CU_MULTICAST_GRANULARITY_RECOMMENDED); printf("gran %d %zu\n", r, g);
  CUmemGenericAllocationHandle mc; r = cuMulticastCreate(&mc,&p); const char* s; cuGetErrorString(r,&s); printf("create %d %s\n", r, s);
  if (r) return 1;
  r = cuMulticastAddDevice(mc,d); printf("add %d\n", r);
  CUmemAllocationProp ap = {0}; ap.type=CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type=CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id=0; ap.requestedHandleTypes=CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle ph; r = cuMemCreate(&ph, 2<<20, &ap, 0); printf("memcreate %d\n", r);
  r = cuMulticastBindMem(mc, 0, ph, 0, 2<<20, 0); printf("bind %d\n", r);
  CUdeviceptr va; cuMemAddressReserve(&va, 2<<20, 2<<20, 0, 0); r = cuMemMap(va, 2<<20, 0, mc, 0); printf("map mc %d\n", r);
  CUmemAccessDesc ad = {{CU_MEM_LOCATION_TYPE_DEVICE, 0}, CU_MEM_ACCESS_FLAGS_PROT_READWRITE}; r = cuMemSetAccess(va, 2<<20, &ad, 1); printf("access %d\n", r);
  return 0;
}
