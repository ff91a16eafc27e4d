// NVLS multicast feasibility probe: cuMulticastCreate / AddDevice / BindMem / Map on this GPU, then
// multimem.st and multimem.ld_reduce through the multicast address.  nvcc -gencode arch=compute_100a,code=sm_100a
// -o mc_probe mc_probe.cu -lcuda.  Result on the r02 1-GPU lease: profiles/r02/multicast_probe.txt.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("%s -> %d %s\n", #x, (int)r, s); return 1; } } while (0)
__global__ void st_kernel(float* mc, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i * 4 < n) {
    float a = i, b = i + 0.5f, c = -i, d = 2 * i;
    asm volatile("multimem.st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + 4 * i), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
  }
}
__global__ void ldred_kernel(const float* mc, float* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i * 4 < n) {
    float a, b, c, d;
    asm volatile("multimem.ld_reduce.global.add.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(mc + 4 * i) : "memory");
    out[4 * i] = a; out[4 * i + 1] = b; out[4 * i + 2] = c; out[4 * i + 3] = d;
  }
}
int main() {
  CK(cuInit(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));
  int mcs = 0; cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  printf("multicast supported %d\n", mcs);
  const size_t n = 1 << 20; size_t bytes = n * 4;
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1; mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR; mp.size = bytes;
  size_t gran = 0; CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  bytes = (bytes + gran - 1) / gran * gran; mp.size = bytes;
  printf("min granularity %zu bytes %zu\n", gran, bytes);
  CUmemGenericAllocationHandle mc;
  CUresult r0 = cuMulticastCreate(&mc, &mp);
  printf("create posix fd: %d\n", (int)r0);
  if (r0 != CUDA_SUCCESS) { mp.handleTypes = CU_MEM_HANDLE_TYPE_NONE; r0 = cuMulticastCreate(&mc, &mp); printf("create none: %d\n", (int)r0); }
  if (r0 != CUDA_SUCCESS) { mp.handleTypes = CU_MEM_HANDLE_TYPE_FABRIC; r0 = cuMulticastCreate(&mc, &mp); printf("create fabric: %d\n", (int)r0); }
  if (r0 != CUDA_SUCCESS) return 1;
  CK(cuMulticastAddDevice(mc, dev));
  CUmemAllocationProp ap = {}; ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = dev;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g2 = 0; CK(cuMemGetAllocationGranularity(&g2, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  printf("mem granularity %zu\n", g2);
  CUmemGenericAllocationHandle phys; CK(cuMemCreate(&phys, bytes, &ap, 0));
  CK(cuMulticastBindMem(mc, 0, phys, 0, bytes, 0));
  CUdeviceptr uc, mcp;
  CK(cuMemAddressReserve(&uc, bytes, gran, 0, 0)); CK(cuMemMap(uc, bytes, 0, phys, 0));
  CK(cuMemAddressReserve(&mcp, bytes, gran, 0, 0)); CK(cuMemMap(mcp, bytes, 0, mc, 0));
  CUmemAccessDesc acc = {}; acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE; acc.location.id = dev; acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc, bytes, &acc, 1)); CK(cuMemSetAccess(mcp, bytes, &acc, 1));
  st_kernel<<<(n / 4 + 255) / 256, 256>>>((float*)mcp, n);
  printf("st launch %s sync %s\n", cudaGetErrorString(cudaGetLastError()), cudaGetErrorString(cudaDeviceSynchronize()));
  float* out; cudaMalloc(&out, n * 4);
  ldred_kernel<<<(n / 4 + 255) / 256, 256>>>((const float*)mcp, out, n);
  printf("ldred launch %s sync %s\n", cudaGetErrorString(cudaGetLastError()), cudaGetErrorString(cudaDeviceSynchronize()));
  float h[8], hu[8];
  cudaMemcpy(h, out + 40, 32, cudaMemcpyDeviceToHost);
  cudaMemcpy(hu, (float*)uc + 40, 32, cudaMemcpyDeviceToHost);
  printf("ldred %g %g %g %g | unicast %g %g %g %g\n", h[0], h[1], h[2], h[3], hu[0], hu[1], hu[2], hu[3]);
  int fd = -1; CUresult r = cuMemExportToShareableHandle(&fd, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
  printf("export multicast fd rc %d fd %d\n", (int)r, fd);
  return 0;
}
