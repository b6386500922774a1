// Probe: a 1-device NVLS multicast object on this B200 -- create, bind, map, then multimem.ld_reduce /
// multimem.st / multimem.red from a kernel. nvcc -gencode arch=compute_100a,code=sm_100a nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s; cuGetErrorString(r_, &s); printf("%s -> %s\n", #x, s); return 1; } } while (0)
__global__ void k(float* mc, float* uc, float* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(mc + i) : "memory");
  out[i] = v;
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(mc + n + i), "f"(2.f * v) : "memory");
}
int main() {
  CK(cuInit(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));
  int mcs = 0; CK(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  printf("multicast supported: %d\n", mcs);
  const int n = 1 << 20;
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1;
  mp.handleTypes = (CUmemAllocationHandleType)(getenv("HT") ? atoi(getenv("HT")) : 0);
  size_t gran = 0;
  mp.size = 2 * n * sizeof(float);
  CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  mp.size = (mp.size + gran - 1) / gran * gran;
  printf("granularity %zu size %zu\n", gran, mp.size);
  CUmemGenericAllocationHandle mc; CK(cuMulticastCreate(&mc, &mp));
  CK(cuMulticastAddDevice(mc, dev));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = 0;
  ap.requestedHandleTypes = (CUmemAllocationHandleType)mp.handleTypes;
  CUmemGenericAllocationHandle mem; CK(cuMemCreate(&mem, mp.size, &ap, 0));
  CK(cuMulticastBindMem(mc, 0, mem, 0, mp.size, 0));
  CUdeviceptr uc, mcp;
  CK(cuMemAddressReserve(&uc, mp.size, gran, 0, 0)); CK(cuMemMap(uc, mp.size, 0, mem, 0));
  CK(cuMemAddressReserve(&mcp, mp.size, gran, 0, 0)); CK(cuMemMap(mcp, mp.size, 0, mc, 0));
  CUmemAccessDesc ad = {}; ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ad.location.id = 0; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc, mp.size, &ad, 1)); CK(cuMemSetAccess(mcp, mp.size, &ad, 1));
  float* h = new float[n]; for (int i = 0; i < n; ++i) h[i] = 0.5f * i;
  cudaMemcpy((void*)uc, h, n * 4, cudaMemcpyHostToDevice);
  float* out; cudaMalloc(&out, n * 4);
  k<<<n / 256, 256>>>((float*)mcp, (float*)uc, out, n);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  float* r = new float[n]; cudaMemcpy(r, out, n * 4, cudaMemcpyDeviceToHost);
  float* r2 = new float[n]; cudaMemcpy(r2, (float*)uc + n, n * 4, cudaMemcpyDeviceToHost);
  int bad = 0; for (int i = 0; i < n; ++i) bad += (r[i] != h[i]) + (r2[i] != 2.f * h[i]);
  printf("mismatches: %d (of %d)\n", bad, 2 * n);
  return 0;
}
