// Microbenchmark: issue rate / latency of tcgen05.mma kind::f16 (M=128) for various N, with and
// without a commit + wait per group, from one thread. Prints cycles per MMA.
#include <cstdio>
#include "../../paper_2511_20340_b200/csrc/common.cuh"
using namespace sf;

__global__ void mma_rate(int N, int iters, int group, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint64_t bars[8];
  __shared__ uint32_t slot;
  uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); for (int j = 0; j < 8; ++j) mbar_init(&bars[j], 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 32) {
    const uint32_t idesc = idesc_bf16_f32(128, N);
    const uint64_t da = sw128_kmajor_desc(smem_u32(base));
    const uint64_t db = sw128_kmajor_desc(smem_u32(base + 16384));
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      umma_bf16(tmem, da + (i & 3) * 2, db + (i & 3) * 2, idesc, i > 0);
      if (group > 0 && (i % group) == group - 1) {
        umma_commit(&bar);
        mbar_wait(&bar, ph); ph ^= 1;
      } else if (group < 0 && (i % (-group)) == (-group) - 1) {
        umma_commit(&bars[(i / (-group)) % 8]);  // commit without waiting (8 rotating barriers)
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, ph);
    long long t1 = clock64();
    out[0] = t1 - t0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int Ns[] = {16, 32, 64, 128, 256};
  const int groups[] = {0, -4, -1, 4};
  for (int g : groups) for (int N : Ns) {
    const int iters = 4096;
    mma_rate<<<1, 128, 90 * 1024>>>(N, iters, g, d);
    long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    printf("group=%d N=%3d: %.1f cycles/MMA (%s)\n", g, N, (double)c / iters, cudaGetErrorString(e));
  }
  return 0;
}
