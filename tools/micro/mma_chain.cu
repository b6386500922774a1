// Is back-to-back tcgen05.mma into ONE accumulator latency-bound at small N? cycles per MMA
// (kind::f16, M = 128, K = 16, SS operands, cta_group::1) issued by one thread, cycling over C
// independent accumulators (columns c * N), no commits inside the loop.
#include <cstdio>
#include "../../paper_2511_20340_b200/csrc/common.cuh"
using namespace sf;

__global__ void chain(int N, int C, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 32) {
    const uint32_t idesc = idesc_bf16_f32(128, N);
    const uint64_t da = sw128_kmajor_desc(smem_u32(base));
    const uint64_t db = sw128_kmajor_desc(smem_u32(base + 16384));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int c = i % C;
      umma_bf16(tmem + (uint32_t)(c * N), da + ((i / C) & 3) * 2, db + ((i / C) & 3) * 2, idesc, i >= C);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    out[0] = clock64() - t0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(chain, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int N : {16, 64, 128, 160, 256}) for (int C : {1, 2, 3, 4}) {
    if (N * C > 512) continue;
    const int iters = 4096;
    chain<<<1, 128, 90 * 1024>>>(N, C, iters, d);
    long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("N=%3d C=%d: %6.1f cycles/MMA  floor %5.1f  (%s)\n", N, C, (double)c / iters, 128.0 * N / 256,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
