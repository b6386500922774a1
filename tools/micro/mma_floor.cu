// tcgen05.mma (kind::f16, M = 128, K = 16, cta_group::1) issue floor with loop-invariant descriptors:
// 4 MMAs per iteration at k offsets 0..3 (one 64-deep k-block of a 128B-swizzled K-major tile),
// one accumulator; A and B from shared memory (SS). cycles per MMA vs N.
#include <cstdio>
#include "../../paper_2511_20340_b200/csrc/common.cuh"
using namespace sf;

template <int N>
__global__ void floor_k(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 1) {
    constexpr uint32_t idesc = idesc_bf16_f32(128, N);
    const uint64_t da = sw128_kmajor_desc(smem_u32(base));
    const uint64_t db = sw128_kmajor_desc(smem_u32(base + 16384));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) umma_bf16(tmem, da + kk * 2, db + kk * 2, idesc, (i | kk) ? 1u : 0u);
      }
      __syncwarp();
    }
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    if ((threadIdx.x & 31) == 0) out[0] = clock64() - t0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int N>
void run(long long* d) {
  cudaFuncSetAttribute(floor_k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 2048;
  floor_k<N><<<1, 128, 90 * 1024>>>(iters, d);
  long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("N=%3d: %6.1f cycles/MMA  floor %5.1f  (%s)\n", N, (double)c / (4 * iters), 128.0 * N / 256,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  long long* d; cudaMalloc(&d, 8);
  run<16>(d); run<32>(d); run<64>(d); run<128>(d); run<160>(d); run<256>(d);
  return 0;
}
