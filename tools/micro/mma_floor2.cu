// Which per-k-block operation of the GEMM's MMA loop costs tensor-pipe time? cycles per k-block
// (4 MMAs, M = 128, N = NN, cta_group::1, loop-invariant operands unless noted) when adding:
//  bit0: mbar_wait on an already-completed barrier;  bit1: tcgen05.fence::after_thread_sync;
//  bit2: tcgen05.commit every 2 k-blocks (8 rotating barriers, never waited);
//  bit3: descriptors from a runtime ring slot (s = i % stages, runtime stage bytes)
#include <cstdio>
#include "../../paper_2511_20340_b200/csrc/common.cuh"
using namespace sf;

template <int NN>
__global__ void k(int mode, int stages, int stage_bytes, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar, done, bars[8];
  __shared__ uint32_t slot;
  uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1); mbar_init(&done, 1);
    for (int j = 0; j < 8; ++j) mbar_init(&bars[j], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x == 0) mbar_arrive(&bar);  // phase 0 completes
  __syncthreads();
  const uint32_t tmem = slot;
  if (warp == 1) {
    constexpr uint32_t idesc = idesc_bf16_f32(128, NN);
    const uint64_t da0 = sw128_kmajor_desc(smem_u32(base));
    const uint64_t db0 = sw128_kmajor_desc(smem_u32(base + 16384));
    int s = 0, g = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (mode & 1) mbar_wait(&bar, 0);
      if (mode & 2) tc_fence_after();
      if (elect_one()) {
        uint64_t da = da0, db = db0;
        if (mode & 8) {
          da = sw128_kmajor_desc(smem_u32(base + (size_t)s * stage_bytes));
          db = da + (16384 >> 4);
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) umma_bf16(tmem, da + kk * 2, db + kk * 2, idesc, (i | kk) ? 1u : 0u);
        if ((mode & 4) && (i & 1)) umma_commit(&bars[(g++) & 7]);
      }
      __syncwarp();
      if (++s == stages) s = 0;
    }
    if (elect_one()) umma_commit(&done);
    __syncwarp();
    mbar_wait(&done, 0);
    if ((threadIdx.x & 31) == 0) out[0] = clock64() - t0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int NN>
void run(long long* d) {
  cudaFuncSetAttribute(k<NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int mode : {0, 1, 2, 4, 8, 3, 7, 15}) {
    const int iters = 2048;
    k<NN><<<1, 128, 200 * 1024>>>(mode, 6, 32768, iters, d);
    long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("N=%3d mode %2d: %6.1f cycles/k-block (floor %5.1f) (%s)\n", NN, mode, (double)c / iters, 4 * 128.0 * NN / 256,
           cudaGetErrorString(cudaGetLastError()));
  }
}
int main() {
  long long* d; cudaMalloc(&d, 8);
  run<16>(d); run<160>(d); run<256>(d);
  return 0;
}
