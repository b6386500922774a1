// Which per-k-block operation stalls the tcgen05 pipe? cycles per MMA (M=128, N=16) for:
//  0 plain; 1 fence::after_thread_sync every 4; 2 try_wait(completed barrier) every 4;
//  3 both; 4 commit(no wait) every 16; 5 commit every 4 + fence every 4
#include <cstdio>
#include "../../paper_2511_20340_b200/csrc/common.cuh"
using namespace sf;

__global__ void k(int mode, int N, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t done_bar, bars[8];
  __shared__ uint32_t slot;
  uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&done_bar, 1);
    for (int j = 0; j < 8; ++j) mbar_init(&bars[j], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x == 0) mbar_arrive(&bars[0]);  // complete phase 0 of bars[0]
  __syncthreads();
  const uint32_t tmem = slot;
  if (threadIdx.x == 32 && (blockIdx.x == 0 || mode >= 0)) {
    const uint32_t idesc = idesc_bf16_f32(128, N);
    const uint64_t da = sw128_kmajor_desc(smem_u32(base));
    const uint64_t db = sw128_kmajor_desc(smem_u32(base + 6 * 16384));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if ((i & 3) == 0) {
        if (mode == 1 || mode == 3 || mode == 5) tc_fence_after();
        if (mode == 2 || mode == 3) mbar_wait(&bars[0], 0);
      }
      const int tile = (mode >= 10) ? ((i >> 2) % 6) : 0;  // rotate through 6 distinct 16 KB A tiles
      umma_bf16(tmem, da + (i & 3) * 2 + tile * 1024, db + (i & 3) * 2, idesc, i > 0);
      if (mode == 4 && (i & 15) == 15) umma_commit(&bars[1 + ((i >> 4) % 7)]);
      if (mode == 5 && (i & 3) == 3) umma_commit(&bars[1 + ((i >> 2) % 7)]);
    }
    umma_commit(&done_bar);
    mbar_wait(&done_bar, 0);
    if (blockIdx.x == 0) out[0] = clock64() - t0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  for (int grid : {1}) for (int N : {16, 160, 256}) for (int mode : {0, 10}) {
    const int iters = 8192;
    k<<<grid, 128, 200 * 1024>>>(mode, N, iters, d);
    long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("grid %3d N %3d mode %d: %.1f cycles/MMA (%s)\n", grid, N, mode, (double)c / iters, cudaGetErrorString(cudaGetLastError()));
  }
}
