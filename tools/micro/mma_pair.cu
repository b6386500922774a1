// CTA-pair (cta_group::2, M = 256) MMA loop rate, cycles per 64-deep k-block (4 MMAs, N = NN):
//  mode 0: back-to-back, loop-invariant operands
//  mode 1: + commit (multicast to both CTAs) every 2 k-blocks, never waited
//  mode 2: ring emulation as in gemm_sk_kernel with no loads (SF_GEMM_PROBE): a producer warp
//          waits empty[group], arrives full[s]; the MMA warp waits full[s], fence, 4 MMAs, commits
//          empty every 2 stages; STAGES slots
#include <cstdio>
#include "../../paper_2511_20340_b200/csrc/common.cuh"
using namespace sf;

__device__ uint32_t crank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ void csync() { asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ void commit2(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(smem_u32(bar)), "h"(mask) : "memory");
}

constexpr int ST = 6;
template <int NN>
__global__ void __cluster_dims__(2, 1, 1) k(int mode, int iters, long long* out, const uint4* src) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t done, bars[8], full[ST], empty[ST];
  __shared__ uint32_t slot;
  uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  const int warp = threadIdx.x / 32;
  const uint32_t rank = crank();
  if (src)  // random operands (tensor-core power depends on the data)
    for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(base)[i] = src[i];
  fence_proxy_async();
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    for (int j = 0; j < 8; ++j) mbar_init(&bars[j], 1);
    for (int j = 0; j < ST; ++j) mbar_init(&full[j], 1), mbar_init(&empty[j], 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before(); __syncthreads(); csync(); tc_fence_after();
  const uint32_t tmem = slot;
  if (rank == 0 && warp == 1) {
    constexpr uint32_t idesc = idesc_bf16_f32(256, NN);
    const uint64_t da0 = sw128_kmajor_desc(smem_u32(base));
    const uint64_t db0 = sw128_kmajor_desc(smem_u32(base + 16384));
    int s = 0, g = 0;
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (mode == 2) { mbar_wait(&full[s], ph); tc_fence_after(); }
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma2(tmem, da0 + kk * 2, db0 + kk * 2, idesc, (i | kk) ? 1u : 0u);
        if (mode == 1 && (i & 1)) commit2(&bars[(g++) & 7], 3);
        if (mode == 2 && (s & 1)) commit2(&empty[s], 3);
      }
      __syncwarp();
      if (++s == ST) s = 0, ph ^= 1;
    }
    if (elect_one()) commit2(&done, 3);
    __syncwarp();
    mbar_wait(&done, 0);
    if ((threadIdx.x & 31) == 0 && blockIdx.x == 0) out[0] = clock64() - t0;
  } else if (rank == 0 && warp == 2 && mode == 2) {
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
      const int gl = s | 1;
      if (i >= ST) mbar_wait(&empty[gl], ph ^ 1);
      if (elect_one()) mbar_arrive(&full[s]);
      __syncwarp();
      if (++s == ST) s = 0, ph ^= 1;
    }
  } else if (rank == 1 && warp == 1) {
    mbar_wait(&done, 0);
  }
  tc_fence_before(); __syncthreads(); csync(); tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

template <int NN>
void run(long long* d, int grid, const uint4* src) {
  cudaFuncSetAttribute(k<NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  for (int mode : {0, 2}) {
    int iters = 16384;
    k<NN><<<grid, 128, 190 * 1024>>>(mode, iters, d, src);  // warm
    cudaEventRecord(e0);
    k<NN><<<grid, 128, 190 * 1024>>>(mode, iters * 8, d, src);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    iters *= 8;
    printf("%s grid %3d pair N=%3d mode %d: %7.1f cycles/k-block (floor %5.1f), %.3f us/k-block wall -> %.0f MHz, %.0f TFLOP/s (%s)\n",
           src ? "rand" : "zero", grid, NN, mode, (double)c / iters, 4 * 256.0 * NN / 512, ms * 1e3 / iters, c / (ms * 1e3),
           (grid / 2) * 2.0 * 256 * NN * 64 * iters / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
}
int main() {
  long long* d; cudaMalloc(&d, 8);
  uint16_t* h = new uint16_t[160 * 1024 / 2];
  unsigned x = 12345;
  for (int i = 0; i < 160 * 1024 / 2; ++i) {  // bf16 ~ N(0, 0.02)-ish magnitudes, random signs / mantissas
    x = x * 1664525u + 1013904223u;
    h[i] = (uint16_t)(0x3C00 + ((x >> 9) & 0x3FF)) | (uint16_t)((x >> 31) << 15);
  }
  uint4* src;
  cudaMalloc(&src, 160 * 1024);
  cudaMemcpy(src, h, 160 * 1024, cudaMemcpyHostToDevice);
  cudaMemset(d, 0, 8);
  for (const uint4* s : {(const uint4*)nullptr, (const uint4*)src}) { run<160>(d, 148, s); run<256>(d, 148, s); }
  return 0;
}
