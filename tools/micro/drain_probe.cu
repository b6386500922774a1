// How long does a GEMM epilogue drain of one 128 x T fp32 accumulator (TMEM -> registers -> global,
// the [T][128] partial-slot layout) take per CTA, and what bounds it? 148 CTAs x 8 epilogue warps
// (two groups of four lane quadrants, alternating 32-column chunks as in gemm_sk_kernel), T = 320.
//  mode 0: tcgen05.ld x32 + wait + 32 coalesced 4-byte stores per chunk (the kernel's drain)
//  mode 1: loads only;  mode 2: stores only (values from registers)
//  mode 3: x32 load of the next chunk issued before the current chunk's stores (double-buffered)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -cudart shared drain_probe.cu -o drain_probe
#include <cstdio>
#include "../../paper_2511_20340_b200/csrc/common.cuh"
using namespace sf;
constexpr int BM = 128;

__global__ void __launch_bounds__(384, 1) drain(float* out, int T, int mode, int reps, long long* cyc) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  long long t0 = clock64();
  if (warp >= 4) {
    const int quad = warp & 3, gid = (warp - 4) >> 2, m = quad * 32 + lane;
    const uint32_t t_row = tmem + ((uint32_t)(quad * 32) << 16);
    float* dst = out + (size_t)blockIdx.x * T * BM;
    for (int rep = 0; rep < reps; ++rep) {
      if (mode == 3) {
        uint32_t ra[32], rb[32];
        int c0 = gid * 32;
        tmem_ld32_async(t_row + (uint32_t)c0, ra);
        tmem_ld_wait();
        for (; c0 < T; c0 += 64) {
          const bool more = c0 + 64 < T;
          if (more) tmem_ld32_async(t_row + (uint32_t)(c0 + 64), rb);
#pragma unroll
          for (int cc = 0; cc < 32; ++cc) dst[(size_t)(c0 + cc) * BM + m] = __uint_as_float(ra[cc]);
          if (more) {
            tmem_ld_wait();
#pragma unroll
            for (int cc = 0; cc < 32; ++cc) ra[cc] = rb[cc];
          }
        }
        continue;
      }
      for (int c0 = gid * 32; c0 < T; c0 += 64) {
        uint32_t r[32];
        if (mode != 2) {
          tmem_ld32_async(t_row + (uint32_t)c0, r);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int cc = 0; cc < 32; ++cc) r[cc] = (uint32_t)(c0 + cc + m);
        }
        if (mode != 1) {
#pragma unroll
          for (int cc = 0; cc < 32; ++cc) dst[(size_t)(c0 + cc) * BM + m] = __uint_as_float(r[cc]);
        } else if (r[0] == 0xFFFFFFFFu && r[31] == 0x12345u) {
          dst[m] = 1.f;  // (keeps the loads alive)
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 128 && blockIdx.x == 0) *cyc = clock64() - t0;
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int T = 320, reps = 8;
  float* out;
  long long* cyc;
  cudaMalloc(&out, (size_t)sms * T * BM * 4);
  cudaMalloc(&cyc, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  const char* names[] = {"ld + 32 STG (kernel)", "ld only", "STG only", "ld double-buffered"};
  for (int mode = 0; mode < 4; ++mode) {
    drain<<<sms, 384>>>(out, T, mode, reps, cyc);
    cudaEventRecord(e0);
    drain<<<sms, 384>>>(out, T, mode, reps, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-24s %.2f us per drain (%lld cycles in CTA 0 / %d), %.0f GB/s stored chip-wide (%s)\n", names[mode],
           ms * 1e3 / reps, c / reps, reps, mode == 1 ? 0.0 : (double)sms * T * BM * 4 * reps / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
