// DRAM read bandwidth of B-byte blocks placed S bytes apart (attention KV pages: a head's 4 KB page
// blocks sit Hkv * 4 KB apart in the [page][head][16][hd] layout) vs contiguous.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stride_bw stride_bw.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const uint4* __restrict__ p, long long nblk, int blk16, long long stride16, int per_cta, unsigned long long* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  // each CTA walks per_cta consecutive blocks of one "head" (stride apart); heads spread over CTAs
  const long long heads = stride16 / blk16;
  const long long h = blockIdx.x % heads, run = blockIdx.x / heads;
  for (int i = 0; i < per_cta; ++i) {
    const long long b = run * per_cta + i;
    if (b >= nblk) break;
    const uint4* q = p + b * stride16 + h * blk16;
    for (int j = threadIdx.x; j < blk16; j += blockDim.x) {
      uint4 v = __ldcs(q + j);
      acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) atomicAdd(sink, 1ull);
}
int main() {
  const size_t bytes = 8ull << 30;
  uint4* p; cudaMalloc(&p, bytes); cudaMemset(p, 1, bytes);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int blk = 4096;
  for (int heads : {1, 8, 32}) {
    for (int per : {8, 40}) {
      const long long stride = (long long)blk * heads;
      const long long nblk = bytes / stride;
      const long long ctas = (nblk + per - 1) / per * heads;
      for (int it = 0; it < 2; ++it) {
        cudaEventRecord(a);
        rd<<<(unsigned)ctas, 256>>>(p, nblk, blk / 16, stride / 16, per, sink);
        cudaEventRecord(b); cudaEventSynchronize(b);
      }
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("block %d B, heads(stride/block) %2d, blocks per CTA %2d: %.0f GB/s\n", blk, heads, per, bytes / (ms * 1e6));
    }
  }
  return 0;
}
