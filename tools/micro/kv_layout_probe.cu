// Does the paged KV layout limit the decode attention's load rate? 148 CTAs stream 64 KB chunks (K and V
// of 128 keys x 128 dims bf16 for one (sequence, kv head)) through a 3-stage TMA ring, no math, the
// attention kernel's item order (item = (b, head), 5 chunks each, chunks = 8 consecutive pages):
//  layout 0 (the kernel's): pool [pages][Hkv][16 keys][128 dims]; a chunk half = 4-D box {64 dims, 16 keys,
//           1 head, 8 pages} (SWIZZLE_128B): 128-byte pieces at a 256-byte row stride, 4 KB per page
//  layout 1: pool [pages][Hkv][2 halves][16 keys][64 dims]: the same box reads 2 KB contiguous per page
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -cudart shared kv_layout_probe.cu -o kv_layout_probe
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include "../../paper_2511_20340_b200/csrc/common.cuh"
using namespace sf;

constexpr int NST = 3, STAGE = 64 * 1024, HKV = 32, PAGES_PER_SEQ = 40, CHUNKS = 5;

SF_DEV void tma4(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "l"(kEvictFirst)
      : "memory");
}

__global__ void __launch_bounds__(64, 1) probe(const __grid_constant__ CUtensorMap mk, const __grid_constant__ CUtensorMap mv,
                                               int layout, int n_items) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024 - (smem_u32(sm_raw) & 1023)) & 1023);
  __shared__ uint64_t full[NST], empty[NST];
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int seq = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int b = item / HKV, h = item % HKV;
      for (int c = 0; c < CHUNKS; ++c, ++seq) {
        const int st = seq % NST;
        mbar_wait(&empty[st], ((seq / NST) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[st], STAGE);
        const int pg0 = b * PAGES_PER_SEQ + c * 8;
        uint8_t* kb = sm + st * STAGE;
        for (int hf = 0; hf < 2; ++hf) {
          if (layout == 0) {  // coords {dim, key, head, page}
            tma4(kb + hf * 16384, &mk, &full[st], hf * 64, 0, h, pg0);
            tma4(kb + 32768 + hf * 16384, &mv, &full[st], hf * 64, 0, h, pg0);
          } else {  // coords {dim (64), key, half*Hkv... flattened (head, half), page}
            tma4(kb + hf * 16384, &mk, &full[st], 0, 0, h * 2 + hf, pg0);
            tma4(kb + 32768 + hf * 16384, &mv, &full[st], 0, 0, h * 2 + hf, pg0);
          }
        }
      }
    }
  } else if (threadIdx.x == 32) {
    int seq = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x)
      for (int c = 0; c < CHUNKS; ++c, ++seq) {
        const int st = seq % NST;
        mbar_wait(&full[st], (seq / NST) & 1);
        mbar_arrive(&empty[st]);
      }
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc;
static void map4(CUtensorMap* m, void* p, int layout, long long pages) {
  // layout 0: dims {128, 16, HKV, pages}; layout 1: dims {64, 16, 2*HKV, pages}
  cuuint64_t dims[4], strides[3];
  cuuint32_t box[4] = {64, 16, 1, 8}, es[4] = {1, 1, 1, 1};
  if (layout == 0) {
    dims[0] = 128, dims[1] = 16, dims[2] = HKV, dims[3] = pages;
    strides[0] = 256, strides[1] = 16 * 256, strides[2] = (cuuint64_t)HKV * 16 * 256;
  } else {
    dims[0] = 64, dims[1] = 16, dims[2] = 2 * HKV, dims[3] = pages;
    strides[0] = 128, strides[1] = 16 * 128, strides[2] = (cuuint64_t)2 * HKV * 16 * 128;
  }
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode %d\n", (int)r);
}

int main() {
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int B = 64, n_items = B * HKV;
  const long long pages = (long long)B * PAGES_PER_SEQ;
  const size_t bytes = pages * HKV * 16 * 128 * 2;
  void *k, *v;
  cudaMalloc(&k, bytes);
  cudaMalloc(&v, bytes);
  cudaMemset(k, 1, bytes);
  cudaMemset(v, 1, bytes);
  const int smem = NST * STAGE + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  for (int layout = 0; layout < 2; ++layout) {
    CUtensorMap mk, mv;
    map4(&mk, k, layout, pages);
    map4(&mv, v, layout, pages);
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      probe<<<sms, 64, smem>>>(mk, mv, layout, n_items);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    const double moved = (double)n_items * CHUNKS * STAGE;
    printf("layout %d: %.1f us, %.0f GB/s (%s)\n", layout, best * 1e3, moved / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
