// Is the T = 320 GEMM main loop bound by L2 -> SM delivery, and does k-aligned activation reuse
// across SMs help? 148 CTAs stream units of {16 KB unique weight tile (HBM) + 20 KB activation tile
// (L2-resident, [160 rows x 64 cols] bf16 at k-block kb)} through a 5-stage TMA ring; no MMA.
//   mode 0: weights + activation, k-block (37 c + i) % 64  (stream-K-like: SMs at different k)
//   mode 1: weights + activation, k-block i % 64           (every SM at the same k at once)
//   mode 2: weights only
//   mode 3: activation only, spread;  mode 4: activation only, aligned
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda tma_act_probe.cu -o /tmp/tma_act_probe
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>

#include "../../paper_2511_20340_b200/csrc/common.cuh"
using namespace sf;

constexpr int W_BYTES = 128 * 64 * 2, A_ROWS = 160, A_BYTES = A_ROWS * 64 * 2, STAGES = 5;
constexpr int STAGE = W_BYTES + A_BYTES;

__global__ void __launch_bounds__(64, 1) probe(const __grid_constant__ CUtensorMap mw, const __grid_constant__ CUtensorMap ma,
                                               int mode, int units) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024 - (smem_u32(sm_raw) & 1023)) & 1023);
  __shared__ uint64_t full[STAGES], empty[STAGES];
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int c = blockIdx.x;
  const bool ldw = mode <= 2, lda = mode != 2;
  const bool aligned = mode == 1 || mode == 4;
  if (threadIdx.x == 0) {
    for (int i = 0; i < units; ++i) {
      const int s = i % STAGES;
      mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], (ldw ? W_BYTES : 0) + (lda ? A_BYTES : 0));
      uint8_t* st = sm + s * STAGE;
      if (ldw) tma_load_2d(st, &mw, &full[s], 0, (c * units + i) * 128, kEvictFirst);
      const int kb = aligned ? i % 64 : (37 * c + i) % 64;
      if (lda) tma_load_2d(st + W_BYTES, &ma, &full[s], kb * 64, (c & 1) * A_ROWS, kEvictLast);
    }
  } else if (threadIdx.x == 32) {
    for (int i = 0; i < units; ++i) {
      const int s = i % STAGES;
      mbar_wait(&full[s], (i / STAGES) & 1);
      mbar_arrive(&empty[s]);
    }
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc;
static void map2d(CUtensorMap* m, void* p, long long rows, int cols, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
}

int main() {
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int units = 256;
  const long long wrows = (long long)sms * units * 128;
  void *w, *a;
  cudaMalloc(&w, wrows * 64 * 2);
  cudaMalloc(&a, (size_t)2 * A_ROWS * 4096 * 2);
  cudaMemset(w, 1, wrows * 64 * 2);
  cudaMemset(a, 1, (size_t)2 * A_ROWS * 4096 * 2);
  CUtensorMap mw, ma;
  map2d(&mw, w, wrows, 64, 128);
  map2d(&ma, a, 2 * A_ROWS, 4096, A_ROWS);
  const int smem = STAGES * STAGE + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  const char* names[] = {"W+A spread", "W+A aligned", "W only", "A only spread", "A only aligned"};
  for (int mode = 0; mode < 5; ++mode) {
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      probe<<<sms, 64, smem>>>(mw, ma, mode, units);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double bytes = (double)sms * units * ((mode <= 2 ? W_BYTES : 0) + (mode != 2 ? A_BYTES : 0));
    printf("%-16s %8.2f us  %.3f us/unit  %7.0f GB/s to SMs  (%s)\n", names[mode], best * 1e3, best * 1e3 / units,
           bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
