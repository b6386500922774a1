// gemm.cuh -- GEMM launch interface shared by the runtime.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sf {

enum EpiMode : int {
  EPI_STORE_ACT = 0,   // out_act[t, n] = acc                     (next GEMM's operand)
  EPI_STORE_F32 = 1,   // out_f32[t, n] = acc                     (logits, residual init)
  EPI_ADD_F32 = 2,     // out_f32[t, n] += acc; tap[t, n] = result (residual stream, Eq.7)
  EPI_BIAS_F32 = 3,    // out_f32[t, n] = acc + bias[n]           (positional FFN, Eq.9)
  EPI_SWIGLU_ACT = 4,  // W rows interleaved in 64-row groups [gate_i; up_i]:
                       // out_act[t, 64 i + m] = silu(gate) * up  (SwiGLU, P197)
};

struct GemmEpi {
  int mode = EPI_STORE_ACT;
  void* out = nullptr;
  int ldo = 0;             // row stride of out (elements)
  const float* bias = nullptr;
  float* tap = nullptr;    // optional extra copy (ADD_F32 only), row stride ldo
};

struct GemmScratch {
  float* partial = nullptr;   // split-K partials
  int64_t partial_elems = 0;
  int* counters = nullptr;    // per-N-tile arrival counters (zeroed; kernels re-zero them)
  int n_counters = 0;
};

// out = A[T, K] . W[N, K]^T with fp32 accumulation.
// is_bf16: A, W bf16 (tcgen05 path, requires N % 128 == 0, K % 64 == 0); W either row-major
// [N, K] (w_tiled = false) or in the tile-contiguous layout written by gemm_pack_weight.
// Otherwise fp32 (SIMT path, W row-major). act outputs are in the same dtype as A.
cudaError_t gemm_launch(bool is_bf16, const void* A, int lda, const void* W, bool w_tiled, int T, int N, int K,
                        const GemmEpi& epi, const GemmScratch& scratch, cudaStream_t s);
// Row-major bf16 W[N, K] -> tile-contiguous 128x64 pre-swizzled layout (same byte count).
cudaError_t gemm_pack_weight(const void* src, void* dst, int N, int K, cudaStream_t s);

// scratch floats needed by gemm_launch for (T, N, K)
int64_t gemm_partial_elems(bool is_bf16, int T, int N, int K);

}  // namespace sf
