// gemm.cu -- the dense contractions of the hot path (QKV / O / SwiGLU / down / W_D / W_P /
// LM head; PAPER Eq.7-10 and the base decoder).
//
// bf16: a swap-AB tcgen05 GEMM. The weight W[N, K] is the MMA "A" operand (M = 128 weight rows
// per CTA), the skinny activation block X[T, K] (T = B(k+1) = 5..512 rows) is the MMA "B"
// operand (N = T rounded to 16, up to 2 x 256 accumulators), so the weight -- the bytes that
// bound the step at small batch -- streams through shared memory exactly once per launch.
// TMA (128B swizzle) feeds a multi-stage mbarrier ring; one thread issues tcgen05.mma into a
// TMEM fp32 accumulator; 4 epilogue warps read TMEM with tcgen05.ld and apply the fused
// epilogue. Split-K (a function of the weight shape only -> batch-invariant, reading C23) is
// reduced deterministically by the last-arriving CTA in split order.
// fp32: a plain smem-tiled SIMT kernel (the fp32 parity mode; no TF32).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <mutex>

#include "common.cuh"
#include "gemm.cuh"

namespace sf {

constexpr int BM = 128;  // weight rows per CTA (MMA M)
constexpr int BK = 64;   // K per stage (one 128-byte swizzle atom of bf16)

struct TcParams {
  int T, N, K;
  int NT;          // MMA N (columns per accumulator), multiple of 16
  int n_sub;       // accumulators (n_sub * NT >= T)
  int stages;
  int kb_total;
  int splits;
  uint32_t tmem_cols;
  GemmEpi epi;
  float* partial;
  int* counters;
};

template <typename TA>
SF_DEV void epi_apply(const GemmEpi& e, int t, int n, float v) {
  const size_t off = (size_t)t * e.ldo + n;
  switch (e.mode) {
    case EPI_STORE_ACT: reinterpret_cast<TA*>(e.out)[off] = Elt<TA>::from_f(v); break;
    case EPI_STORE_F32: reinterpret_cast<float*>(e.out)[off] = v; break;
    case EPI_ADD_F32: {
      float* o = reinterpret_cast<float*>(e.out) + off;
      const float r = *o + v;
      *o = r;
      if (e.tap) e.tap[off] = r;
    } break;
    case EPI_BIAS_F32: reinterpret_cast<float*>(e.out)[off] = v + e.bias[n]; break;
    default: break;
  }
}
SF_DEV float silu_f(float g) { return g / (1.f + expf(-g)); }

// ------------------------------------------------------------------------ tcgen05 kernel
__global__ void __launch_bounds__(128, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmA, const TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
  const int a_bytes = p.n_sub * p.NT * BK * 2;
  const int stage_bytes = BM * BK * 2 + a_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)p.stages * stage_bytes);
  uint64_t* empty = full + p.stages;
  uint64_t* accum = empty + p.stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);
  int* flag_s = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile_n = blockIdx.x, split = blockIdx.y;
  const int n0 = tile_n * BM;
  const int kb_per = p.kb_total / p.splits, kb_rem = p.kb_total % p.splits;
  const int kb_begin = split * kb_per + min(split, kb_rem);
  const int kb_count = kb_per + (split < kb_rem ? 1 : 0);

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmW);
    prefetch_tmap(&tmA);
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accum, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---- TMA producer
    for (int i = 0; i < kb_count; ++i) {
      const int s = i % p.stages;
      const uint32_t ph = (uint32_t)(i / p.stages) & 1u;
      mbar_wait(&empty[s], ph ^ 1u);
      uint8_t* st = smem + (size_t)s * stage_bytes;
      mbar_arrive_expect_tx(&full[s], (uint32_t)stage_bytes);
      const int kc = (kb_begin + i) * BK;
      tma_load_2d(st, &tmW, &full[s], kc, n0, kEvictFirst);
      for (int j = 0; j < p.n_sub; ++j)
        tma_load_2d(st + BM * BK * 2 + j * p.NT * BK * 2, &tmA, &full[s], kc, j * p.NT, kEvictLast);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer (single thread)
    const uint32_t idesc = idesc_bf16_f32(BM, p.NT);
    for (int i = 0; i < kb_count; ++i) {
      const int s = i % p.stages;
      const uint32_t ph = (uint32_t)(i / p.stages) & 1u;
      mbar_wait(&full[s], ph);
      tc_fence_after();
      const uint32_t wa = smem_u32(smem + (size_t)s * stage_bytes);
      const uint64_t dw = sw128_kmajor_desc(wa);
#pragma unroll
      for (int kk = 0; kk < BK / 16; ++kk) {
        for (int j = 0; j < p.n_sub; ++j) {
          const uint64_t da = sw128_kmajor_desc(wa + BM * BK * 2 + j * p.NT * BK * 2);
          umma_bf16(tmem + (uint32_t)(j * p.NT), dw + (uint64_t)(kk * 2), da + (uint64_t)(kk * 2), idesc,
                    (i > 0 || kk > 0) ? 1u : 0u);
        }
      }
      umma_commit(&empty[s]);  // frees the smem slot once these MMAs have read it
    }
    umma_commit(accum);
  }
  __syncwarp();

  // ---- epilogue: all 4 warps; thread owns accumulator row m = weight row n0 + m
  mbar_wait(accum, 0);
  tc_fence_after();
  const int m = warp * 32 + lane;
  const int n = n0 + m;
  const uint32_t t_row = tmem + ((uint32_t)(warp * 32) << 16);
  bool do_epi = true;
  if (p.splits > 1) {
    for (int c0 = 0; c0 < p.T; c0 += 16) {
      float v[16];
      tmem_ld16(t_row + (uint32_t)c0, v);
#pragma unroll
      for (int c = 0; c < 16; ++c)
        if (c0 + c < p.T) p.partial[((size_t)split * p.T + c0 + c) * p.N + n] = v[c];
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int old = atomicAdd(&p.counters[tile_n], 1);
      const int last = (old == p.splits - 1);
      if (last) p.counters[tile_n] = 0;  // re-arm for the next launch (stream-ordered)
      *flag_s = last;
    }
    __syncthreads();
    do_epi = *flag_s != 0;
    __threadfence();
  }
  if (do_epi) {
    float* xch = reinterpret_cast<float*>(smem);  // stage buffers are idle now
    const bool swiglu = p.epi.mode == EPI_SWIGLU_ACT;
    for (int c0 = 0; c0 < p.T; c0 += 16) {
      float v[16];
      tmem_ld16(t_row + (uint32_t)c0, v);
      if (p.splits > 1) {
        float acc[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) acc[c] = 0.f;
        for (int s = 0; s < p.splits; ++s) {  // fixed order 0..S-1
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            float x = v[c];
            if (s != split)
              x = (c0 + c < p.T) ? __ldcg(&p.partial[((size_t)s * p.T + c0 + c) * p.N + n]) : 0.f;
            acc[c] = (s == 0) ? x : acc[c] + x;
          }
        }
#pragma unroll
        for (int c = 0; c < 16; ++c) v[c] = acc[c];
      }
      if (!swiglu) {
#pragma unroll
        for (int c = 0; c < 16; ++c)
          if (c0 + c < p.T) epi_apply<__nv_bfloat16>(p.epi, c0 + c, n, v[c]);
      } else {
        __syncthreads();
        if (m >= 64) {
#pragma unroll
          for (int c = 0; c < 16; ++c) xch[(m - 64) * 17 + c] = v[c];
        }
        __syncthreads();
        if (m < 64) {
          const int f = tile_n * 64 + m;
          __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.epi.out);
#pragma unroll
          for (int c = 0; c < 16; ++c)
            if (c0 + c < p.T)
              o[(size_t)(c0 + c) * p.epi.ldo + f] = __float2bfloat16_rn(silu_f(v[c]) * xch[m * 17 + c]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, p.tmem_cols);
}

// ------------------------------------------------------------------------ SIMT fp32 kernel
// grid (ceil(Nout/32), ceil(T/32)), block (32, 8). Each output element reduces k = 0..K-1 in
// order (batch-invariant). DUAL: SwiGLU over the 64-row interleaved gate/up layout.
template <bool DUAL>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const float* __restrict__ A, int lda,
                                                         const float* __restrict__ W, int T, int N, int K,
                                                         GemmEpi epi) {
  __shared__ float As[32][33];
  __shared__ float Ws[32][33];
  __shared__ float Us[DUAL ? 32 : 1][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int Nout = DUAL ? N / 2 : N;
  const int ob = blockIdx.x * 32, tb = blockIdx.y * 32;
  float acc[4] = {0, 0, 0, 0}, accu[4] = {0, 0, 0, 0};
  auto wrow = [&](int o) { return DUAL ? (o / 64) * 128 + (o % 64) : o; };
  for (int kt = 0; kt < K; kt += 32) {
    for (int i = ty; i < 32; i += 8) {
      const int t = tb + i, kk = kt + tx;
      As[i][tx] = (t < T && kk < K) ? A[(size_t)t * lda + kk] : 0.f;
      const int o = ob + i;
      Ws[i][tx] = (o < Nout && kk < K) ? W[(size_t)wrow(o) * K + kk] : 0.f;
      if (DUAL) Us[i][tx] = (o < Nout && kk < K) ? W[(size_t)(wrow(o) + 64) * K + kk] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int c = 0; c < 32; ++c) {
      const float w = Ws[tx][c];
      const float u = DUAL ? Us[tx][c] : 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float a = As[ty + 8 * i][c];
        acc[i] = fmaf(a, w, acc[i]);
        if (DUAL) accu[i] = fmaf(a, u, accu[i]);
      }
    }
    __syncthreads();
  }
  const int o = ob + tx;
  if (o >= Nout) return;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = tb + ty + 8 * i;
    if (t >= T) continue;
    if (DUAL)
      reinterpret_cast<float*>(epi.out)[(size_t)t * epi.ldo + o] = silu_f(acc[i]) * accu[i];
    else
      epi_apply<float>(epi, t, o, acc[i]);
  }
}

// ------------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_once;
static bool g_attr_set = false;

static bool ensure_encode() {
  std::call_once(g_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode != nullptr;
}

static bool make_map(CUtensorMap* m, const void* ptr, int rows, int K, int ld_elems, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld_elems * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int gemm_splits(int N, int K) {
  const int tiles = N / BM;
  const int kb = K / BK;
  if (tiles >= 148) return 1;
  int s = (int)std::lround(148.0 / tiles);
  s = std::max(1, std::min(s, kb / 4));
  return std::max(1, s);
}

static void tc_shape(int T, int* NT, int* n_sub) {
  const int Tp = std::max(16, (T + 15) / 16 * 16);
  if (Tp <= 256) {
    *NT = Tp;
    *n_sub = 1;
  } else {
    *n_sub = (Tp + 255) / 256;
    *NT = ((Tp + *n_sub - 1) / *n_sub + 15) / 16 * 16;
  }
}

int64_t gemm_partial_elems(bool is_bf16, int T, int N, int K) {
  if (!is_bf16) return 0;
  const int s = gemm_splits(N, K);
  return s > 1 ? (int64_t)s * T * N : 0;
}

static cudaError_t gemm_launch_chunk(bool is_bf16, const void* A, int lda, const void* W, int T, int N, int K,
                                     const GemmEpi& epi, const GemmScratch& scratch, cudaStream_t st);

// Rows beyond 512 (the two 256-column TMEM accumulators) are processed as independent column
// chunks; per-element arithmetic is unchanged, so results do not depend on the chunking.
cudaError_t gemm_launch(bool is_bf16, const void* A, int lda, const void* W, int T, int N, int K,
                        const GemmEpi& epi, const GemmScratch& scratch, cudaStream_t st) {
  if (!is_bf16 || T <= 512) return gemm_launch_chunk(is_bf16, A, lda, W, T, N, K, epi, scratch, st);
  for (int t0 = 0; t0 < T; t0 += 512) {
    GemmEpi e = epi;
    const size_t out_elt = (epi.mode == EPI_STORE_ACT || epi.mode == EPI_SWIGLU_ACT) ? 2 : 4;
    e.out = (char*)epi.out + (size_t)t0 * epi.ldo * out_elt;
    if (epi.tap) e.tap = epi.tap + (size_t)t0 * epi.ldo;
    cudaError_t r = gemm_launch_chunk(true, (const char*)A + (size_t)t0 * lda * 2, lda, W, std::min(512, T - t0), N,
                                      K, e, scratch, st);
    if (r != cudaSuccess) return r;
  }
  return cudaSuccess;
}

static cudaError_t gemm_launch_chunk(bool is_bf16, const void* A, int lda, const void* W, int T, int N, int K,
                                     const GemmEpi& epi, const GemmScratch& scratch, cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  if (!is_bf16) {
    const int Nout = epi.mode == EPI_SWIGLU_ACT ? N / 2 : N;
    dim3 grid((Nout + 31) / 32, (T + 31) / 32), block(32, 8);
    if (epi.mode == EPI_SWIGLU_ACT)
      gemm_simt_kernel<true><<<grid, block, 0, st>>>((const float*)A, lda, (const float*)W, T, N, K, epi);
    else
      gemm_simt_kernel<false><<<grid, block, 0, st>>>((const float*)A, lda, (const float*)W, T, N, K, epi);
    return cudaGetLastError();
  }
  if (N % BM || K % BK || T > 512) return cudaErrorInvalidValue;
  if (!ensure_encode()) return cudaErrorNotSupported;
  TcParams p{};
  p.T = T;
  p.N = N;
  p.K = K;
  tc_shape(T, &p.NT, &p.n_sub);
  p.kb_total = K / BK;
  p.splits = gemm_splits(N, K);
  p.epi = epi;
  p.partial = scratch.partial;
  p.counters = scratch.counters;
  if (p.splits > 1) {
    if (!scratch.partial || scratch.partial_elems < (int64_t)p.splits * T * N || !scratch.counters ||
        scratch.n_counters < N / BM)
      return cudaErrorInvalidValue;
  }
  const int cols = p.n_sub * p.NT;
  p.tmem_cols = 32;
  while ((int)p.tmem_cols < cols) p.tmem_cols <<= 1;
  const int stage_bytes = BM * BK * 2 + p.n_sub * p.NT * BK * 2;
  // Size the ring so that every CTA of the launch is resident at once (no tail wave): a
  // memory-bound launch then shares HBM evenly across all its weight streams.
  const int ctas = (N / BM) * p.splits;
  int per_sm = std::min(4, (ctas + 147) / 148);
  int stages = 0;
  for (; per_sm >= 1; --per_sm) {
    const int budget = (226 * 1024) / per_sm - 2048;
    stages = std::min(8, budget / stage_bytes);
    if (stages >= 3 || per_sm == 1) break;
  }
  p.stages = std::max(2, stages);
  const size_t smem = (size_t)p.stages * stage_bytes + 1024 + (2 * p.stages + 1) * 8 + 16;
  if (!g_attr_set) {
    cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    g_attr_set = true;
  }
  CUtensorMap mw, ma;
  if (!make_map(&mw, W, N, K, K, BM)) return cudaErrorInvalidValue;
  if (!make_map(&ma, A, T, K, lda, p.NT)) return cudaErrorInvalidValue;
  dim3 grid(N / BM, p.splits);
  gemm_tc_kernel<<<grid, 128, smem, st>>>(mw, ma, p);
  return cudaGetLastError();
}

}  // namespace sf
