// gemm.cu -- the dense contractions of the hot path (QKV / O / SwiGLU / down / W_D / W_P /
// LM head; PAPER Eq.7-10 and the base decoder).
//
// bf16: a swap-AB, persistent stream-K tcgen05 GEMM. The weight W[N, K] is the MMA "A" operand
// (M = 128 weight rows per tile), the skinny activation block X[T, K] (T = B(k+1) = 5..512 rows)
// is the MMA "B" operand (N = T rounded to 16, up to 2 x 256 accumulator columns), so the weight
// -- the bytes that bound the step at small batch -- streams through shared memory exactly once
// per launch, from a tile-contiguous pre-swizzled HBM layout (one 16 KB bulk copy per stage).
// An mbarrier ring feeds one MMA-issuing thread; TMEM holds the fp32 accumulators; 4 epilogue
// warps read them with tcgen05.ld and apply the fused epilogue.
// fp32: a plain smem-tiled SIMT kernel (the fp32 parity mode; no TF32).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "gemm.cuh"

namespace sf {

constexpr int BM = 128;  // weight rows per CTA (MMA M)
constexpr int BK = 64;   // K per stage (one 128-byte swizzle atom of bf16)
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
// ------------------------------------------------------------------------ persistent stream-K kernel
// Grid = G CTAs (G = min(#SMs, units), a function of (N, K) only). The (128-row tile, 64-wide
// k-block) units of the whole GEMM are split into G contiguous equal ranges, so every SM streams
// the same number of weight bytes (no wave quantisation). A tile cut between CTAs is finished by
// the CTA owning its k = 0 segment, which adds the other segments' fp32 partials in k order:
// segment boundaries depend only on (N, K, G) -> the same rounding for every T (batch invariance).
// Warps: 0 = TMA producer, 1 = MMA issuer, 2 = TMEM allocator, 4..7 = epilogue (TMEM lanes 32(w-4)..).
// Two TMEM accumulator buffers (when they fit) let the epilogue of one segment overlap the MMAs
// of the next.
struct SkParams {
  int T, N, K;
  int NT, n_sub, stages, kb_total, n_tiles, G, nbuf, w_tiled;
  int cgrp;  // ring slots released per tcgen05.commit (a commit drains the tensor pipe)
  uint32_t tmem_cols;
  const __nv_bfloat16* w_tiles;  // tile-contiguous weights (w_tiled)
  GemmEpi epi;
  float* partial;  // [G][T][128]
  int* flags;      // [G]
};

SF_DEV void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
SF_DEV int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
SF_DEV void st_release(int* p, int v) { asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }

__global__ void __launch_bounds__(256, 1)
gemm_sk_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmA, const SkParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
  const int a_bytes = p.n_sub * p.NT * BK * 2;
  const int stage_bytes = BM * BK * 2 + a_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)p.stages * stage_bytes);
  uint64_t* empty = full + p.stages;
  uint64_t* accf = empty + p.stages;  // [2]
  uint64_t* acce = accf + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + 2);
  float* xch = reinterpret_cast<float*>(tmem_slot + 4);  // [64][17] SwiGLU exchange

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x;
  const int kb = p.kb_total;
  const long long U = (long long)p.n_tiles * kb;
  const long long u0 = U * c / p.G, u1 = U * (c + 1) / p.G;
  const int cols = p.n_sub * p.NT;

  if (threadIdx.x == 0) {
    if (!p.w_tiled) prefetch_tmap(&tmW);
    prefetch_tmap(&tmA);
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---- TMA producer warp (converged; one elected lane issues)
    int t = (int)(u0 / kb), k = (int)(u0 % kb);
    int s = 0, grp_last = p.cgrp - 1;  // ring slot and the last slot of its release group
    uint32_t ph = 0;
    for (long long u = u0; u < u1; ++u) {
      mbar_wait(&empty[grp_last], ph ^ 1u);  // slot group released
      if (elect_one()) {
        uint8_t* st = smem + (size_t)s * stage_bytes;
        mbar_arrive_expect_tx(&full[s], (uint32_t)stage_bytes);
        if (p.w_tiled)  // tile-contiguous, pre-swizzled weights: one 16 KB bulk copy per stage
          bulk_load(st, p.w_tiles + ((size_t)t * kb + k) * (BM * BK), BM * BK * 2, &full[s], kEvictFirst);
        else
          tma_load_2d(st, &tmW, &full[s], k * BK, t * BM, kEvictFirst);
        for (int j = 0; j < p.n_sub; ++j)
          tma_load_2d(st + BM * BK * 2 + j * p.NT * BK * 2, &tmA, &full[s], k * BK, j * p.NT, kEvictLast);
      }
      __syncwarp();
      if (++k == kb) {
        k = 0;
        ++t;
      }
      if (++s == p.stages) {
        s = 0;
        ph ^= 1u;
      }
      if (s > grp_last) grp_last += p.cgrp;
      if (s == 0) grp_last = p.cgrp - 1;
    }
  } else if (warp == 1) {
    // ---- MMA warp (converged; one elected lane issues every tcgen05 op so commits track them)
    const uint32_t idesc = idesc_bf16_f32(BM, p.NT);
    const uint32_t a_off = (uint32_t)(BM * BK * 2) >> 4;       // B-operand tile offset (16 B units)
    const uint32_t sub_off = (uint32_t)(p.NT * BK * 2) >> 4;   // between activation sub-tiles
    int i = 0, seg = 0;
    int s = 0, gcnt = 0;
    uint32_t ph = 0;
    long long u = u0;
    int t = (int)(u0 / kb);
#ifdef SF_GEMM_PROFILE
    long long tm0 = clock64(), twf = 0, twa = 0;
#endif
    while (u < u1) {
      const long long se = min(u1, (long long)(t + 1) * kb);
      const int b = seg % p.nbuf;
#ifdef SF_GEMM_PROFILE
      long long ta = clock64();
#endif
      mbar_wait(&acce[b], ((uint32_t)(seg / p.nbuf) & 1u) ^ 1u);
#ifdef SF_GEMM_PROFILE
      twa += clock64() - ta;
#endif
      tc_fence_after();
      const uint32_t dacc = tmem + (uint32_t)(b * cols);
      for (long long uu = u; uu < se; ++uu, ++i) {
#ifdef SF_GEMM_PROFILE
        long long tf = clock64();
#endif
        mbar_wait(&full[s], ph);
#ifdef SF_GEMM_PROFILE
        twf += clock64() - tf;
#endif
        tc_fence_after();
        if (elect_one()) {
          const uint64_t dw = sw128_kmajor_desc(smem_u32(smem + (size_t)s * stage_bytes));
          const uint64_t da = dw + a_off;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            for (int j = 0; j < p.n_sub; ++j)
              umma_bf16(dacc + (uint32_t)(j * p.NT), dw + (uint64_t)(kk * 2), da + (uint64_t)(j * sub_off + kk * 2),
                        idesc, (uu > u || kk > 0) ? 1u : 0u);
          if (++gcnt == p.cgrp) umma_commit(&empty[s]);  // frees slots s-cgrp+1..s
        }
        __syncwarp();
        if (gcnt == p.cgrp) gcnt = 0;
        if (++s == p.stages) {
          s = 0;
          ph ^= 1u;
        }
      }
      if (elect_one()) umma_commit(&accf[b]);
      __syncwarp();
      u = se;
      ++seg;
      ++t;
    }
#ifdef SF_GEMM_PROFILE
    if (lane == 0 && (c == 0 || c == p.G / 2))
      printf("T=%d cta %d: %d kb, %.0f cyc/kb total, wait-full %.0f/kb, wait-acc %lld\n", p.T, c, i,
             (double)(clock64() - tm0) / max(i, 1), (double)twf / max(i, 1), twa);
#endif
  } else if (warp >= 4) {
    // ---- epilogue warps
    const int ew = warp - 4;
    const int m = ew * 32 + lane;
    const int etid = threadIdx.x - 128;
    const bool swiglu = p.epi.mode == EPI_SWIGLU_ACT;
    int seg = 0;
    long long u = u0;
    while (u < u1) {
      const int t = (int)(u / kb);
      const long long ts = (long long)t * kb, te = ts + kb;
      const long long se = min(u1, te);
      const int b = seg % p.nbuf;
      mbar_wait_sleep(&accf[b], (uint32_t)(seg / p.nbuf) & 1u);
      tc_fence_after();
      const uint32_t t_row = tmem + (uint32_t)(b * cols) + ((uint32_t)(ew * 32) << 16);
      const int n = t * BM + m;
      const bool is_full = (u == ts) && (se == te);
      const bool is_head = (u == ts) && !is_full;
      if (!is_full && !is_head) {
        // publish this segment's fp32 partial (slot = this CTA; at most one per CTA)
        float* dst = p.partial + (size_t)c * p.T * BM;
        for (int c0 = 0; c0 < p.T; c0 += 16) {
          float v[16];
          tmem_ld16(t_row + (uint32_t)c0, v);
#pragma unroll
          for (int cc = 0; cc < 16; ++cc)
            if (c0 + cc < p.T) dst[(size_t)(c0 + cc) * BM + m] = v[cc];
        }
        __threadfence();
        named_sync(1, 128);
        if (etid == 0) st_release(&p.flags[c], 1);
      } else {
        // owners of the other k segments of this tile (they publish them first thing)
        int c_lo = c + 1, c_hi = c;
        if (is_head) {
          const long long ul = te - 1;
          c_hi = (int)(((ul + 1) * p.G + U - 1) / U) - 1;
          if (etid == 0)
            for (int cc = c_lo; cc <= c_hi; ++cc)
              while (ld_acquire(&p.flags[cc]) == 0) {
              }
          named_sync(1, 128);
        }
        for (int c0 = 0; c0 < p.T; c0 += 16) {
          float v[16];
          tmem_ld16(t_row + (uint32_t)c0, v);
          for (int cc = c_lo; cc <= c_hi; ++cc) {  // fixed k order
            const float* src = p.partial + (size_t)cc * p.T * BM;
#pragma unroll
            for (int q = 0; q < 16; ++q)
              if (c0 + q < p.T) v[q] += __ldcg(&src[(size_t)(c0 + q) * BM + m]);
          }
          if (!swiglu) {
#pragma unroll
            for (int q = 0; q < 16; ++q)
              if (c0 + q < p.T) epi_apply<__nv_bfloat16>(p.epi, c0 + q, n, v[q]);
          } else {
            named_sync(1, 128);
            if (m >= 64) {
#pragma unroll
              for (int q = 0; q < 16; ++q) xch[(m - 64) * 17 + q] = v[q];
            }
            named_sync(1, 128);
            if (m < 64) {
              const int f = t * 64 + m;
              __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.epi.out);
#pragma unroll
              for (int q = 0; q < 16; ++q)
                if (c0 + q < p.T)
                  o[(size_t)(c0 + q) * p.epi.ldo + f] = __float2bfloat16_rn(silu_f(v[q]) * xch[m * 17 + q]);
            }
          }
        }
        if (is_head) {
          named_sync(1, 128);
          if (etid == 0)
            for (int cc = c_lo; cc <= c_hi; ++cc) p.flags[cc] = 0;  // re-arm for the next launch
        }
      }
      tc_fence_before();
      named_sync(1, 128);
      if (etid == 0) mbar_arrive(&acce[b]);
      u = se;
      ++seg;
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

// ------------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_once;

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

constexpr int kMaxSMs = 160;
static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    n = std::min(std::max(n, 1), kMaxSMs);
  }
  return n;
}

int64_t gemm_partial_elems(bool is_bf16, int T, int N, int K) {
  (void)N;
  (void)K;
  if (!is_bf16) return 0;
  return (int64_t)kMaxSMs * BM * std::min(T, 512);
}

// Tile-contiguous weight layout: block (t, k) = rows [128t, +128) x cols [64k, +64) stored as the
// exact 16 KB shared-memory image of a 128B-swizzled K-major tile (16-byte chunk c of row r at
// chunk position c ^ (r & 7)); blocks ordered t-major then k. A stream-K range of consecutive
// (t, k) units is then one contiguous stretch of HBM.
__global__ void pack_tiled_kernel(const __nv_bfloat16* __restrict__ src, __nv_bfloat16* __restrict__ dst, int K) {
  const int kb = K / BK;
  const int blk = blockIdx.x;
  const int t = blk / kb, k = blk % kb;
  const int r = threadIdx.x;  // 128 rows
  const uint4* s = reinterpret_cast<const uint4*>(src + ((size_t)t * BM + r) * K + (size_t)k * BK);
  uint4* d = reinterpret_cast<uint4*>(dst + (size_t)blk * BM * BK + (size_t)r * BK);
#pragma unroll
  for (int c = 0; c < 8; ++c) d[c ^ (r & 7)] = s[c];
}

cudaError_t gemm_pack_weight(const void* src, void* dst, int N, int K, cudaStream_t st) {
  if (N % BM || K % BK) return cudaErrorInvalidValue;
  pack_tiled_kernel<<<(N / BM) * (K / BK), BM, 0, st>>>((const __nv_bfloat16*)src, (__nv_bfloat16*)dst, K);
  return cudaGetLastError();
}

static cudaError_t launch_sk(const void* A, int lda, const void* W, bool w_tiled, int T, int N, int K,
                             const GemmEpi& epi, const GemmScratch& scratch, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_sk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  SkParams p{};
  p.T = T;
  p.N = N;
  p.K = K;
  tc_shape(T, &p.NT, &p.n_sub);
  p.kb_total = K / BK;
  p.n_tiles = N / BM;
  const long long U = (long long)p.n_tiles * p.kb_total;
  p.G = (int)std::min<long long>(num_sms(), U);  // depends on (N, K) only
  const int cols = p.n_sub * p.NT;
  p.nbuf = (2 * cols <= 512) ? 2 : 1;
  p.tmem_cols = 32;
  while ((int)p.tmem_cols < p.nbuf * cols) p.tmem_cols <<= 1;
  const int stage_bytes = BM * BK * 2 + p.n_sub * p.NT * BK * 2;
  // deep ring: ~200 KB in flight per SM covers loaded-HBM latency (Little's law)
  static const int env_st = getenv("SF_GEMM_STAGES") ? atoi(getenv("SF_GEMM_STAGES")) : 0;
  p.stages = std::max(2, std::min(16, (216 * 1024) / stage_bytes));
  if (env_st >= 2 && env_st * stage_bytes <= 216 * 1024) p.stages = env_st;
  // release slots in groups of cgrp (>= 3 groups in the ring; cgrp divides stages)
  static const int env_cg = getenv("SF_GEMM_CGRP") ? atoi(getenv("SF_GEMM_CGRP")) : 0;
  p.cgrp = 1;
  for (int c = 8; c >= 2; c >>= 1)
    if (c * 3 <= p.stages || (c * 2 <= p.stages && c == 2)) {
      p.cgrp = c;
      break;
    }
  if (env_cg >= 1 && env_cg * 2 <= p.stages) p.cgrp = env_cg;
  p.stages = (p.stages / p.cgrp) * p.cgrp;
  p.epi = epi;
  p.partial = scratch.partial;
  p.flags = scratch.counters;
  p.w_tiled = w_tiled ? 1 : 0;
  p.w_tiles = (const __nv_bfloat16*)W;
  if (!scratch.partial || scratch.partial_elems < (int64_t)p.G * T * BM || scratch.n_counters < p.G)
    return cudaErrorInvalidValue;
  const size_t smem = (size_t)p.stages * stage_bytes + 1024 + (2 * p.stages + 4) * 8 + 16 + 64 * 17 * 4;
  CUtensorMap mw, ma;
  memset(&mw, 0, sizeof(mw));
  if (!w_tiled && !make_map(&mw, W, N, K, K, BM)) return cudaErrorInvalidValue;
  if (!make_map(&ma, A, T, K, lda, p.NT)) return cudaErrorInvalidValue;
  gemm_sk_kernel<<<p.G, 256, smem, st>>>(mw, ma, p);
  return cudaGetLastError();
}

static cudaError_t gemm_launch_chunk(bool is_bf16, const void* A, int lda, const void* W, bool w_tiled, int T,
                                     int N, int K, const GemmEpi& epi, const GemmScratch& scratch,
                                     cudaStream_t st) {
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
  return launch_sk(A, lda, W, w_tiled, T, N, K, epi, scratch, st);
}

// Rows beyond 512 (the TMEM accumulator capacity) are processed as independent column chunks;
// per-element arithmetic is unchanged, so results do not depend on the chunking.
cudaError_t gemm_launch(bool is_bf16, const void* A, int lda, const void* W, bool w_tiled, int T, int N, int K,
                        const GemmEpi& epi, const GemmScratch& scratch, cudaStream_t st) {
  if (!is_bf16 || T <= 512) return gemm_launch_chunk(is_bf16, A, lda, W, w_tiled, T, N, K, epi, scratch, st);
  for (int t0 = 0; t0 < T; t0 += 512) {
    GemmEpi e = epi;
    const size_t out_elt = (epi.mode == EPI_STORE_ACT || epi.mode == EPI_SWIGLU_ACT) ? 2 : 4;
    e.out = (char*)epi.out + (size_t)t0 * epi.ldo * out_elt;
    if (epi.tap) e.tap = epi.tap + (size_t)t0 * epi.ldo;
    cudaError_t r = gemm_launch_chunk(true, (const char*)A + (size_t)t0 * lda * 2, lda, W, w_tiled,
                                      std::min(512, T - t0), N, K, e, scratch, st);
    if (r != cudaSuccess) return r;
  }
  return cudaSuccess;
}

}  // namespace sf
