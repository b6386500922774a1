// common.cuh -- shared device helpers for the SpecFormer sm_100a kernels.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <utility>

#define SF_DEV __device__ __forceinline__

namespace sf {

// ---------------------------------------------------------------- element types
template <typename T> struct Elt;
template <> struct Elt<float> {
  static SF_DEV float to_f(float v) { return v; }
  static SF_DEV float from_f(float v) { return v; }
};
template <> struct Elt<__nv_bfloat16> {
  static SF_DEV float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
  static SF_DEV __nv_bfloat16 from_f(float v) { return __float2bfloat16_rn(v); }  // RNE (reading C17)
};

template <typename T> SF_DEV float ld_f(const T* p) { return Elt<T>::to_f(*p); }
template <typename T> SF_DEV void st_f(T* p, float v) { *p = Elt<T>::from_f(v); }

// ---------------------------------------------------------------- RoPE (reading C5)
// Rotate-half pair (x1 = dim i, x2 = dim i + hd/2) at angle (c, s), with explicitly rounded
// operations (no FMA contraction) so every kernel that applies it -- the RoPE/append kernels and
// the QKV GEMM's fused epilogue -- produces the same bits from the same bf16 inputs.
SF_DEV float rope_y1(float x1, float x2, float c, float s) { return __fsub_rn(__fmul_rn(x1, c), __fmul_rn(x2, s)); }
SF_DEV float rope_y2(float x1, float x2, float c, float s) { return __fadd_rn(__fmul_rn(x2, c), __fmul_rn(x1, s)); }

// ---------------------------------------------------------------- warp reductions
SF_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
SF_DEV float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum with a FIXED reduction tree (batch-invariant: depends only on blockDim).
template <int NT>
SF_DEV float block_sum(float v, float* red /* >= NT/32 floats */) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
  if (w == 0) {
    s = (l < NT / 32) ? red[l] : 0.f;
    s = warp_sum(s);
    if (l == 0) red[0] = s;
  }
  __syncthreads();
  return red[0];
}

// Block-wide sum for a runtime blockDim (multiple of 32, <= 1024) with a fixed tree: warp shuffles,
// then warp 0 over the per-warp sums in warp order (depends on blockDim only -> batch-invariant).
SF_DEV float block_sum_dyn(float v, float* red /* >= 32 floats */) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    float s = (l < (int)(blockDim.x >> 5)) ? red[l] : 0.f;
    s = warp_sum(s);
    if (l == 0) red[0] = s;
  }
  __syncthreads();
  return red[0];
}

// ---------------------------------------------------------------- programmatic dependent launch
// Every kernel of the step is launched with programmatic stream serialisation: it may start while
// its predecessor drains, does only dependency-free work (barrier init, TMEM alloc, smem clears,
// weight prefetch) before pdl_wait(), and lets its own successor launch once all of its CTAs have
// passed pdl_wait() (pdl_trigger()). pdl_wait() returns when every prerequisite grid has completed
// and its memory is visible, so the chain stays fully ordered. No-ops without the launch attribute.
SF_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
SF_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = !(getenv("SF_NO_PDL") && atoi(getenv("SF_NO_PDL")) > 0);
  return on;
}
// Host: cuTensorMapEncodeTiled results cached by their arguments (the same weights, KV pools and
// activation buffers are described again at every eager launch -- prefill runs thousands of them).
struct TmapKey {
  uint64_t w[18];
  bool operator==(const TmapKey& o) const { return memcmp(w, o.w, sizeof(w)) == 0; }
};
struct TmapHash {
  size_t operator()(const TmapKey& k) const {
    uint64_t h = 1469598103934665603ull;
    for (uint64_t v : k.w) h = (h ^ v) * 1099511628211ull;
    return (size_t)h;
  }
};
inline CUresult encode_tmap_cached(PFN_cuTensorMapEncodeTiled_v12000 enc, CUtensorMap* m, CUtensorMapDataType dt,
                                   cuuint32_t rank, void* ptr, const cuuint64_t* dims, const cuuint64_t* strides,
                                   const cuuint32_t* box, CUtensorMapSwizzle swz) {
  TmapKey k;
  memset(&k, 0, sizeof(k));
  k.w[0] = (uint64_t)ptr;
  k.w[1] = ((uint64_t)dt << 32) | ((uint64_t)swz << 8) | rank;
  for (cuuint32_t i = 0; i < rank && i < 5; ++i) {
    k.w[2 + i] = dims[i];
    k.w[7 + i] = box[i];
    if (i + 1 < rank) k.w[12 + i] = strides[i];
  }
  static std::mutex mu;
  static std::unordered_map<TmapKey, CUtensorMap, TmapHash> cache;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(k);
    if (it != cache.end()) {
      *m = it->second;
      return CUDA_SUCCESS;
    }
  }
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  const CUresult r = enc(m, dt, rank, ptr, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r == CUDA_SUCCESS) {
    std::lock_guard<std::mutex> lk(mu);
    if (cache.size() > 4096) cache.clear();  // (buffers of destroyed handles)
    cache.emplace(k, *m);
  }
  return r;
}

// <<<grid, block, smem, stream>>> with the PDL attribute (and an optional cluster shape).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------- kernel timeline (tools only)
// With SF_KTRACE=1 every kernel's recorder thread appends (kernel id, SM, start, dependency
// resolved, end) %globaltimer stamps to a device log (tools/ktrace.py reconstructs the per-launch
// timeline of a CUDA-graph step). Off by default: one predicated load per CTA.
enum KtKind : uint32_t {
  KT_GEMM = 1, KT_RESID_NORM, KT_ROPE, KT_ATTN, KT_RMSNORM, KT_GROUP_RMS, KT_EMBED, KT_ARGMAX_P, KT_ARGMAX_F,
  KT_ACCEPT, KT_BIDIR, KT_GATHER, KT_ROWS, KT_GEMM_SIMT, KT_ATTN_PART, KT_ATTN_COMB, KT_MISC, KT_ITEM, KT_GEMM_SEQ
};

struct KtRec {
  uint32_t kid, smid;
  unsigned long long t0, tw, t1;
  unsigned long long pad;
};
struct KtBuf {
  KtRec* rec;
  unsigned* cnt;
  unsigned cap;
};
static __device__ KtBuf g_kt;  // one per translation unit, set by kt_setup_*()
SF_DEV unsigned long long kt_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
struct KtScope {
  unsigned long long t0 = 0, tw = 0;
  uint32_t kid = 0;
  bool on = false;
  SF_DEV KtScope(uint32_t kind, uint32_t param, int who = 0) {
    if (g_kt.rec && (int)threadIdx.x == who) {
      on = true;
      kid = (kind << 24) | (param & 0xFFFFFFu);
      t0 = kt_now();
    }
  }
  SF_DEV void mark() {
    if (on) tw = kt_now();
  }
  SF_DEV ~KtScope() {
    if (!on) return;
    const unsigned i = atomicAdd(g_kt.cnt, 1u);
    if (i < g_kt.cap) {
      uint32_t sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      KtRec r;
      r.kid = kid;
      r.smid = sm;
      r.t0 = t0;
      r.tw = tw ? tw : t0;
      r.t1 = kt_now();
      r.pad = 0;
      g_kt.rec[i] = r;
    }
  }
};
// one free-form record (t0, tw, t1) -- e.g. a work item inside a persistent kernel
SF_DEV void kt_item(uint32_t param, unsigned long long t0, unsigned long long tw, unsigned long long t1) {
  if (!g_kt.rec) return;
  const unsigned i = atomicAdd(g_kt.cnt, 1u);
  if (i >= g_kt.cap) return;
  KtRec r;
  r.kid = (KT_ITEM << 24) | (param & 0xFFFFFFu);
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r.smid));
  r.t0 = t0;
  r.tw = tw;
  r.t1 = t1;
  r.pad = 0;
  g_kt.rec[i] = r;
}
static inline cudaError_t kt_setup_tu(const KtBuf& b) { return cudaMemcpyToSymbol(g_kt, &b, sizeof(b)); }

// ---------------------------------------------------------------- PTX wrappers (sm_100a)
SF_DEV uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

SF_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
SF_DEV void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
SF_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
SF_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
SF_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
SF_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
SF_DEV void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// One lane of a converged warp (deterministic: the same lane every call when all 32 are active).
SF_DEV bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// Wait with back-off: for warps that idle for long stretches (epilogue warps), so their polling
// does not steal issue slots from the single-thread TMA / MMA roles on the same SM sub-partition.
SF_DEV void mbar_wait_sleep(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    if (done) return;
    __nanosleep(256);
  }
}

// TMA 2-D tile load (global -> shared), completion via mbarrier transaction bytes.
SF_DEV void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
// TMA 4-D tile load (global -> shared), completion via mbarrier transaction bytes.
SF_DEV void tma_load_4d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2, int c3,
                        uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "l"(policy)
      : "memory");
}
// 1-D bulk copy global -> shared (contiguous bytes, multiple of 16), mbarrier completion.
SF_DEV void bulk_load(void* smem_dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(smem_dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// L2 prefetch of a contiguous global range (TMA engine; no shared memory, no completion)
SF_DEV void prefetch_l2(const void* src, uint32_t bytes, uint64_t policy) {
  asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(src), "r"(bytes), "l"(policy)
               : "memory");
}
SF_DEV void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
constexpr uint64_t kEvictFirst = 0x12F0000000000000ull;
constexpr uint64_t kEvictLast = 0x14F0000000000000ull;

// tcgen05 / TMEM
SF_DEV void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
SF_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
SF_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
SF_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem desc] * B[smem desc]^T, kind::f16 (bf16 in, fp32 accumulate)
SF_DEV void umma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
SF_DEV void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// 32 lanes x 32 bit, 16 consecutive columns per thread
SF_DEV void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 lanes x 32 bit, 32 consecutive columns per thread; no wait (pair with tmem_ld_wait)
SF_DEV void tmem_ld32_async(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
SF_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor: K-major tile, 128-byte swizzle, rows of 64 bf16 (128 B),
// 8-row core groups 1024 B apart (SBO), version 1 (sm_100), LBO unused for swizzled K-major.
SF_DEV uint64_t sw128_kmajor_desc(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                 // LBO (ignored)
  d |= (uint64_t)(1024 >> 4) << 32;       // SBO
  d |= (uint64_t)1 << 46;                 // version
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}
// Instruction descriptor, kind::f16: D=f32, A=B=bf16, both K-major, shape M x N.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int M, int N) {
  return (1u << 4)              // c_format = F32
         | (1u << 7)            // a_format = BF16
         | (1u << 10)           // b_format = BF16
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

}  // namespace sf
