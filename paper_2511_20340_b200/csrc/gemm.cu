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
// Work groups: CG = 1 (one CTA, M = 128 weight rows per MMA) or CG = 2 (a cluster pair issuing
// tcgen05.mma.cta_group::2, M = 256: each CTA stages its own 128 weight rows and HALF of the
// activation tile; the leader CTA issues every MMA, commits multicast to both CTAs). G work groups
// (a function of (N, K) only) split the (256/128-row tile, 64-wide k-block) units of the whole GEMM
// into G contiguous equal ranges, so every SM streams the same number of weight bytes (no wave
// quantisation). A tile cut between groups is finished by the group owning its k = 0 segment,
// which adds the other segments' fp32 partials in k order: segment boundaries depend only on
// (N, K, G) -> the same rounding for every T (batch invariance, reading C23).
// Warps: 0 = TMA producer, 1 = MMA issuer (leader CTA), 2 = TMEM allocator, 4..7 = epilogue.
// Two TMEM accumulator buffers (when they fit) overlap the epilogue of one segment with the MMAs
// of the next.
// Stream-K partition with a tile-entry cost. Group g of G owns the units [sk_begin(g), sk_begin(g+1))
// of the n_tiles x kb (tile, k-block) sequence. Every tile is preceded by `drain` virtual units --
// the MMA stall a group pays when its range enters a new tile after finishing another one (the
// accumulator's epilogue must drain TMEM first; one TMEM buffer at T > 256) -- and the virtual
// sequence is cut evenly, so a range that crosses a tile boundary gets fewer real units. The cut
// depends on (n_tiles, kb, G, drain) only: the same k segmentation at every T (batch invariance).
// (32-bit arithmetic: n_tiles (kb + drain) G < 2^31 for every supported shape, checked at launch)
__host__ __device__ inline int sk_real(int v, int kb, int drain) {
  const int t = v / (kb + drain), o = v - t * (kb + drain);
  return t * kb + (o > drain ? o - drain : 0);
}
__host__ __device__ inline int sk_begin(int g, int G, int n_tiles, int kb, int drain) {
  const int V = n_tiles * (kb + drain);
  return sk_real(V * g / G, kb, drain);
}
// the group whose (non-empty) range holds unit u: the largest g with sk_begin(g) <= u
__host__ __device__ inline int sk_group_of(int u, int G, int n_tiles, int kb, int drain) {
  const int V = n_tiles * (kb + drain);
  const int t = u / kb;
  const int v = t * (kb + drain) + drain + (u - t * kb);
  return ((v + 1) * G + V - 1) / V - 1;
}
static bool sk_fits(int G, int n_tiles, int kb, int drain) {
  return (long long)n_tiles * (kb + drain) * (G + 1) + G < (1ll << 31);
}
// Measured on the 7B shapes (profiles/r01/drain_sweep.txt): the entry cost pays off where the
// epilogue of a piece is a plain fp32 publish or a SwiGLU tile (EPI_PARTIAL, EPI_SWIGLU_ACT: -3..-5 us
// per launch at T = 320, +0.5 us at T = 5); for the fixup-heavy ACT / F32 / QKV launches it does not.
// Depends on the epilogue mode only, never on T.
static int sk_drain(int mode) {
  static const int d = getenv("SF_GEMM_DRAIN") ? std::max(0, atoi(getenv("SF_GEMM_DRAIN"))) : 8;
  return (mode == EPI_PARTIAL || mode == EPI_SWIGLU_ACT) ? d : 0;
}

struct SkParams {
  int T, N, K;
  int Tp;  // T rounded up to 32 (row stride of the fixup partial slots)
  int NT, n_sub, stages, kb_total, n_tiles, G, nbuf, w_tiled, w_tma, stage_ok, bulk_ok, npre;
  int cgrp;  // ring slots released per tcgen05.commit
  int probe;  // measurement only (SF_GEMM_PROBE=1): the producer loads nothing
  // three-slot accumulator rotation (two sub-tiles of NT <= 170 columns, one accumulator's worth of
  // TMEM left over): piece g's sub-tile h lives in slot (2 g + h) % 3, so the next piece's MMA waits
  // only for the first half of this piece's drain instead of all of it
  int rot;
  int drain; // tile-entry cost of the stream-K partition (sk_begin)
  int park;  // park mid-range full tiles (T >= 64) for the final phase
  // chain (gate/up -> down in one launch, CHAIN instantiation): phase B's k-blocks, tiles, drain,
  // its partial slots, per-k-block readiness flags of phase A's output and the launch's done counter
  int kbB, n_tilesB, drainB;
  float* partialB;
  int* readyB;
  int* doneB;
  uint32_t tmem_cols;
  const __nv_bfloat16* w_tiles;  // tile-contiguous weights (w_tiled, CG == 1 bulk path)
  GemmEpi epi;
  float* partial;  // [CTAs][T][128]
  int* flags;      // [CTAs]
  unsigned long long* trace;  // optional per-CTA timeline (SF_GEMM_TRACE=1, tools only): [CTA][64]
};

SF_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// trace slots: 0 start, 1 setup done, 2 producer first issue, 3 MMA first full, 4 MMA last issue,
// 5 epilogue done, 6 parked tile done, 8 + 4 s + {0 MMA seg start, 1 MMA seg issued, 2 epi seg ready,
// 3 epi seg done} (s < 4), 24 + i: MMA full-barrier pass of unit i (i < 40), 64 + i: producer issue of
// unit i, final phase 104 flags / 105 fixup loaded / 106 + 2c, 107 + 2c chunk c added / stored,
// 114 + 4c TMEM loaded, 116 + 4c staged (c < 2), small-T head 122 flags / 123 fixed up / 124 stored,
// setup 125 barriers initialised / 126 TMEM allocated / 127 CTA barrier (tools/gemm_trace_step.py)
#define SF_TR(i) \
  do {           \
    if (p.trace) p.trace[(size_t)blockIdx.x * 128 + (i)] = gtimer(); \
  } while (0)

SF_DEV void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
SF_DEV int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
SF_DEV void st_release(int* p, int v) { asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
SF_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
SF_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the mbarrier at the same shared offset in CTA `rank` of the cluster
SF_DEV void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
      "r"(rank)
      : "memory");
}
// 2-SM TMA: data lands in this CTA's smem, transaction bytes are credited to the LEADER's barrier
SF_DEV void tma_load_2d_2sm(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
SF_DEV void umma_bf16_2sm(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
SF_DEV void umma_commit_2sm(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// SwiGLU over a lane pair's 32 tokens of one feature: lane 2i holds gate_i, lane 2i+1 up_i (row-
// interleaved weight). emit(token, y) is called for tokens < nq. Above 16 tokens the pair splits the
// work after one exchange (even lane: tokens 0..15, odd lane: 16..31), so each lane evaluates 16
// SiLUs instead of 32 -- MUFU-bound at T = 320 -- with the same per-element arithmetic
// y = g / (1 + e^-g) * u either way (the same bits).
template <typename Emit>
SF_DEV void swiglu_pair(const float (&v)[32], int nq, int lane, Emit emit) {
  const bool odd = lane & 1;
  if (nq > 16) {
    float x[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = __shfl_xor_sync(0xffffffffu, odd ? v[j] : v[16 + j], 1);
    const int tb = odd ? 16 : 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float g = odd ? x[j] : v[j];
      const float u = odd ? v[16 + j] : x[j];
      const float y = __fdividef(g, 1.f + __expf(-g)) * u;
      if (tb + j < nq) emit(tb + j, y);
    }
    return;
  }
#pragma unroll
  for (int q0 = 0; q0 < 16; q0 += 8) {
    if (q0 >= nq) break;  // (warp-uniform)
    float uu[8], e[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) uu[j] = __shfl_down_sync(0xffffffffu, v[q0 + j], 1);
#pragma unroll
    for (int j = 0; j < 8; ++j) e[j] = __expf(-v[q0 + j]);
#pragma unroll
    for (int j = 0; j < 8; ++j) e[j] = __fdividef(v[q0 + j], 1.f + e[j]) * uu[j];
    if (!odd) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (q0 + j < nq) emit(q0 + j, e[j]);
    }
  }
}

// MODE = the epilogue (EpiMode), a template parameter so each instantiation carries only its own
// store path: the kernel's code is executed cold once per CTA in the final phase, and every
// instruction-cache line it does not need is a fetch that competes with the weight stream.
template <int CG, int MODE, bool CHAIN = false>
__global__ void __launch_bounds__(384, 1)
gemm_sk_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmA,
               const __grid_constant__ CUtensorMap tmWB, const __grid_constant__ CUtensorMap tmAB, const SkParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
  // CG = CTAs per cluster: 1, or 2 = one CTA pair (cta_group::2 MMA, M = 256)
  static_assert(CG == 1 || CG == 2, "CTA groups of 1 or 2");
  constexpr bool kPair = CG == 2;
  const int a_rows = kPair ? p.NT / 2 : p.NT;  // activation rows of each sub-tile in this CTA's smem
  const int a_bytes = p.n_sub * a_rows * BK * 2;
  const int stage_bytes = BM * BK * 2 + a_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)p.stages * stage_bytes);
  uint64_t* empty = full + p.stages;
  uint64_t* accf = empty + p.stages;  // [2]
  uint64_t* acce = accf + 2;          // [2]
  uint64_t* fixb = acce + 2;           // bulk fixup loads (last-segment heads)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + 3);
  uint64_t* sempty = acce + 5;          // [3] (rot) slot released by both CTAs' 8 epilogue warps
  
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = kPair ? cluster_rank() : 0u;
  const uint32_t prank = rank & 1u, pbase = rank & ~1u;  // position in the CTA pair, pair leader rank
  const int c = blockIdx.x / CG;       // work group
  const int slot = blockIdx.x;         // partial / flag slot of this CTA
  const int kb = p.kb_total;
  const long long u0 = sk_begin(c, p.G, p.n_tiles, kb, p.drain), u1 = sk_begin(c + 1, p.G, p.n_tiles, kb, p.drain);
  const int cols = p.n_sub * p.NT;
  // the range's segments: its pieces of consecutive 128-row tiles, in k order
  const int t_first = (int)(u0 / kb);
  const int nseg = u1 > u0 ? (int)((u1 - 1) / kb) - t_first + 1 : 0;
  auto seg_lo = [=](int i) -> long long { return max(u0, (long long)(t_first + i) * kb); };
  auto seg_hi = [=](int i) -> long long { return min(u1, (long long)(t_first + i + 1) * kb); };
  // CHAIN: phase B (the down projection) -- this group's range of its own (tile, k-block) units
  const int kbB = CHAIN ? p.kbB : 1;
  const long long u0B = CHAIN ? sk_begin(c, p.G, p.n_tilesB, kbB, p.drainB) : 0;
  const long long u1B = CHAIN ? sk_begin(c + 1, p.G, p.n_tilesB, kbB, p.drainB) : 0;
  const int tB_first = (int)(u0B / kbB);
  const int nsegB = u1B > u0B ? (int)((u1B - 1) / kbB) - tB_first + 1 : 0;
  auto segB_lo = [=](int i) -> long long { return max(u0B, (long long)(tB_first + i) * kbB); };
  auto segB_hi = [=](int i) -> long long { return min(u1B, (long long)(tB_first + i + 1) * kbB); };
  if (threadIdx.x == 0) SF_TR(0);
  KtScope kt_(KT_GEMM, (uint32_t)p.N | ((uint32_t)min(kb, 511) << 15), 128);  // param: N | (K / 64) << 15

  if (threadIdx.x == 0) {
    if (!(CG == 1 && p.w_tiled && !p.w_tma)) prefetch_tmap(&tmW);
    prefetch_tmap(&tmA);
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);  // pair leader: one arrive_expect_tx covering both CTAs' bytes
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], kPair ? 2 : 1);  // pair leader: both CTAs' epilogues release the accumulator
    }
    mbar_init(fixb, 1);
    for (int x = 0; x < 3; ++x) mbar_init(&sempty[x], kPair ? 16 : 8);
    fence_barrier_init();
    SF_TR(125);
  }
  if (warp == 2) {
    if constexpr (kPair) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(p.tmem_cols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      tmem_alloc(tmem_slot, p.tmem_cols);
    }
    if (lane == 0) SF_TR(126);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) SF_TR(127);
  if constexpr (kPair) cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) SF_TR(1);

  if (warp == 0) {
    // ---- TMA producer warp (converged; one elected lane issues)
    // The weights do not depend on the previous kernel: the first ring's worth of weight tiles is
    // requested before the grid dependency resolves (PDL), the activation tiles after it.
    const long long npre = (p.w_tiled && !p.probe) ? min((long long)p.npre, u1 - u0) : 0;
    if (npre > 0 && elect_one()) {
      int si = 0;
      long long up = seg_lo(0);
      for (int i = 0; i < (int)npre; ++i) {
        if (up == seg_hi(si)) up = seg_lo(++si);
        const int tp = (int)(up / kb), kp = (int)(up % kb);
        ++up;
        uint8_t* st = smem + (size_t)i * stage_bytes;
        if constexpr (CG == 1) {
          mbar_arrive_expect_tx(&full[i], (uint32_t)stage_bytes);
          if (p.w_tma)
            tma_load_2d(st, &tmW, &full[i], 0, (tp * kb + kp) * BM, kEvictFirst);
          else
            bulk_load(st, p.w_tiles + ((size_t)tp * kb + kp) * (BM * BK), BM * BK * 2, &full[i], kEvictFirst);
        } else {
          // the leader arms the barrier for both CTAs' bytes; a fresh phase cannot complete before
          // that arrival, so the peer's bytes may land first
          if (prank == 0) mbar_arrive_expect_tx(&full[i], (uint32_t)(2 * stage_bytes));
          tma_load_2d_2sm(st, &tmW, &full[i], 0, ((tp * CG + (int)rank) * kb + kp) * BM, kEvictFirst);
        }
      }
    }
    __syncwarp();
    pdl_wait();
    pdl_trigger();
    int s = 0, grp_last = p.cgrp - 1;  // ring slot and the last slot of its release group
    uint32_t ph = 0;
    long long j = 0;  // units issued
    for (int si = 0; si < nseg; ++si)
    for (int t = t_first + si, k = (int)(seg_lo(si) - (long long)t * kb), ke = (int)(seg_hi(si) - (long long)t * kb);
         k < ke; ++k, ++j) {
      const bool pre = j < npre;  // weights already requested, slot known free
      if (!pre) mbar_wait(&empty[grp_last], ph ^ 1u);  // slot group released
      if (j == 0 && lane == 0) SF_TR(2);
      if (lane == 0 && j < 40) SF_TR(64 + (int)j);
      if (p.probe) {  // (SF_GEMM_PROBE, measurement only: no loads, the MMA runs on stale tiles)
        if (prank == 0 && elect_one()) mbar_arrive(&full[s]);
      } else if (elect_one()) {
        uint8_t* st = smem + (size_t)s * stage_bytes;
        if constexpr (CG == 1) {
          if (!pre) {
            mbar_arrive_expect_tx(&full[s], (uint32_t)stage_bytes);
            if (p.w_tiled && p.w_tma)  // tiled weights through a 2-D TMA box
              tma_load_2d(st, &tmW, &full[s], 0, (t * kb + k) * BM, kEvictFirst);
            else if (p.w_tiled)  // tile-contiguous, pre-swizzled weights: one 16 KB bulk copy per stage
              bulk_load(st, p.w_tiles + ((size_t)t * kb + k) * (BM * BK), BM * BK * 2, &full[s], kEvictFirst);
            else
              tma_load_2d(st, &tmW, &full[s], k * BK, t * BM, kEvictFirst);
          }
          for (int j = 0; j < p.n_sub; ++j)
            tma_load_2d(st + BM * BK * 2 + j * a_rows * BK * 2, &tmA, &full[s], k * BK, j * p.NT, kEvictLast);
        } else {
          if (!pre) {
            if (prank == 0) mbar_arrive_expect_tx(&full[s], (uint32_t)(2 * stage_bytes));
            // tiled weights viewed as a [blocks*128, 64] tensor: this CTA's 128-row tile of unit tile t
            tma_load_2d_2sm(st, &tmW, &full[s], 0, ((t * CG + (int)rank) * kb + k) * BM, kEvictFirst);
          }
          for (int j = 0; j < p.n_sub; ++j)
            tma_load_2d_2sm(st + BM * BK * 2 + j * a_rows * BK * 2, &tmA, &full[s], k * BK,
                            j * p.NT + (int)rank * a_rows, kEvictLast);
          // no arrival from the peer: its bytes complete_tx on the leader's barrier, which the leader
          // armed for both CTAs; they cannot land before that phase (the slot was released first)
        }
      }
      __syncwarp();
      if (++s == p.stages) {
        s = 0;
        ph ^= 1u;
      }
      if (s > grp_last) grp_last += p.cgrp;
      if (s == 0) grp_last = p.cgrp - 1;
    }
    if constexpr (CHAIN) {
      // phase B: its weights stream into the ring as phase A's last stages free up; activation
      // k-block k = features [64 k, 64 k + 64) of phase A's output, loaded once the CTA that writes
      // them has published it
      for (int si = 0; si < nsegB; ++si)
      for (int t = tB_first + si, k = (int)(segB_lo(si) - (long long)t * kbB), ke = (int)(segB_hi(si) - (long long)t * kbB);
           k < ke; ++k, ++j) {
        mbar_wait(&empty[grp_last], ph ^ 1u);
        if (elect_one()) {
          uint8_t* st = smem + (size_t)s * stage_bytes;
          if (prank == 0) mbar_arrive_expect_tx(&full[s], (uint32_t)(2 * stage_bytes));
          tma_load_2d_2sm(st, &tmWB, &full[s], 0, ((t * CG + (int)rank) * kbB + k) * BM, kEvictFirst);
          while (ld_acquire(&p.readyB[k]) == 0) {
          }
          fence_proxy_async_global();  // phase A's generic stores -> this TMA read
          for (int jj = 0; jj < p.n_sub; ++jj)
            tma_load_2d_2sm(st + BM * BK * 2 + jj * a_rows * BK * 2, &tmAB, &full[s], k * BK,
                            jj * p.NT + (int)rank * a_rows, kEvictLast);
        }
        __syncwarp();
        if (++s == p.stages) {
          s = 0;
          ph ^= 1u;
        }
        if (s > grp_last) grp_last += p.cgrp;
        if (s == 0) grp_last = p.cgrp - 1;
      }
    }
    if (p.epi.pf && p.epi.pf_bytes >= 16 * gridDim.x && elect_one()) {
      // this CTA's slice of the next GEMM's weights -> L2, while the last stages drain and the
      // epilogue runs (the DRAM would otherwise idle through the tail)
      const size_t per = (p.epi.pf_bytes / gridDim.x) & ~(size_t)15;
      const char* base = reinterpret_cast<const char*>(p.epi.pf) + per * blockIdx.x;
      for (size_t off = 0; off < per; off += 65536)
        prefetch_l2(base + off, (uint32_t)std::min<size_t>(65536, per - off), kEvictLast);
    }
    __syncwarp();
  } else if (warp == 1 && prank == 0) {
    // ---- MMA warp (converged; one elected lane issues every tcgen05 op so commits track them)
    const uint32_t idesc = idesc_bf16_f32(kPair ? 2 * BM : BM, p.NT);
    const uint32_t a_off = (uint32_t)(BM * BK * 2) >> 4;           // B-operand tile offset (16 B units)
    const uint32_t sub_off = (uint32_t)(a_rows * BK * 2) >> 4;     // between activation sub-tiles
    const bool two_sub = p.n_sub == 2;                              // (n_sub <= 2: T <= 512 per launch)
    int s = 0, gcnt = 0;
    uint32_t ph = 0;
    long long j = 0;  // units consumed
    for (int seg = 0; seg < nseg + nsegB; ++seg) {  // (phase B segments follow, CHAIN)
      const long long u = seg < nseg ? seg_lo(seg) : segB_lo(seg - nseg);
      const long long se = seg < nseg ? seg_hi(seg) : segB_hi(seg - nseg);
      const int b = seg % p.nbuf;
      if (!p.rot) {
        mbar_wait(&acce[b], ((uint32_t)(seg / p.nbuf) & 1u) ^ 1u);
        tc_fence_after();
      }
      if (lane == 0 && seg < 4) SF_TR(8 + 4 * seg);
      const uint32_t dacc = tmem + (uint32_t)(b * cols), dacc1 = dacc + (uint32_t)p.NT;
      // (rot) half-piece n = 2 seg + h -> slot n % 3; its previous use n - 3 must be drained
      const int n0 = 2 * seg;
      const uint32_t r0 = tmem + (uint32_t)((n0 % 3) * p.NT), r1 = tmem + (uint32_t)(((n0 + 1) % 3) * p.NT);
      for (long long uu = u; uu < se; ++uu) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (lane == 0) {
          if (j == 0) SF_TR(3);
          if (j < 40) SF_TR(24 + (int)j);
        }
        ++j;
        if (kPair && p.rot) {
          const uint64_t dw = sw128_kmajor_desc(smem_u32(smem + (size_t)s * stage_bytes));
          const uint64_t da = dw + a_off;
          const uint32_t acc0 = uu > u ? 1u : 0u;
          if (uu == u) {
            mbar_wait(&sempty[n0 % 3], ((uint32_t)(n0 / 3) & 1u) ^ 1u);
            tc_fence_after();
          }
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
              umma_bf16_2sm(r0, dw + (uint64_t)(kk * 2), da + (uint64_t)(kk * 2), idesc, kk > 0 ? 1u : acc0);
          }
          __syncwarp();
          if (uu == u) {
            mbar_wait(&sempty[(n0 + 1) % 3], ((uint32_t)((n0 + 1) / 3) & 1u) ^ 1u);
            tc_fence_after();
          }
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
              umma_bf16_2sm(r1, dw + (uint64_t)(kk * 2), da + (uint64_t)(sub_off + kk * 2), idesc, kk > 0 ? 1u : acc0);
            if (++gcnt == p.cgrp) umma_commit_2sm(&empty[s], (uint16_t)(3u << pbase));
          }
        } else if (elect_one()) {
          // fully unrolled over (k step, sub-tile) with the operands formed once per stage: a runtime
          // sub-tile loop costs more issue time per MMA than the tensor pipe needs at N <= 160
          const uint64_t dw = sw128_kmajor_desc(smem_u32(smem + (size_t)s * stage_bytes));
          const uint64_t da = dw + a_off;
          const uint32_t acc0 = uu > u ? 1u : 0u;
          auto issue = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
            if constexpr (CG == 1) umma_bf16(d, a, b, idesc, acc);
            else umma_bf16_2sm(d, a, b, idesc, acc);
          };
          if (two_sub) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              issue(dacc, dw + (uint64_t)(kk * 2), da + (uint64_t)(kk * 2), kk > 0 ? 1u : acc0);
              issue(dacc1, dw + (uint64_t)(kk * 2), da + (uint64_t)(sub_off + kk * 2), kk > 0 ? 1u : acc0);
            }
          } else {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
              issue(dacc, dw + (uint64_t)(kk * 2), da + (uint64_t)(kk * 2), kk > 0 ? 1u : acc0);
          }
          if (++gcnt == p.cgrp) {  // frees slots s-cgrp+1..s (in both CTAs of a pair)
            if constexpr (CG == 1) umma_commit(&empty[s]);
            else umma_commit_2sm(&empty[s], (uint16_t)(3u << pbase));
          }
        }
        __syncwarp();
        if (gcnt == p.cgrp) gcnt = 0;
        if (++s == p.stages) {
          s = 0;
          ph ^= 1u;
        }
      }
      if (elect_one()) {
        if constexpr (CG == 1) umma_commit(&accf[b]);
        else umma_commit_2sm(&accf[b], (uint16_t)(3u << pbase));
      }
      __syncwarp();
      if (lane == 0) {
        if (seg < 4) SF_TR(8 + 4 * seg + 1);
        if (seg == nseg + nsegB - 1) SF_TR(4);
      }
    }
  }
  {
    // ---- epilogue (named barriers: 1 = the 8 loop warps, 5 = all 12 in the final phase, 2..4 = the
    // final phase's three groups). Segments before the last: warps 4..11 (two groups of 4 = one warp per TMEM
    // lane quadrant each, warp w reads lanes 32 (w % 4) ..), alternate 32-column chunks, while the
    // MMA streams the next segment. The last segment and a parked full tile ("final phase"): all 12
    // warps (warps 0..3 are done producing / issuing by then) in three groups.
    if (warp >= 4) pdl_wait();  // outputs / partial slots / flags may still be in use by the previous kernel
    if (warp >= 4) kt_.mark();
    uint32_t fix_ph = 0;
    const int quad = warp & 3;
    const int m = quad * 32 + lane;
    const bool lead = threadIdx.x == 128;  // first epilogue thread: flags, barriers' single-thread work
    constexpr int mode = MODE;
    const size_t ldo = (size_t)p.epi.ldo;
    // the output base (a device-selected exchange slot for the fused TP all-reduce; read when storing,
    // after this thread's grid-dependency wait: the selecting counter is written two launches earlier)
    auto eout = [&]() -> uint8_t* {
      uint8_t* o = reinterpret_cast<uint8_t*>(p.epi.out);
      if (p.epi.out_sel)
        o += (size_t)((*(volatile const int*)p.epi.out_sel + 1) & 1) * (size_t)p.epi.out_sel_stride * 2;
      return o;
    };
    // smem ring reuse once every MMA of the CTA has completed (final phase): partial staging
    // [0, ring - 48 KB) and three 16 KB output staging buffers at the end
    constexpr int kStageBytes = 16384;
    const int ring_bytes = p.stages * stage_bytes;
    const int out_elt = mode == EPI_STORE_F32 ? 4 : 2;
    constexpr bool kStageable =
        MODE == EPI_STORE_ACT || MODE == EPI_STORE_F32 || MODE == EPI_SWIGLU_ACT || MODE == EPI_QKV_ROPE;
    const bool can_stage = kStageable && p.stage_ok &&
                           (ldo * out_elt) % 16 == 0 && ring_bytes >= 3 * kStageBytes + 64 * BM * 4;
    const int fix_bytes = can_stage ? ring_bytes - 3 * kStageBytes : ring_bytes;
    uint8_t* stg = smem + ring_bytes - 3 * kStageBytes;
    const float* smf = reinterpret_cast<const float*>(smem);
    float* const slot_base = p.partial + (size_t)slot * p.Tp * BM;                    // published tail
    float* const defer_base = p.partial + (size_t)(p.G * CG + slot) * p.Tp * BM;  // parked full tile

    // EPI_QKV_ROPE: destination row (128 bf16) of token t for head tile vt_: q heads -> q_out,
    // k / v heads -> the token's page slot
    auto rope_dst_row = [&](int tl, int vt_) -> __nv_bfloat16* {
      const RopeEpi& R = p.epi.rope;
      const int t = tl + R.t0;
      const int b = t / R.q_len, pos = R.pos0[b] + t % R.q_len;
      if (vt_ < R.Hq) return reinterpret_cast<__nv_bfloat16*>(R.q_out) + ((size_t)t * R.Hq + vt_) * 128;
      const bool isk = vt_ < R.Hq + R.Hkv;
      const int kvh = isk ? vt_ - R.Hq : vt_ - R.Hq - R.Hkv;
      const int blk = R.bt[b * R.pps + pos / 16];
      return reinterpret_cast<__nv_bfloat16*>(isk ? R.Kp : R.Vp) + (((size_t)blk * R.Hkv + kvh) * 16 + pos % 16) * 128;
    };
    // RoPE on this thread's (dim, token) values: lane pair (2i, 2i+1) holds dims (i, i + 64) of the head
    // (pair-interleaved weight rows). The accumulator is rounded to bf16 first -- exactly the values
    // the unfused path (bf16 QKV output, then the RoPE kernel) rotates -- so both paths give the same
    // bits. Lane l resolves token c0 + l's position and destination row once; emit(q, dim, y, row).
    // (small T) token c0 + lane's position and destination row for tile vt_, resolved while the MMA
    // still runs, and the RoPE table lines of the chunk's tokens pulled into L1: the epilogue then
    // starts from the accumulator instead of a pos -> page table -> table chain of L2 round trips
    int pre_pos = 0, pre_c0 = -1, pre_vt = -1;
    unsigned long long pre_row = 0;
    auto rope_prefetch = [&](int c0, int vt_) {
      const RopeEpi& R = p.epi.rope;
      const int nq = min(32, p.T - c0);
      pre_c0 = c0;
      pre_vt = vt_;
      if (lane < nq) {
        const int t = c0 + lane + R.t0;
        pre_pos = R.pos0[t / R.q_len] + t % R.q_len;
        pre_row = reinterpret_cast<unsigned long long>(rope_dst_row(c0 + lane, vt_));
      }
      if (vt_ < R.Hq + R.Hkv)
        for (int q = 0; q < nq; ++q) {
          const int pq = __shfl_sync(0xffffffffu, pre_pos, q);
          asm volatile("prefetch.global.L1 [%0];" ::"l"(R.table + (size_t)pq * 64 + (m >> 1)));
        }
    };
    auto rope_rows = [&](float (&v)[32], int c0, int nq, int vt_, auto emit) {
      const RopeEpi& R = p.epi.rope;
      const bool odd = lane & 1;
      const int i = m >> 1, dim = odd ? 64 + i : i;
      const bool rot = vt_ < R.Hq + R.Hkv;
      int my_pos = pre_pos;
      unsigned long long my_row = pre_row;
      if (lane < nq && (c0 != pre_c0 || vt_ != pre_vt)) {
        const int t = c0 + lane + R.t0;
        my_pos = R.pos0[t / R.q_len] + t % R.q_len;
        my_row = reinterpret_cast<unsigned long long>(rope_dst_row(c0 + lane, vt_));
      }
#pragma unroll 8
      for (int q = 0; q < 32; ++q) {
        if (q >= nq) break;  // (warp-uniform)
        const int pos = __shfl_sync(0xffffffffu, my_pos, q);
        const unsigned long long row = __shfl_sync(0xffffffffu, my_row, q);
        const float x = __bfloat162float(__float2bfloat16_rn(v[q]));
        const float xo = __shfl_xor_sync(0xffffffffu, x, 1);
        float y = x;
        if (rot) {
          const float2 cs = R.table[(size_t)pos * 64 + i];
          y = odd ? rope_y2(xo, x, cs.x, cs.y) : rope_y1(x, xo, cs.x, cs.y);
        }
        emit(q, dim, y, reinterpret_cast<__nv_bfloat16*>(row));
      }
    };
    // one 32-token chunk of this thread's row m: stage [32 tokens][tile columns] in smem, then
    // write whole rows with 16-byte vectors (per-thread column stores would be 32-byte sectors
    // 10-100 KB apart)
    // (EPI_STORE_F32 + amax) the best (logit, id) key of each of the 32 tokens over this warp's 32
    // rows: a butterfly reduce-scatter (31 exchanges) leaves token c0 + lane's key in lane `lane`
    auto amax_keys = [&](const float (&v)[32], int c0, int nq, int vt_) {
      const unsigned id = p.epi.amax_v0 + (unsigned)(vt_ * BM + m);
      unsigned long long k[32];
      bool bad = false;
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const float x = v[q] == 0.f ? 0.f : v[q];  // -0 -> +0
        bad |= (q < nq) && !isfinite(x);
        unsigned u = __float_as_uint(x);
        u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
        k[q] = (q < nq) ? (((unsigned long long)u << 32) | (0xFFFFFFFFu - id)) : 0ull;
      }
#pragma unroll
      for (int s = 16; s >= 1; s >>= 1) {
        const bool up = (lane & s) != 0;
#pragma unroll
        for (int j = 0; j < s; ++j) {
          const unsigned long long keep = up ? k[j + s] : k[j];
          const unsigned long long r = __shfl_xor_sync(0xffffffffu, up ? k[j] : k[j + s], s);
          k[j] = keep > r ? keep : r;
        }
      }
      if (lane < nq) atomicMax(p.epi.amax + c0 + lane, k[0]);
      if (bad && p.epi.amax_err) atomicOr(p.epi.amax_err, 1);
    };
    auto staged_store = [&](float (&v)[32], int c0, int nq, int vt_, int gid) {
      if constexpr (MODE == EPI_STORE_F32) {
        if (p.epi.amax) {
          amax_keys(v, c0, nq, vt_);
          if (!p.epi.out) return;  // (uniform over the CTA)
        }
      }
      uint8_t* sb = stg + (size_t)gid * kStageBytes;
      const int rowb = mode == EPI_SWIGLU_ACT ? 128 : ((mode == EPI_STORE_ACT || mode == EPI_QKV_ROPE) ? 256 : 512);
      if constexpr (MODE == EPI_QKV_ROPE) {
        // rows: [32][256 B] values, then the 32 destination row pointers (8 KB + 256 B < 16 KB)
        unsigned long long* rows = reinterpret_cast<unsigned long long*>(sb + 32 * 256);
        rope_rows(v, c0, nq, vt_, [&](int q, int dim, float y, __nv_bfloat16* row) {
          reinterpret_cast<__nv_bfloat16*>(sb + q * 256)[dim] = __float2bfloat16_rn(y);
          if (m == 0) rows[q] = reinterpret_cast<unsigned long long>(row);
        });
        named_sync(2 + gid, 128);
        const int ht = quad * 32 + lane;
        for (int i = ht; i < nq * 16; i += 128) {
          const int q = i >> 4, x = i & 15;
          *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(rows[q]) + x * 8) =
              *reinterpret_cast<const uint4*>(sb + q * 256 + x * 16);
        }
        named_sync(2 + gid, 128);
        return;
      }
      if (mode == EPI_STORE_ACT) {
#pragma unroll
        for (int q = 0; q < 32; ++q) reinterpret_cast<__nv_bfloat16*>(sb + q * 256)[m] = __float2bfloat16_rn(v[q]);
      } else if (mode == EPI_STORE_F32) {
#pragma unroll
        for (int q = 0; q < 32; ++q) reinterpret_cast<float*>(sb + q * 512)[m] = v[q];
      } else {
        // lane 2i holds gate_i, lane 2i+1 up_i (row-interleaved weight): the even lane forms the 32
        // tokens of feature i, in batches of 8 independent shuffle / exp / divide chains
        __nv_bfloat16* srow = reinterpret_cast<__nv_bfloat16*>(sb) + quad * 16 + (lane >> 1);
        swiglu_pair(v, nq, lane, [&](int q, float y) { srow[q * 64] = __float2bfloat16_rn(y); });
      }
      named_sync(2 + gid, 128);
      if (lead && c0 < 2 * 96) SF_TR(116 + 4 * (c0 / 96));  // staged in smem
      const int col0 = mode == EPI_SWIGLU_ACT ? vt_ * 64 : vt_ * BM;
      uint8_t* gbase = eout() + ((size_t)c0 * ldo + col0) * out_elt;
      const int vpr = rowb / 16, ht = quad * 32 + lane;
      for (int i = ht; i < nq * vpr; i += 128) {
        const int q = i / vpr, x = i % vpr;
        *reinterpret_cast<uint4*>(gbase + (size_t)q * ldo * out_elt + x * 16) =
            *reinterpret_cast<const uint4*>(sb + q * rowb + x * 16);
      }
      named_sync(2 + gid, 128);
    };
    // per-thread column stores (segments that end while the ring is still streaming)
    auto direct_store = [&](float (&v)[32], int c0, int nq, int vt_) {
      if constexpr (MODE == EPI_QKV_ROPE) {
        rope_rows(v, c0, nq, vt_, [&](int q, int dim, float y, __nv_bfloat16* row) { row[dim] = __float2bfloat16_rn(y); });
        return;
      }
      if constexpr (MODE == EPI_STORE_F32) {
        if (p.epi.amax) {
          amax_keys(v, c0, nq, vt_);
          if (!p.epi.out) return;
        }
      }
      const int n = vt_ * BM + m;
      if (mode == EPI_STORE_ACT) {
        __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(eout()) + (size_t)c0 * ldo + n;
#pragma unroll
        for (int q = 0; q < 32; ++q)
          if (q < nq) o[q * ldo] = __float2bfloat16_rn(v[q]);
      } else if (mode == EPI_STORE_F32) {
        float* o = reinterpret_cast<float*>(p.epi.out) + (size_t)c0 * ldo + n;
#pragma unroll
        for (int q = 0; q < 32; ++q)
          if (q < nq) o[q * ldo] = v[q];
      } else if (mode == EPI_ADD_F32) {
        float* o = reinterpret_cast<float*>(p.epi.out) + (size_t)c0 * ldo + n;
        float old[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) old[q] = (q < nq) ? o[q * ldo] : 0.f;
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = old[q] + v[q];
#pragma unroll
        for (int q = 0; q < 32; ++q)
          if (q < nq) o[q * ldo] = v[q];
        if (p.epi.tap) {
          float* tp = p.epi.tap + (size_t)c0 * ldo + n;
#pragma unroll
          for (int q = 0; q < 32; ++q)
            if (q < nq) tp[q * ldo] = v[q];
        }
      } else if (mode == EPI_BIAS_F32) {
        float* o = reinterpret_cast<float*>(p.epi.out) + (size_t)c0 * ldo + n;
        const float bias = p.epi.bias[n];
#pragma unroll
        for (int q = 0; q < 32; ++q)
          if (q < nq) o[q * ldo] = v[q] + bias;
      } else {  // SwiGLU (see staged_store)
        const int f = vt_ * 64 + (m >> 1);
        __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.epi.out) + (size_t)c0 * ldo + f;
        swiglu_pair(v, nq, lane, [&](int q, float y) { o[q * ldo] = __float2bfloat16_rn(y); });
      }
    };
    // bulk-copy n_src [rows P0..P1) x 128 fp32 partial slots into the idle ring (one TMA request each)
    auto bulk_rows = [&](const float* const* srcs, int n_src, int P0, int P1) {
      if (lead) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        mbar_arrive_expect_tx(fixb, (uint32_t)(n_src * (P1 - P0) * BM * 4));
        for (int o = 0; o < n_src; ++o)
          bulk_load(smem + (size_t)o * (P1 - P0) * BM * 4, srcs[o] + (size_t)P0 * BM, (uint32_t)((P1 - P0) * BM * 4),
                    fixb, kEvictFirst);
      }
      mbar_wait(fixb, fix_ph);
      fix_ph ^= 1u;
    };

    // (small T, head pieces with one or two partner segments) the partners' partials of this
    // thread's chunk, loaded while the MMA still runs -- see the driver loop
    constexpr int kPreT = 8;  // rows (T <= kPreT: B = 1 verify / draft blocks)
    float pf1[kPreT], pf2[kPreT];
    bool pre_fix = false;

    // Epilogue of segment [u, se) of tile t from TMEM buffer b by ng groups (this thread: group
    // gid, barrier over nthr threads). final: every MMA of the CTA has completed (ring idle).
    // (rot) this warp's TMEM reads of half-piece n = 2 seg + h are complete: release its slot
    auto rot_release = [&](int n) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (prank == 0) mbar_arrive(&sempty[n % 3]);
        else mbar_arrive_remote(&sempty[n % 3], pbase);
      }
    };
    int ep_seg = 0;  // the segment being finished (rot slot mapping)
    auto segment_epilogue = [&](long long u, int t, long long se, int b, int gid, int ng, int nthr, bool final,
                                int& defer_vt, bool phase_b) {
      const int kbs = phase_b ? kbB : kb;
      const long long ts = (long long)t * kbs, te = ts + kbs;
      const uint32_t t_row = tmem + (uint32_t)(b * cols) + ((uint32_t)(quad * 32) << 16);
      // TMEM address of this thread's lane row at token column c0 (a 32-column chunk never straddles
      // the two sub-tiles: NT % 32 == 0 under rot)
      auto taddr = [&](int c0) -> uint32_t {
        if (!p.rot) return t_row + (uint32_t)c0;
        const int h = c0 >= p.NT ? 1 : 0;
        return tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(((2 * ep_seg + h) % 3) * p.NT + c0 - h * p.NT);
      };
      const bool rel = p.rot && !final;  // (rot) release the slots as their columns are read
      const int vt = t * CG + (int)rank;  // 128-row tile index of this CTA's rows
      const bool is_full = (u == ts) && (se == te);
      const bool is_head = (u == ts) && !is_full;
      const int cstep = 32 * ng;
      if (phase_b || mode == EPI_PARTIAL || (!is_full && !is_head) ||
          (is_full && !final && can_stage && p.park && p.T >= 64)) {
        // fp32 accumulator -> [T][128] slot (each warp store is one 128-byte line):
        //  EPI_PARTIAL: slot 2 group + (first segment of the range ? 0 : 1), reduced in k order by
        //    the consumer; tail of a tile owned by another group: this CTA's slot, then its flag;
        //  full tile in mid-range: parked, finished in the final phase instead of stalling the MMA
        //  phase B of a chain: as EPI_PARTIAL, into its own partial slots
        const bool tail = !phase_b && mode != EPI_PARTIAL && !is_full && !is_head;
        float* dst = phase_b ? p.partialB + ((size_t)(2 * c + (u == u0B ? 0 : 1)) * CG + (int)rank) * p.T * BM
                     : mode == EPI_PARTIAL
                         ? p.partial + ((size_t)(2 * c + (u == u0 ? 0 : 1)) * CG + (int)rank) * p.T * BM
                         : (tail ? slot_base : defer_base);
        for (int c0 = gid * 32; c0 < p.T; c0 += cstep) {
          uint32_t r[32];
          tmem_ld32_async(taddr(c0), r);
          tmem_ld_wait();
          if (rel && c0 < p.NT && c0 + cstep >= p.NT) rot_release(2 * ep_seg);  // last sub-tile-0 chunk read
#pragma unroll
          for (int cc = 0; cc < 32; ++cc)
            if (c0 + cc < p.T) dst[(size_t)(c0 + cc) * BM + m] = __uint_as_float(r[cc]);
        }
        if (rel) rot_release(2 * ep_seg + 1);
        if (tail) {
          __threadfence();
          named_sync(final ? 5 : 1, nthr);
          if (lead) st_release(&p.flags[slot], 1);
        }
        if (!phase_b && mode != EPI_PARTIAL && is_full) defer_vt = vt;
        return;
      }
      // head or full tile: add the other groups' k segments of this tile (they publish them first
      // thing), in k order, then the output epilogue
      int c_lo = c + 1, c_hi = c;
      if (is_head) c_hi = sk_group_of((int)(te - 1), p.G, p.n_tiles, kb, p.drain);
      if (is_head && !pre_fix) {
        if (lead)
          for (int cc = c_lo; cc <= c_hi; ++cc)
            while (ld_acquire(&p.flags[cc * CG + (int)rank]) == 0) {
            }
        named_sync(final ? 5 : 1, nthr);
      }
      if (lead && !final) SF_TR(122);  // (small T) partners' partials published
      if (lead && final) SF_TR(104);
      const int n_o = c_hi - c_lo + 1;
      // (small T: a few rows -- direct loads / stores beat the TMA round trip and the staging barriers)
      const bool stage_out = final && can_stage && p.T >= 64;
      const bool bulk = final && p.bulk_ok && p.T >= 64 && n_o > 0 && n_o <= 8 && fix_bytes >= 64 * BM * 4 * n_o;
      const int Tc = bulk ? (fix_bytes / (n_o * BM * 4)) / 64 * 64 : p.T;
      const float* srcs[8];
      for (int o = 0; o < n_o && o < 8; ++o) srcs[o] = p.partial + (size_t)((c_lo + o) * CG + (int)rank) * p.Tp * BM;
      for (int P0 = 0; P0 < p.T; P0 += Tc) {
        const int P1 = min(p.T, P0 + Tc);
        if (bulk) bulk_rows(srcs, n_o, P0, P1);
        if (lead && final && P0 == 0) SF_TR(105);
        for (int c0 = P0 + gid * 32; c0 < P1; c0 += cstep) {
          uint32_t r[32];
          tmem_ld32_async(taddr(c0), r);
          tmem_ld_wait();
          if (lead && final && c0 < 2 * cstep) SF_TR(114 + 4 * (c0 / cstep));  // TMEM loaded
          float v[32];
#pragma unroll
          for (int q = 0; q < 32; ++q) v[q] = __uint_as_float(r[q]);
          if (bulk) {
            for (int o = 0; o < n_o; ++o) {  // fixed k order
              const float* sp = smf + (size_t)o * (P1 - P0) * BM + (size_t)(c0 - P0) * BM + m;
#pragma unroll
              for (int q = 0; q < 32; ++q)
                if (c0 + q < p.T) v[q] += sp[q * BM];
            }
          } else if (pre_fix) {  // fixed k order
#pragma unroll
            for (int q = 0; q < kPreT; ++q) v[q] += pf1[q];
            if (n_o == 2) {
#pragma unroll
              for (int q = 0; q < kPreT; ++q) v[q] += pf2[q];
            }
          } else {
            for (int cc = c_lo; cc <= c_hi; cc += 2) {  // fixed k order; two segments' loads in flight
              const float* s0 = p.partial + (size_t)(cc * CG + (int)rank) * p.Tp * BM + m;
              const bool two = cc + 1 <= c_hi;
              const float* s1 = s0 + (two ? (size_t)CG * p.Tp * BM : 0);
              float a0[32], a1[32];
#pragma unroll
              for (int q = 0; q < 32; ++q) a0[q] = (c0 + q < p.T) ? __ldcg(&s0[(size_t)(c0 + q) * BM]) : 0.f;
              if (two) {
#pragma unroll
                for (int q = 0; q < 32; ++q) a1[q] = (c0 + q < p.T) ? __ldcg(&s1[(size_t)(c0 + q) * BM]) : 0.f;
              }
#pragma unroll
              for (int q = 0; q < 32; ++q) v[q] += a0[q];
              if (two) {
#pragma unroll
                for (int q = 0; q < 32; ++q) v[q] += a1[q];
              }
            }
          }
          const int nq = min(32, p.T - c0);
          if (lead && !final && c0 == 0) SF_TR(123);
          if (lead && final && c0 < 4 * cstep) SF_TR(106 + 2 * (c0 / cstep));  // TMEM + adds done
          if constexpr (kStageable) {
            if (stage_out) staged_store(v, c0, nq, vt, gid);
            else direct_store(v, c0, nq, vt);
          } else {
            direct_store(v, c0, nq, vt);
          }
          if (lead && !final && c0 == 0) SF_TR(124);
          if (lead && final && c0 < 4 * cstep) SF_TR(107 + 2 * (c0 / cstep));  // stored
        }
        if (bulk) named_sync(final ? 5 : 1, nthr);  // smem pass consumed before the next one overwrites it
      }
      if (rel) {  // (not taken by construction under rot: every non-final piece is drained above)
        rot_release(2 * ep_seg);
        rot_release(2 * ep_seg + 1);
      }
      if (is_head) {
        named_sync(final ? 5 : 1, nthr);
        if (lead)
          for (int cc = c_lo; cc <= c_hi; ++cc) p.flags[cc * CG + (int)rank] = 0;  // re-arm for the next launch
      }
      if constexpr (CHAIN) {  // this CTA's output features of tile t are in memory: phase B may load them
        __threadfence();
        named_sync(final ? 5 : 1, nthr);
        if (lead) st_release(&p.readyB[vt], 1);
      }
    };

    // segments of [u0, u1): all but the last by the 8 epilogue warps while the MMA streams on; the
    // last one (and a parked full tile) by all 12 warps -- one inlined copy of the epilogue
    const int nseg_total = nseg + nsegB;
    int defer_vt = -1;
    int gid = 0;
    for (int seg = 0; seg < nseg_total; ++seg) {
      const bool phase_b = seg >= nseg;  // (CHAIN)
      const long long u = phase_b ? segB_lo(seg - nseg) : seg_lo(seg);
      const long long se = phase_b ? segB_hi(seg - nseg) : seg_hi(seg);
      const int t = (int)(u / (phase_b ? kbB : kb));
      // the 12-warp final phase pays off for large T only (small T: a few rows per chunk, the
      // extra barriers would dominate)
      const bool final = seg == nseg_total - 1 && p.T >= 64;
      if (warp >= 4 || final) {
        const int b = seg % p.nbuf;
        int ng = 2, nthr = 256;
        gid = warp >= 4 ? (warp - 4) >> 2 : 0;
        if (final) {
          if (warp < 4) pdl_wait();  // (already resolved: the producer waited before its first load)
          int* s_defer = reinterpret_cast<int*>(tmem_slot + 1);  // share the parked tile index
          if (lead) *s_defer = defer_vt;
          named_sync(5, 384);
          defer_vt = *s_defer;
          ng = 3;
          nthr = 384;
          gid = warp < 4 ? 2 : gid;
        }
        if constexpr (MODE == EPI_QKV_ROPE) {
          const bool out_seg = u == (long long)t * kb;  // head or full tile: this CTA writes the rows
          if (!final && out_seg && gid * 32 < p.T) rope_prefetch(gid * 32, t * CG + (int)rank);
        }
        // small T, a head piece with one or two partner segments: wait for the partners' flags and
        // load their partials of this thread's chunk now, off the critical path after the last MMA
        pre_fix = false;
        if (!phase_b && mode != EPI_PARTIAL && !final && p.T <= kPreT && u == (long long)t * kb &&
            se < (long long)(t + 1) * kb) {
          const int c_hi = sk_group_of(t * kb + kb - 1, p.G, p.n_tiles, kb, p.drain);
          const int n_o = c_hi - c;
          if (n_o >= 1 && n_o <= 2) {
            for (int cc = c + 1; cc <= c_hi; ++cc)
              while (ld_acquire(&p.flags[cc * CG + (int)rank]) == 0) {
              }
            if (gid == 0) {
              const float* s0 = p.partial + (size_t)((c + 1) * CG + (int)rank) * p.Tp * BM + m;
              const float* s1 = s0 + (size_t)CG * p.Tp * BM;
#pragma unroll
              for (int q = 0; q < kPreT; ++q) pf1[q] = q < p.T ? __ldcg(&s0[(size_t)q * BM]) : 0.f;
              if (n_o == 2) {
#pragma unroll
                for (int q = 0; q < kPreT; ++q) pf2[q] = q < p.T ? __ldcg(&s1[(size_t)q * BM]) : 0.f;
              }
            }
            pre_fix = true;
          }
        }
        mbar_wait_sleep(&accf[b], (uint32_t)(seg / p.nbuf) & 1u);
        if (lead && seg < 4) SF_TR(8 + 4 * seg + 2);
        tc_fence_after();
        ep_seg = seg;
        segment_epilogue(u, t, se, b, gid, ng, nthr, final, defer_vt, phase_b);
        if (!final) {
          tc_fence_before();
          named_sync(1, 256);
          if (lead && seg < nseg_total - 1 && !p.rot) {  // (the MMA never waits for the last buffer)
            if (CG == 1 || prank == 0) mbar_arrive(&acce[b]);
            else mbar_arrive_remote(&acce[b], pbase);
          }
        } else {
          named_sync(5, 384);
          if (lead) SF_TR(5);
        }
        if (lead && seg < 4) SF_TR(8 + 4 * seg + 3);
      }
    }
    if constexpr (kStageable) {
      if (defer_vt >= 0) {
        // the parked full tile, through the idle ring
        __threadfence();
        named_sync(5, 384);
        const int Tc = (fix_bytes / (BM * 4)) / 64 * 64;
        const float* src = defer_base;
        for (int P0 = 0; P0 < p.T; P0 += Tc) {
          const int P1 = min(p.T, P0 + Tc);
          bulk_rows(&src, 1, P0, P1);
          for (int c0 = P0 + gid * 32; c0 < P1; c0 += 96) {
            float v[32];
            const float* sp = smf + (size_t)(c0 - P0) * BM + m;
#pragma unroll
            for (int q = 0; q < 32; ++q) v[q] = (c0 + q < p.T) ? sp[q * BM] : 0.f;
            staged_store(v, c0, min(32, p.T - c0), defer_vt, gid);
          }
          named_sync(5, 384);
        }
        if (lead) SF_TR(6);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CHAIN) {
    // the last CTA out re-arms the readiness flags for the next launch (every producer is done with them)
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(p.doneB, 1) == (int)gridDim.x - 1) {
        for (int k = 0; k < p.kbB; ++k) p.readyB[k] = 0;
        *p.doneB = 0;
        __threadfence();
      }
    }
  }
  if constexpr (kPair) cluster_sync();
  tc_fence_after();
  if (warp == 2) {
    if constexpr (kPair)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols) : "memory");
    else
      tmem_dealloc(tmem, p.tmem_cols);
  }
}

// ------------------------------------------------------------------------ SIMT fp32 kernel
// grid (ceil(Nout/32), ceil(T/32)), block (32, 8). Each output element sums k in 32-wide blocks,
// each block in k order, the block sums in k order (fixed for every T: batch-invariant). DUAL:
// SwiGLU over the 64-row interleaved gate/up layout.
template <bool DUAL>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const float* __restrict__ A, int lda,
                                                         const float* __restrict__ W, int T, int N, int K,
                                                         GemmEpi epi) {
  KtScope kt_(KT_GEMM_SIMT, (uint32_t)(N));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  __shared__ float As[32][33];
  __shared__ float Ws[32][33];
  __shared__ float Us[DUAL ? 32 : 1][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int Nout = DUAL ? N / 2 : N;
  const int ob = blockIdx.x * 32, tb = blockIdx.y * 32;
  float acc[4] = {0, 0, 0, 0}, accu[4] = {0, 0, 0, 0};
  auto wrow = [&](int o) { return DUAL ? 2 * o : o; };
  for (int kt = 0; kt < K; kt += 32) {
    for (int i = ty; i < 32; i += 8) {
      const int t = tb + i, kk = kt + tx;
      As[i][tx] = (t < T && kk < K) ? A[(size_t)t * lda + kk] : 0.f;
      const int o = ob + i;
      Ws[i][tx] = (o < Nout && kk < K) ? W[(size_t)wrow(o) * K + kk] : 0.f;
      if (DUAL) Us[i][tx] = (o < Nout && kk < K) ? W[(size_t)(wrow(o) + 1) * K + kk] : 0.f;
    }
    __syncthreads();
    // blocked k order: each 32-wide k block is summed on its own, then added to the running total
    // (rounding error grows with 32 + K/32 terms instead of K; the order depends on K only)
    float blk[4] = {0, 0, 0, 0}, blku[4] = {0, 0, 0, 0};
#pragma unroll 8
    for (int c = 0; c < 32; ++c) {
      const float w = Ws[tx][c];
      const float u = DUAL ? Us[tx][c] : 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float a = As[ty + 8 * i][c];
        blk[i] = fmaf(a, w, blk[i]);
        if (DUAL) blku[i] = fmaf(a, u, blku[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      acc[i] += blk[i];
      if (DUAL) accu[i] += blku[i];
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
  return encode_tmap_cached(g_encode, m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                            box, CU_TENSOR_MAP_SWIZZLE_128B) == CUDA_SUCCESS;
}

// MMA N tiling of T token columns (granularity g = 16)
static void tc_shape(int T, int* NT, int* n_sub, int g = 16) {
  const int Tp = std::max(g, (T + g - 1) / g * g);
  if (Tp <= 256) {
    *NT = Tp;
    *n_sub = 1;
  } else {
    *n_sub = (Tp + 255) / 256;
    *NT = ((Tp + *n_sub - 1) / *n_sub + g - 1) / g * g;
  }
}

constexpr int kMaxSMs = 160;
// Optional per-CTA timeline of the last GEMM launch (SF_GEMM_TRACE=1; tools/gemm_trace.py only).
static unsigned long long* g_trace_buf = nullptr;
static unsigned long long* gemm_trace_buffer() {
  static const bool on = getenv("SF_GEMM_TRACE") && atoi(getenv("SF_GEMM_TRACE")) > 0;
  if (!on) return nullptr;
  if (!g_trace_buf) {
    if (cudaMalloc((void**)&g_trace_buf, (size_t)2 * kMaxSMs * 128 * 8) != cudaSuccess) return nullptr;
    cudaMemset(g_trace_buf, 0, (size_t)2 * kMaxSMs * 128 * 8);
  }
  return g_trace_buf;
}
int gemm_trace_copy(unsigned long long* host, int n) {
  if (!g_trace_buf) return 0;
  n = std::min(n, 2 * kMaxSMs * 128);
  if (cudaMemcpy(host, g_trace_buf, (size_t)n * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  cudaMemset(g_trace_buf, 0, (size_t)2 * kMaxSMs * 128 * 8);
  return n;
}
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
  return (int64_t)2 * kMaxSMs * BM * std::min((T + 31) / 32 * 32, 512);  // 2 slots per CTA
}

// Tile-contiguous weight layout: block (t, k) = rows [128t, +128) x cols [64k, +64) stored as the
// exact 16 KB shared-memory image of a 128B-swizzled K-major tile (16-byte chunk c of row r at
// chunk position c ^ (r & 7)); blocks ordered t-major then k. A stream-K range of consecutive
// (t, k) units is then one contiguous stretch of HBM.
__global__ void pack_tiled_kernel(const __nv_bfloat16* __restrict__ src, __nv_bfloat16* __restrict__ dst, int K) {
  KtScope kt_(KT_MISC, (uint32_t)(5));
  pdl_wait();
  kt_.mark();
  // no pdl_trigger(): a GEMM may prefetch these weights before its grid dependency resolves, so
  // dependents launch only once the packed weights are complete
  const int kb = K / BK;
  const int blk = blockIdx.x;
  const int t = blk / kb, k = blk % kb;
  const int r = threadIdx.x;  // 128 rows
  const uint4* s = reinterpret_cast<const uint4*>(src + ((size_t)t * BM + r) * K + (size_t)k * BK);
  uint4* d = reinterpret_cast<uint4*>(dst + (size_t)blk * BM * BK + (size_t)r * BK);
#pragma unroll
  for (int c = 0; c < 8; ++c) d[c ^ (r & 7)] = s[c];
}

// Launched WITHOUT the PDL attribute after weight packing: it starts only when the pack kernel has
// fully completed, so a following GEMM that prefetches weights before its own grid dependency
// resolves (launched with PDL relative to this kernel) can never observe a partially packed tile.
__global__ void stream_fence_kernel() {}

cudaError_t gemm_pack_weight(const void* src, void* dst, int N, int K, cudaStream_t st) {
  if (N % BM || K % BK) return cudaErrorInvalidValue;
  launch_k(pack_tiled_kernel, dim3((N / BM) * (K / BK)), dim3(BM), 0, st, (const __nv_bfloat16*)src, (__nv_bfloat16*)dst, K);
  stream_fence_kernel<<<1, 32, 0, st>>>();
  return cudaGetLastError();
}

static bool make_map_tiled(CUtensorMap* m, const void* ptr, long long rows) {
  // tile-contiguous weights as a [rows, 64] bf16 tensor: each 128-row box is one contiguous 16 KB
  // block already in the swizzled shared-memory image, so no TMA swizzle is applied
  cuuint64_t dims[2] = {(cuuint64_t)BK, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)BK * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)BM};
  return encode_tmap_cached(g_encode, m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                            box, CU_TENSOR_MAP_SWIZZLE_NONE) == CUDA_SUCCESS;
}

// CTA-pair (cta_group::2) mode for a weight shape: a function of (N, K) only (batch invariance)
// Persistent groups for a cluster size: the co-resident clusters of a 1-CTA-per-SM kernel (GPCs
// with an odd SM count or not a multiple of 4 leave SMs out: 74 pairs but only 33 quads on a B200).
static int max_groups(int cg) {
  static int cache[5] = {0, 0, 0, 0, 0};
  if (cache[cg]) return cache[cg];
  int n = num_sms() / cg;
  if (cg > 1) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(num_sms() / cg * cg);
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = 200 * 1024;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cg;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int m = 0;
    cudaFuncSetAttribute(gemm_sk_kernel<2, EPI_STORE_F32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (cudaOccupancyMaxActiveClusters(&m, (const void*)gemm_sk_kernel<2, EPI_STORE_F32>, &cfg) == cudaSuccess && m > 0)
      n = std::min(n, m);
    cudaGetLastError();
  }
  cache[cg] = n;
  return n;
}

// Stream-K groups of a weight shape: the co-resident groups, but at least kMinUnits (tile, k-block)
// units per group -- small weights (the Small config's 0.6-5 MB GEMMs) otherwise split every tile over
// dozens of groups and spend the launch in the fixup. A function of (N, K) and the device only (batch
// invariance); every 7B / 13B shape keeps all 74 groups.
static int sk_groups(int cg, long long n_tiles, int kb) {
  static const int min_u = getenv("SF_GEMM_MINU") ? std::max(1, atoi(getenv("SF_GEMM_MINU"))) : 4;
  const long long U = n_tiles * kb;
  return (int)std::max<long long>(1, std::min<long long>(max_groups(cg), std::max<long long>(1, U / min_u)));
}

// CTA-pair mode halves each SM's share of the activation tile (the MMA reads the B operand from
// both CTAs' shared memory), the L2->SM traffic that bounds the skinny GEMM at large T.
// (A 4-CTA variant multicasting the activation between two pairs deadlocked in round 1 and was
// removed.) SF_GEMM_CG=1 forces single-CTA groups (tests / experiments).
static int gemm_cg(int N, int K) {
  (void)K;
  static const int env = getenv("SF_GEMM_CG") ? atoi(getenv("SF_GEMM_CG")) : 2;
  if (env >= 2 && N % (2 * BM) == 0) return 2;
  return 1;
}

using SkKernel = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap, const SkParams);
static SkKernel sk_kernel_for(int cg, int mode) {
#define SF_SK(CGV)                                              \
  switch (mode) {                                               \
    case EPI_STORE_ACT: return gemm_sk_kernel<CGV, EPI_STORE_ACT>;   \
    case EPI_STORE_F32: return gemm_sk_kernel<CGV, EPI_STORE_F32>;   \
    case EPI_ADD_F32: return gemm_sk_kernel<CGV, EPI_ADD_F32>;       \
    case EPI_BIAS_F32: return gemm_sk_kernel<CGV, EPI_BIAS_F32>;     \
    case EPI_SWIGLU_ACT: return gemm_sk_kernel<CGV, EPI_SWIGLU_ACT>; \
    case EPI_QKV_ROPE: return gemm_sk_kernel<CGV, EPI_QKV_ROPE>;     \
    default: return gemm_sk_kernel<CGV, EPI_PARTIAL>;           \
  }
  if (cg == 2) SF_SK(2);
  SF_SK(1);
#undef SF_SK
}

// phase B of a chain launch (gate/up -> down): the down projection over the SwiGLU output
struct ChainB {
  const void* W;   // tiled weights [N, K]
  int N, K;
  const void* act;  // [T, K] bf16, row stride K (phase A's output)
  float* partial;   // its EPI_PARTIAL slots
  int* ready;       // [K / 64] readiness flags (zero)
  int* done;        // launch counter (zero)
};

static cudaError_t launch_sk(const void* A, int lda, const void* W, bool w_tiled, int T, int N, int K,
                             const GemmEpi& epi, const GemmScratch& scratch, cudaStream_t st,
                             const ChainB* chain = nullptr) {
  static bool attr = false;
  if (!attr) {
    for (int cg = 1; cg <= 2; cg *= 2)
      for (int md = 0; md <= EPI_QKV_ROPE; ++md)
        cudaFuncSetAttribute(sk_kernel_for(cg, md), cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(gemm_sk_kernel<2, EPI_SWIGLU_ACT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    attr = true;
  }
  const int CG = (w_tiled && T >= 1) ? gemm_cg(N, K) : 1;
  SkParams p{};
  p.T = T;
  p.N = N;
  p.K = K;
  p.Tp = (T + 31) / 32 * 32;
  tc_shape(T, &p.NT, &p.n_sub);
  if (p.n_sub > 2) return cudaErrorInvalidValue;  // (callers split T > 512)
  p.kb_total = K / BK;
  p.n_tiles = N / (BM * CG);
  const long long U = (long long)p.n_tiles * p.kb_total;
  p.G = sk_groups(CG, p.n_tiles, p.kb_total);  // depends on (N, K) and the device only
  (void)U;
  const int cols = p.n_sub * p.NT;
  p.nbuf = (2 * cols <= 512) ? 2 : 1;
  p.tmem_cols = 32;
  while ((int)p.tmem_cols < p.nbuf * cols) p.tmem_cols <<= 1;
  const int stage_bytes = BM * BK * 2 + p.n_sub * (CG >= 2 ? p.NT / 2 : p.NT) * BK * 2;
  // deep ring: ~200 KB in flight per SM covers loaded-HBM latency (Little's law)
  static const int env_st = getenv("SF_GEMM_STAGES") ? atoi(getenv("SF_GEMM_STAGES")) : 0;
  p.stages = std::max(2, std::min(16, (216 * 1024) / stage_bytes));
  if (env_st >= 2 && env_st * stage_bytes <= 216 * 1024) p.stages = env_st;
  // release slots in groups of cgrp (>= 3 groups in the ring; cgrp divides stages)
  p.cgrp = 1;
  for (int cg = 8; cg >= 2; cg >>= 1)
    if (cg * 3 <= p.stages || (cg * 2 <= p.stages && cg == 2)) {
      p.cgrp = cg;
      break;
    }
  static const int env_cg = getenv("SF_GEMM_CGRP") ? atoi(getenv("SF_GEMM_CGRP")) : 0;
  if (env_cg >= 1 && env_cg <= p.stages) p.cgrp = env_cg;
  p.stages = (p.stages / p.cgrp) * p.cgrp;
  static const int env_probe = getenv("SF_GEMM_PROBE") ? atoi(getenv("SF_GEMM_PROBE")) : 0;
  p.probe = env_probe;
  p.epi = epi;
  p.partial = scratch.partial;
  p.flags = scratch.counters;
  p.w_tiled = w_tiled ? 1 : 0;
  p.w_tiles = (const __nv_bfloat16*)W;
  p.trace = gemm_trace_buffer();
  // bit0 bulk fixup loads; bits 1..3 smem-staged stores for ACT / F32 / SwiGLU outputs; bit 4 park
  // mid-range full tiles (T >= 64) for the final phase
  static const int env_epi = getenv("SF_GEMM_EPI") ? atoi(getenv("SF_GEMM_EPI")) : 31;
  p.bulk_ok = env_epi & 1;
  // weight stages requested before the grid dependency resolves: a few, not the whole ring -- the
  // first activation tile is served behind them, and it gates the first MMA
  static const int env_npre = getenv("SF_GEMM_NPRE") ? atoi(getenv("SF_GEMM_NPRE")) : 4;
  p.npre = std::max(1, std::min(env_npre, p.stages));
  p.drain = epi.drain >= 0 ? epi.drain : sk_drain(epi.mode);
  if (!sk_fits(p.G, p.n_tiles, p.kb_total, p.drain)) return cudaErrorInvalidValue;
  p.park = (env_epi >> 4) & 1;
  p.stage_ok = (env_epi >> 1) & 7;
  {  // three-slot accumulator rotation: every non-final piece must take the drain-to-partial path
    static const int env_rot = getenv("SF_GEMM_ROT") ? atoi(getenv("SF_GEMM_ROT")) : 1;
    const int m = epi.mode;
    const bool stageable = m == EPI_STORE_ACT || m == EPI_STORE_F32 || m == EPI_SWIGLU_ACT || m == EPI_QKV_ROPE;
    const int out_elt = m == EPI_STORE_F32 ? 4 : 2;
    const bool can_stage = stageable && p.stage_ok && ((size_t)epi.ldo * out_elt) % 16 == 0 &&
                           p.stages * stage_bytes >= 3 * 16384 + 64 * BM * 4;
    p.rot = (env_rot && !chain && CG == 2 && p.n_sub == 2 && p.NT % 32 == 0 && 3 * p.NT <= 512 && p.nbuf == 1 && T >= 64 &&
             (m == EPI_PARTIAL || (can_stage && p.park)))
                ? 1
                : 0;
  }
  static const int trace_n = getenv("SF_GEMM_TRACE_N") ? atoi(getenv("SF_GEMM_TRACE_N")) : 0;
  if (trace_n && trace_n != N) p.trace = nullptr;  // trace one weight shape only
  if (!scratch.partial || scratch.partial_elems < (int64_t)2 * p.G * CG * p.Tp * BM || scratch.n_counters < p.G * CG)
    return cudaErrorInvalidValue;
  if (epi.mode == EPI_PARTIAL && p.n_tiles > p.G) return cudaErrorInvalidValue;
  const size_t smem = (size_t)p.stages * stage_bytes + 1024 + (2 * p.stages + 10) * 8;
  CUtensorMap mw, ma;
  memset(&mw, 0, sizeof(mw));
  static const int env_wtma = getenv("SF_GEMM_WTMA") ? atoi(getenv("SF_GEMM_WTMA")) : 0;
  p.w_tma = (CG == 1 && w_tiled && env_wtma) ? 1 : 0;
  if (CG >= 2 || p.w_tma) {
    if (!make_map_tiled(&mw, W, (long long)N * (K / BK))) return cudaErrorInvalidValue;
  } else if (!w_tiled && !make_map(&mw, W, N, K, K, BM)) {
    return cudaErrorInvalidValue;
  }
  if (!make_map(&ma, A, T, K, lda, p.NT / CG)) return cudaErrorInvalidValue;
  CUtensorMap mwB = mw, maB = ma;
  if (chain) {
    if (CG != 2 || epi.mode != EPI_SWIGLU_ACT || gemm_cg(chain->N, chain->K) != 2 || chain->K * 2 != N)
      return cudaErrorInvalidValue;
    p.kbB = chain->K / BK;
    p.n_tilesB = chain->N / (BM * CG);
    if (sk_groups(CG, p.n_tilesB, p.kbB) != p.G || p.n_tilesB > p.G)
      return cudaErrorInvalidValue;  // both phases on the same groups; phase B published as EPI_PARTIAL
    p.drainB = sk_drain(EPI_PARTIAL);
    if (!sk_fits(p.G, p.n_tilesB, p.kbB, p.drainB)) return cudaErrorInvalidValue;
    p.partialB = chain->partial;
    p.readyB = chain->ready;
    p.doneB = chain->done;
    p.park = 0;  // (a parked tile's output would be written after phase B needs it)
    if (!make_map_tiled(&mwB, chain->W, (long long)chain->N * p.kbB) ||
        !make_map(&maB, chain->act, T, chain->K, chain->K, p.NT / CG))
      return cudaErrorInvalidValue;
  }
  if (CG == 1) {
    launch_k(sk_kernel_for(1, epi.mode), dim3(p.G), dim3(384), smem, st, mw, ma, mw, ma, p);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.G * CG);
  cfg.blockDim = dim3(384);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = CG;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  if (chain) return cudaLaunchKernelEx(&cfg, gemm_sk_kernel<2, EPI_SWIGLU_ACT, true>, mw, ma, mwB, maB, p);
  return cudaLaunchKernelEx(&cfg, sk_kernel_for(2, epi.mode), mw, ma, mw, ma, p);
}

// Gate/up (SwiGLU) -> down in one launch (see gemm_sk_kernel CHAIN). Phase B's partial slots start
// at scratch.partial + gemm_chain_partial_offset(T) floats; its k segmentation is the standalone
// down GEMM's (same groups, same drain), so gemm_partial_geom / launch_resid_norm read it unchanged.
static constexpr int kChainReady = 1024, kChainDone = 4000;  // GemmScratch::counters layout
int64_t gemm_chain_partial_offset(int T) {
  return (int64_t)2 * max_groups(2) * 2 * ((T + 31) / 32 * 32) * BM;
}
int64_t gemm_chain_partial_elems(int T) { return 2 * gemm_chain_partial_offset(T); }
bool gemm_chain_supported(int T, int NA, int KA, int NB) {
  const int KB = NA / 2;
  if (T < 1 || T > 512 || NA % (2 * BM) || KA % BK || NB % (2 * BM) || KB % BK || KB / BK > kChainDone - kChainReady)
    return false;
  if (gemm_cg(NA, KA) != 2 || gemm_cg(NB, KB) != 2) return false;
  const long long UA = (long long)(NA / (2 * BM)) * (KA / BK), UB = (long long)(NB / (2 * BM)) * (KB / BK);
  const int G = max_groups(2);
  PartialGeom g;
  return UA >= G && UB >= G && NB / (2 * BM) <= G && gemm_partial_geom(T, NB, KB, &g);
}
cudaError_t gemm_chain_launch(const void* A, int lda, const void* WA, int NA, int KA, void* act, const void* WB,
                              int NB, int T, const GemmScratch& scratch, cudaStream_t st) {
  if (!gemm_chain_supported(T, NA, KA, NB) || !ensure_encode()) return cudaErrorInvalidValue;
  if (scratch.n_counters <= kChainDone || scratch.partial_elems < gemm_chain_partial_elems(T))
    return cudaErrorInvalidValue;
  GemmEpi e;
  e.mode = EPI_SWIGLU_ACT;
  e.out = act;
  e.ldo = NA / 2;
  ChainB cb{WB, NB, NA / 2, act, scratch.partial + gemm_chain_partial_offset(T), scratch.counters + kChainReady,
            scratch.counters + kChainDone};
  return launch_sk(A, lda, WA, true, T, NA, KA, e, scratch, st, &cb);
}

bool gemm_partial_geom(int T, int N, int K, PartialGeom* g, int drain) {
  if (N % BM || K % BK || T > 512) return false;
  const int CG = gemm_cg(N, K);
  const int n_tiles = N / (BM * CG);
  const long long U = (long long)n_tiles * (K / BK);
  const int G = sk_groups(CG, n_tiles, K / BK);
  (void)U;
  if (n_tiles > G) return false;  // a group must touch at most 2 tiles
  g->G = G * CG;                  // slots are per CTA: consumer addresses (2 * group + which) * CG + rank
  g->kb = K / BK;
  g->n_tiles = N / BM;
  g->T = T;
  g->drain = drain >= 0 ? drain : sk_drain(EPI_PARTIAL);
  if (!sk_fits(G, n_tiles, K / BK, g->drain)) return false;
  return true;
}

// One CTA per virtual row, d / (4 NG) threads (<= 1024): thread t owns the float4 column groups
// 4t + 4 nthr j (j < NG). Per 128-column tile the k-segment slot offsets are precomputed in shared
// memory; the segments' 16-byte partial loads are issued in batches of kRnBatch before the k-ordered
// sums, so a row streams at memory speed and a few rows (B = 1) still spread over many warps.
constexpr int kRnMaxSeg = 16;  // k segments per 128-column tile (stream-K: <= G / n_tiles + 2)
constexpr int kRnMaxTiles = 128;
// float4 groups per virtual thread of the row's canonical reduction tree: the fewest that fit 1024
// threads (the tree -- and so every bit -- depends on d only)
static int rn_ng(int d) {
  for (int ng = 1; ng <= 4; ++ng)
    if (d % (4 * ng * 32) == 0 && d / (4 * ng) <= 1024) return ng;
  return 0;
}

// The canonical row kernel has nv = d / (4 NG) virtual threads; virtual thread v owns float4 column
// groups v + nv j (j < NG), its sum of squares is an fma chain over them, a warp_sum per 32-thread
// virtual warp and one final warp_sum over the virtual warps' sums. A launch runs it with F virtual
// threads per real thread (v = tid + nthr f): F = 2 halves the threads of a row so two rows are
// resident per SM at a 320-row block (one wave instead of 2.2); the arithmetic -- and every bit -- is
// the same for either F, so F is chosen per launch (T) without breaking batch invariance.
template <int NG, int F>
__global__ void __launch_bounds__(1024) resid_norm_kernel(
    const float* __restrict__ partial, int G, int kb, int drain, int CG, int n_tiles_cta, int T, int rep, int d,
    const float* resid, const float* __restrict__ add, const float* __restrict__ bias, float* out, float* tap,
    const float* __restrict__ gamma, float eps, __nv_bfloat16* xn, TpSrc tp) {
  constexpr int kRnBatch = (8 / NG) / F;  // partial loads in flight per column group
  __shared__ int seg_n[kRnMaxTiles];
  __shared__ int seg_off[kRnMaxTiles][kRnMaxSeg];  // slot * T * 128 (the tile's k segments, k order)
  __shared__ float red[32];
  const int nthr = blockDim.x, nv = nthr * F;
  const int r = blockIdx.x;
  const int src_row = r / rep, col0 = (r % rep) * d;
  const int tid = threadIdx.x;
  if (partial) {  // geometry only (no dependency on the previous kernel)
    const int groups = G / CG;
    const int n_tiles_grp = n_tiles_cta / CG;
    for (int vt = tid; vt < n_tiles_cta; vt += nthr) {
      const int tg = vt / CG, rk = vt % CG;
      const int ua = tg * kb, ub = ua + kb - 1;
      const int lo = sk_group_of(ua, groups, n_tiles_grp, kb, drain);
      const int hi = sk_group_of(ub, groups, n_tiles_grp, kb, drain);
      const int w0 = (sk_begin(lo, groups, n_tiles_grp, kb, drain) / kb == tg) ? 0 : 1;
      seg_n[vt] = hi - lo + 1;
      for (int q = 0; q < kRnMaxSeg && lo + q <= hi; ++q)
        seg_off[vt][q] = ((2 * (lo + q) + (q == 0 ? w0 : 0)) * CG + rk) * T * BM;
    }
    __syncthreads();
  }
  KtScope kt_(KT_RESID_NORM, (uint32_t)(d));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  __shared__ int tp_epoch;
  if (tp.n > 0) {
    // NEXT-3: every peer has published this epoch's slot (system-scope acquire of the flag it wrote
    // into this rank's region after its GEMM); bounded, so a missing peer cannot hang the device
    if (tid == 0) {
      const int e = *(volatile const int*)tp.ctr;
      const unsigned long long t0 = gtimer();
      for (int q = 0; q < tp.n; ++q) {
        if (q == tp.own) continue;
        int f;
        for (;;) {
          asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(f) : "l"(tp.flags + q) : "memory");
          if (f >= e) break;
          if (gtimer() - t0 > 5000000000ull) {  // 5 s
            atomicOr(tp.err, 4);  // (specformer_sync: SF_ERR_NCCL)
            break;
          }
          __nanosleep(64);
        }
      }
      tp_epoch = e;
    }
    __syncthreads();
  }
  float4 x[F][NG];
#pragma unroll
  for (int f = 0; f < F; ++f)
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      const int i = 4 * (tid + nthr * f) + 4 * nv * j;  // column within the virtual row
      x[f][j] = resid ? *reinterpret_cast<const float4*>(resid + (size_t)r * d + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      if (add) {  // (tensor parallelism: the all-reduced row-parallel GEMM output)
        const float4 a = *reinterpret_cast<const float4*>(add + (size_t)r * d + i);
        x[f][j].x += a.x;
        x[f][j].y += a.y;
        x[f][j].z += a.z;
        x[f][j].w += a.w;
      }
      if (tp.n > 0) {  // (NEXT-3: the ranks' bf16 GEMM outputs, read over peer memory, summed in rank order)
        const size_t off = (size_t)(tp_epoch & 1) * (size_t)tp.slot_elems + (size_t)r * d + i;
        uint2 raw[kTpMax];
#pragma unroll
        for (int q = 0; q < kTpMax; ++q)
          if (q < tp.n) raw[q] = __ldcg(reinterpret_cast<const uint2*>(tp.slot[q] + off));
#pragma unroll
        for (int q = 0; q < kTpMax; ++q)
          if (q < tp.n) {
            const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw[q].x));
            const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw[q].y));
            x[f][j].x += lo.x;
            x[f][j].y += lo.y;
            x[f][j].z += hi.x;
            x[f][j].w += hi.y;
          }
      }
      if (bias) {
        const float4 bb = *reinterpret_cast<const float4*>(bias + col0 + i);
        x[f][j].x += bb.x;
        x[f][j].y += bb.y;
        x[f][j].z += bb.z;
        x[f][j].w += bb.w;
      }
    }
  if (partial) {
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      // the F column groups' segment loads in flight together, then each group's k-ordered sums
      int vt[F], ns[F], nsm = 0;
      const float* bp[F];
#pragma unroll
      for (int f = 0; f < F; ++f) {
        const int n = col0 + 4 * (tid + nthr * f) + 4 * nv * j;
        vt[f] = n / BM;
        ns[f] = seg_n[vt[f]];
        nsm = max(nsm, ns[f]);
        bp[f] = partial + (size_t)src_row * BM + n % BM;
      }
      for (int q0 = 0; q0 < nsm; q0 += kRnBatch) {
        float4 pv[F][kRnBatch];
#pragma unroll
        for (int q = 0; q < kRnBatch; ++q)
#pragma unroll
          for (int f = 0; f < F; ++f)
            if (q0 + q < ns[f]) pv[f][q] = __ldcg(reinterpret_cast<const float4*>(bp[f] + seg_off[vt[f]][q0 + q]));
#pragma unroll
        for (int q = 0; q < kRnBatch; ++q)
#pragma unroll
          for (int f = 0; f < F; ++f)
            if (q0 + q < ns[f]) {  // k order
              x[f][j].x += pv[f][q].x;
              x[f][j].y += pv[f][q].y;
              x[f][j].z += pv[f][q].z;
              x[f][j].w += pv[f][q].w;
            }
      }
    }
  }
  float ss[F];
#pragma unroll
  for (int f = 0; f < F; ++f) {
    ss[f] = 0.f;
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      const int i = 4 * (tid + nthr * f) + 4 * nv * j;
      if (out) *reinterpret_cast<float4*>(out + (size_t)r * d + i) = x[f][j];
      if (tap) *reinterpret_cast<float4*>(tap + (size_t)r * d + i) = x[f][j];
      ss[f] = fmaf(x[f][j].x, x[f][j].x, ss[f]);
      ss[f] = fmaf(x[f][j].y, x[f][j].y, ss[f]);
      ss[f] = fmaf(x[f][j].z, x[f][j].z, ss[f]);
      ss[f] = fmaf(x[f][j].w, x[f][j].w, ss[f]);
    }
  }
  if (!gamma) return;
  // the canonical tree: a warp_sum per virtual warp, then warp 0 over the virtual warps' sums in order
#pragma unroll
  for (int f = 0; f < F; ++f) {
    const float v = warp_sum(ss[f]);
    if ((tid & 31) == 0) red[(tid >> 5) + (nthr >> 5) * f] = v;
  }
  __syncthreads();
  if (tid < 32) {
    float v = (tid < (nv >> 5)) ? red[tid] : 0.f;
    v = warp_sum(v);
    if (tid == 0) red[0] = v;
  }
  __syncthreads();
  const float rs = 1.0f / sqrtf(red[0] / (float)d + eps);
#pragma unroll
  for (int f = 0; f < F; ++f)
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      const int i = 4 * (tid + nthr * f) + 4 * nv * j;
      const float4 gg = *reinterpret_cast<const float4*>(gamma + i);
      __nv_bfloat162 lo = __floats2bfloat162_rn(x[f][j].x * rs * gg.x, x[f][j].y * rs * gg.y);
      __nv_bfloat162 hi = __floats2bfloat162_rn(x[f][j].z * rs * gg.z, x[f][j].w * rs * gg.w);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(xn + (size_t)r * d + i) = pk;
    }
}

cudaError_t launch_resid_norm(const float* partial, const PartialGeom* g, int T, int rep, int d, const float* resid,
                              const float* add, const float* bias, float* out, float* tap, const float* gamma,
                              float eps, __nv_bfloat16* xn, cudaStream_t st, const TpSrc* tps) {
  if (T * rep <= 0) return cudaSuccess;
  TpSrc tp;
  if (tps) {
    if (tps->n < 1 || tps->n > kTpMax || rep != 1 || partial) return cudaErrorInvalidValue;
    tp = *tps;
  }
  const int ng = rn_ng(d);
  if (!ng) return cudaErrorInvalidValue;
  int G = 1, kb = 1, CG = 1, nt = 1, Tslot = T, drain = 0;
  if (partial) {
    G = g->G;
    kb = g->kb;
    drain = g->drain;
    nt = g->n_tiles;
    CG = gemm_cg(nt * BM, kb * BK);
    Tslot = g->T;
    if (nt > kRnMaxTiles) return cudaErrorInvalidValue;
    const int groups = G / CG;
    if ((groups + nt / CG - 1) / (nt / CG) + 1 > kRnMaxSeg) return cudaErrorInvalidValue;
  }
  const int nv = d / (4 * ng);  // the canonical tree's virtual threads
  // more rows than SMs: half the threads per row (two virtual threads each) so two rows fit an SM
  const char* env_fs = getenv("SF_RN_FOLD");  // (read per launch: tests force 1 / 2)
  const int env_f = env_fs ? atoi(env_fs) : -1;
  const bool fold = env_f >= 0 ? env_f == 2 : T * rep > num_sms();
  const dim3 grid(T * rep);
#define SF_RN(NGV)                                                                                                  \
  return (fold && ng == 1 && nv % 64 == 0)                                                                          \
             ? launch_k(resid_norm_kernel<NGV, 2>, grid, dim3(nv / 2), 0, st, partial, G, kb, drain, CG, nt, Tslot,  \
                        rep, d, resid, add, bias, out, tap, gamma, eps, xn, tp)                                      \
             : launch_k(resid_norm_kernel<NGV, 1>, grid, dim3(nv), 0, st, partial, G, kb, drain, CG, nt, Tslot, rep, \
                        d, resid, add, bias, out, tap, gamma, eps, xn, tp)
  switch (ng) {
    case 1: SF_RN(1);
    case 2: SF_RN(2);
    case 3: SF_RN(3);
    default: SF_RN(4);
  }
#undef SF_RN
}

// NEXT-3 epoch publication: one warp. The GEMM that wrote this epoch's slot has completed (stream
// order); the system-scope fence orders its stores before the flags the peers acquire.
__global__ void tp_signal_kernel(int* ctr, TpPeers pf, int n, int own) {
  __shared__ int e;
  if (threadIdx.x == 0) {
    e = *ctr + 1;
    *ctr = e;
    __threadfence_system();
  }
  __syncthreads();
  const int q = threadIdx.x;
  if (q < n && q != own)
    asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(pf.p[q] + own), "r"(e) : "memory");
}

cudaError_t launch_tp_signal(int* ctr, int* const* peer_flags, int n, int own, cudaStream_t s) {
  if (n < 1 || n > kTpMax || own < 0 || own >= n) return cudaErrorInvalidValue;
  TpPeers pf;
  for (int q = 0; q < n; ++q) pf.p[q] = peer_flags[q];
  tp_signal_kernel<<<1, 32, 0, s>>>(ctr, pf, n, own);
  return cudaGetLastError();
}

// Whether the fused consumer supports this (d, N, K): callers use the unfused path otherwise.
bool resid_norm_supported(int d, int T, int N, int K) {
  if (!rn_ng(d)) return false;
  PartialGeom g;
  if (!gemm_partial_geom(T, N, K, &g)) return false;
  const int CG = gemm_cg(N, K);
  const int groups = g.G / CG, ntg = g.n_tiles / CG;
  return (groups + ntg - 1) / ntg + 1 <= kRnMaxSeg && g.n_tiles <= kRnMaxTiles;
}

// ------------------------------------------------------------------------ QKV partial consumer
// The k-segments of 128-column tile vt of an EPI_PARTIAL launch (stream-K over `groups` work groups of
// CG CTAs, ntg group tiles, kb k-blocks, tile-entry cost drain), in k order: count, and the float
// offset of segment q's slot ((2 group + which) CG + rank) * Tslot * 128 (launch_resid_norm's table).
SF_DEV int pseg_count(int vt, int groups, int ntg, int kb, int drain, int CG) {
  const int tg = vt / CG, ua = tg * kb;
  return sk_group_of(ua + kb - 1, groups, ntg, kb, drain) - sk_group_of(ua, groups, ntg, kb, drain) + 1;
}
SF_DEV size_t pseg_off(int vt, int q, int groups, int ntg, int kb, int drain, int CG, int Tslot) {
  const int tg = vt / CG, rk = vt % CG, ua = tg * kb;
  const int lo = sk_group_of(ua, groups, ntg, kb, drain);
  const int w0 = (sk_begin(lo, groups, ntg, kb, drain) / kb == tg) ? 0 : 1;
  return (size_t)((2 * (lo + q) + (q == 0 ? w0 : 0)) * CG + rk) * Tslot * BM;
}

// One (row t, head h) item of the QKV partial consumer, by one warp: the head's k-segment partials
// summed in k order, rounded to bf16, rotated (q / k heads) or copied (v heads) into q_out / the page.
// Lane l owns the pair-interleaved positions 4l..4l+3 = dims (2l, 2l+64, 2l+1, 2l+65) of the head.
// `seg(q)` returns the float offset of the head's segment q; ns segments.
template <typename SegOff>
SF_DEV void rope_partial_item(const float* __restrict__ partial, int t, int h, int ns, SegOff seg, int q_len,
                              const int* __restrict__ pos0, const float2* __restrict__ rope, int Hq, int Hkv,
                              const int* __restrict__ bt, int pps, __nv_bfloat16* Kp, __nv_bfloat16* Vp,
                              __nv_bfloat16* q_out) {
  const int lane = threadIdx.x & 31;
  const int pos = pos0[t / q_len] + t % q_len;
  const float* base = partial + (size_t)t * BM + 4 * lane;
  float4 x = __ldcg(reinterpret_cast<const float4*>(base + seg(0)));
  for (int q0 = 1; q0 < ns; q0 += 4) {  // k order; up to four loads in flight
    float4 pv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q0 + q < ns) pv[q] = __ldcg(reinterpret_cast<const float4*>(base + seg(q0 + q)));
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q0 + q < ns) {
        x.x += pv[q].x;
        x.y += pv[q].y;
        x.z += pv[q].z;
        x.w += pv[q].w;
      }
  }
  // positions (4l, 4l+1, 4l+2, 4l+3) = dims (2l, 2l+64, 2l+1, 2l+65), rounded as the GEMM would
  const __nv_bfloat162 lo = __floats2bfloat162_rn(x.x, x.z);  // dims 2l, 2l+1
  const __nv_bfloat162 hi = __floats2bfloat162_rn(x.y, x.w);  // dims 2l+64, 2l+65
  const uint32_t a = *reinterpret_cast<const uint32_t*>(&lo), bb = *reinterpret_cast<const uint32_t*>(&hi);
  const int b = t / q_len;
  if (h >= Hq + Hkv) {  // value head: plain copy into the page
    const int blk = bt[b * pps + pos / 16], slot = pos % 16;
    __nv_bfloat16* dst = Vp + (((size_t)blk * Hkv + (h - Hq - Hkv)) * 16 + slot) * 128;
    *reinterpret_cast<uint32_t*>(dst + 2 * lane) = a;
    *reinterpret_cast<uint32_t*>(dst + 64 + 2 * lane) = bb;
    return;
  }
  const float4 cs = *reinterpret_cast<const float4*>(rope + (size_t)pos * 64 + 2 * lane);
  const float2 x1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&a));
  const float2 x2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&bb));
  const float y10 = rope_y1(x1.x, x2.x, cs.x, cs.y), y20 = rope_y2(x1.x, x2.x, cs.x, cs.y);
  const float y11 = rope_y1(x1.y, x2.y, cs.z, cs.w), y21 = rope_y2(x1.y, x2.y, cs.z, cs.w);
  __nv_bfloat16* dst;
  if (h < Hq) {
    dst = q_out + ((size_t)t * Hq + h) * 128;
  } else {
    const int blk = bt[b * pps + pos / 16], slot = pos % 16;
    dst = Kp + (((size_t)blk * Hkv + (h - Hq)) * 16 + slot) * 128;
  }
  *reinterpret_cast<__nv_bfloat162*>(dst + 2 * lane) = __floats2bfloat162_rn(y10, y11);
  *reinterpret_cast<__nv_bfloat162*>(dst + 64 + 2 * lane) = __floats2bfloat162_rn(y20, y21);
}

// One warp per (row, head) item (persistent grid, two items in flight per warp): the arithmetic of
// rope_partial_item (the layer-sequence kernel's consumer), with both items' loads issued first.
__global__ void __launch_bounds__(256) rope_partial_kernel(const float* __restrict__ partial, int G, int kb, int drain,
                                                           int CG, int H, int Tslot, int T, int q_len,
                                                           const int* __restrict__ pos0, const float2* __restrict__ rope,
                                                           int Hq, int Hkv, const int* __restrict__ bt, int pps,
                                                           __nv_bfloat16* Kp, __nv_bfloat16* Vp, __nv_bfloat16* q_out) {
  __shared__ int seg_n[kRnMaxTiles];
  __shared__ int seg_off[kRnMaxTiles][kRnMaxSeg];  // slot * Tslot * 128, k order
  {  // geometry only (no dependency on the previous kernel)
    const int groups = G / CG, n_tiles_grp = H / CG;
    for (int vt = threadIdx.x; vt < H; vt += blockDim.x) {
      seg_n[vt] = pseg_count(vt, groups, n_tiles_grp, kb, drain, CG);
      for (int q = 0; q < kRnMaxSeg && q < seg_n[vt]; ++q)
        seg_off[vt][q] = (int)pseg_off(vt, q, groups, n_tiles_grp, kb, drain, CG, Tslot);
    }
    __syncthreads();
  }
  KtScope kt_(KT_ROPE, (uint32_t)Hq);
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * (blockDim.x >> 5);
  const int items = T * H;
  for (int i0 = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i0 < items; i0 += 2 * nw) {
    uint32_t a[2], bb[2];
    float4 cs[2];
    int t[2], h[2], pos[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int it = min(i0 + u * nw, items - 1);
      t[u] = it / H;
      h[u] = it % H;
      pos[u] = pos0[t[u] / q_len] + t[u] % q_len;
      const float* base = partial + (size_t)t[u] * BM + 4 * lane;
      const int ns = seg_n[h[u]];
      float4 x = __ldcg(reinterpret_cast<const float4*>(base + seg_off[h[u]][0]));
      for (int q0 = 1; q0 < ns; q0 += 4) {  // k order; up to four loads in flight
        float4 pv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q0 + q < ns) pv[q] = __ldcg(reinterpret_cast<const float4*>(base + seg_off[h[u]][q0 + q]));
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (q0 + q < ns) {
            x.x += pv[q].x;
            x.y += pv[q].y;
            x.z += pv[q].z;
            x.w += pv[q].w;
          }
      }
      // positions (4l, 4l+1, 4l+2, 4l+3) = dims (2l, 2l+64, 2l+1, 2l+65), rounded as the GEMM would
      const __nv_bfloat162 lo = __floats2bfloat162_rn(x.x, x.z);  // dims 2l, 2l+1
      const __nv_bfloat162 hi = __floats2bfloat162_rn(x.y, x.w);  // dims 2l+64, 2l+65
      a[u] = *reinterpret_cast<const uint32_t*>(&lo);
      bb[u] = *reinterpret_cast<const uint32_t*>(&hi);
      cs[u] = *reinterpret_cast<const float4*>(rope + (size_t)pos[u] * 64 + 2 * lane);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (i0 + u * nw >= items) break;
      const int b = t[u] / q_len;
      if (h[u] >= Hq + Hkv) {  // value head: plain copy into the page
        const int blk = bt[b * pps + pos[u] / 16], slot = pos[u] % 16;
        __nv_bfloat16* dst = Vp + (((size_t)blk * Hkv + (h[u] - Hq - Hkv)) * 16 + slot) * 128;
        *reinterpret_cast<uint32_t*>(dst + 2 * lane) = a[u];
        *reinterpret_cast<uint32_t*>(dst + 64 + 2 * lane) = bb[u];
        continue;
      }
      const float2 x1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&a[u]));
      const float2 x2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&bb[u]));
      const float y10 = rope_y1(x1.x, x2.x, cs[u].x, cs[u].y), y20 = rope_y2(x1.x, x2.x, cs[u].x, cs[u].y);
      const float y11 = rope_y1(x1.y, x2.y, cs[u].z, cs[u].w), y21 = rope_y2(x1.y, x2.y, cs[u].z, cs[u].w);
      __nv_bfloat16* dst;
      if (h[u] < Hq) {
        dst = q_out + ((size_t)t[u] * Hq + h[u]) * 128;
      } else {
        const int blk = bt[b * pps + pos[u] / 16], slot = pos[u] % 16;
        dst = Kp + (((size_t)blk * Hkv + (h[u] - Hq)) * 16 + slot) * 128;
      }
      *reinterpret_cast<__nv_bfloat162*>(dst + 2 * lane) = __floats2bfloat162_rn(y10, y11);
      *reinterpret_cast<__nv_bfloat162*>(dst + 64 + 2 * lane) = __floats2bfloat162_rn(y20, y21);
    }
  }
}

bool rope_partial_supported(int T, int N, int K, int Hq, int Hkv, int drain) {
  PartialGeom g;
  if (N != (Hq + 2 * Hkv) * BM || !gemm_partial_geom(T, N, K, &g, drain)) return false;
  const int CG = gemm_cg(N, K);
  const int groups = g.G / CG, ntg = g.n_tiles / CG;
  return (groups + ntg - 1) / ntg + 1 <= kRnMaxSeg && g.n_tiles <= kRnMaxTiles;
}

cudaError_t launch_rope_partial(const float* partial, const PartialGeom* g, int T, int q_len, const int* pos0,
                                const float2* rope, int Hq, int Hkv, const int* bt, int pps, void* Kp, void* Vp,
                                void* q_out, cudaStream_t st) {
  const int H = Hq + 2 * Hkv;
  if (!partial || !g || g->n_tiles != H || H > kRnMaxTiles || T < 1) return cudaErrorInvalidValue;
  const int CG = gemm_cg(g->n_tiles * BM, g->kb * BK);
  const int groups = g->G / CG;
  if ((groups + H / CG - 1) / (H / CG) + 1 > kRnMaxSeg) return cudaErrorInvalidValue;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // CTAs per SM: 4 = one resident wave at 64 registers (6 left a half-empty second wave: T = 320 13.4 ->
  // 10.8 us per launch); small blocks need fewer CTAs than that anyway
  static const int env_g = getenv("SF_ROPE_GRID") ? atoi(getenv("SF_ROPE_GRID")) : 4;
  const int grid = std::max(1, std::min(std::max(1, env_g) * sms, (T * H + 15) / 16));
  return launch_k(rope_partial_kernel, dim3(grid), dim3(256), 0, st, partial, g->G, g->kb, g->drain, CG, H, g->T, T,
                  q_len, pos0, rope, Hq, Hkv, bt, pps, (__nv_bfloat16*)Kp, (__nv_bfloat16*)Vp, (__nv_bfloat16*)q_out);
}

static cudaError_t gemm_launch_chunk(bool is_bf16, const void* A, int lda, const void* W, bool w_tiled, int T,
                                     int N, int K, const GemmEpi& epi, const GemmScratch& scratch,
                                     cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  if (!is_bf16) {
    const int Nout = epi.mode == EPI_SWIGLU_ACT ? N / 2 : N;
    dim3 grid((Nout + 31) / 32, (T + 31) / 32), block(32, 8);
    if (epi.mode == EPI_SWIGLU_ACT)
      launch_k(gemm_simt_kernel<true>, dim3(grid), dim3(block), 0, st, (const float*)A, lda, (const float*)W, T, N, K, epi);
    else
      launch_k(gemm_simt_kernel<false>, dim3(grid), dim3(block), 0, st, (const float*)A, lda, (const float*)W, T, N, K, epi);
    return cudaGetLastError();
  }
  if (N % BM || K % BK || T > 512) return cudaErrorInvalidValue;
  if (!ensure_encode()) return cudaErrorNotSupported;
  return launch_sk(A, lda, W, w_tiled, T, N, K, epi, scratch, st);
}

// Rows beyond 512 (the TMEM accumulator capacity) are processed as independent column chunks of
// equal size (576 rows: 2 x 288, not 512 + 64 -- each chunk streams the weights once, and two
// half-size chunks finish sooner than a full one plus a DRAM-bound sliver); per-element
// arithmetic is unchanged (the k segmentation depends on (N, K) only), so results do not depend
// on the chunking.
cudaError_t gemm_launch(bool is_bf16, const void* A, int lda, const void* W, bool w_tiled, int T, int N, int K,
                        const GemmEpi& epi, const GemmScratch& scratch, cudaStream_t st) {
  if (!is_bf16 || T <= 512) return gemm_launch_chunk(is_bf16, A, lda, W, w_tiled, T, N, K, epi, scratch, st);
  const int n_chunks = (T + 511) / 512;
  const int chunk = std::min(512, ((T + n_chunks - 1) / n_chunks + 15) / 16 * 16);
  for (int t0 = 0; t0 < T; t0 += chunk) {
    GemmEpi e = epi;
    const size_t out_elt = (epi.mode == EPI_STORE_ACT || epi.mode == EPI_SWIGLU_ACT) ? 2 : 4;
    if (epi.mode == EPI_QKV_ROPE) e.rope.t0 = epi.rope.t0 + t0;
    else e.out = (char*)epi.out + (size_t)t0 * epi.ldo * out_elt;
    if (epi.tap) e.tap = epi.tap + (size_t)t0 * epi.ldo;
    if (epi.amax) e.amax = epi.amax + t0;
    if (!epi.out) e.out = nullptr;
    cudaError_t r = gemm_launch_chunk(true, (const char*)A + (size_t)t0 * lda * 2, lda, W, w_tiled,
                                      std::min(chunk, T - t0), N, K, e, scratch, st);
    if (r != cudaSuccess) return r;
  }
  return cudaSuccess;
}

#include "gemm_seq.cuh"

cudaError_t kt_setup_gemm(void* rec, unsigned* cnt, unsigned cap) {
  KtBuf b;
  b.rec = reinterpret_cast<KtRec*>(rec);
  b.cnt = cnt;
  b.cap = cap;
  return kt_setup_tu(b);
}

}  // namespace sf
