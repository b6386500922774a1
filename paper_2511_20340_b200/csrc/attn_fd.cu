// attn_fd.cu -- bf16 hybrid-mask paged decode attention (mode CAUSAL_PREFIX), flash-decoding form.
//
// One CTA item = (sequence b, kv head, 16-row query tile, 512-key segment); persistent CTAs walk the
// items, so even a single sequence spreads over (heads x segments) SMs. A
// producer warp streams the item's 128-key K/V chunks with TMA (one 2-D 128B-swizzled box per
// (16-key page, 64-dim half)) into a 3-stage mbarrier ring. Compute warp w owns keys
// [32w, 32w+32) of every chunk and keeps its own online-softmax state (m, l, O[16x128]) across
// the chunks -- no cross-warp synchronisation per chunk, P never leaves registers:
//   S = Q K_w^T (mma.sync m16n8k16 bf16 -> fp32), masked (key <= row position), m_new = max,
//   O = O e^(m_old - m_new) + P V_w,  l = l e^(m_old - m_new) + sum P.
// At the end of the item the 4 warp states are merged in the fixed order w = 0..3 into the
// segment's unnormalised (M, L, acc). A row whose keys span one segment is normalised directly;
// otherwise each segment is written to the partial buffer and the CTA that completes the last
// segment of the (b, kv head, tile) group (arrival counter) merges segments 0, 1, ... in order:
// out = sum_s acc_s 2^(M_s - M) / sum_s L_s 2^(M_s - M) -- for one segment exactly acc / L.
// Every row's arithmetic (chunk and segment boundaries at fixed absolute key positions, per-warp
// key slices, merge orders) is independent of batch size and block length (batch invariance, C23).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cfloat>
#include <cmath>

#include "common.cuh"
#include "kernels.cuh"

namespace sf {
namespace {

constexpr int HD = 128;
constexpr int CH = 128;
constexpr int NST = 3;
constexpr int KV_BYTES = CH * HD * 2;      // 32 KB
constexpr int STAGE_BYTES = 2 * KV_BYTES;  // 64 KB
constexpr int MERGE_BYTES = 4 * 16 * (HD + 2) * 4;  // per-warp O, m, l for the final merge
constexpr int SMEM = NST * STAGE_BYTES + MERGE_BYTES + 2 * NST * 8 + 1024 + 64 + 16;

SF_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
SF_DEV void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
SF_DEV void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
SF_DEV uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
// 16-byte chunk c (0..15) of key row j in a [2 halves][128 keys][128 B] tile, 128B-swizzled the
// way TMA SWIZZLE_128B writes each 128-byte row (chunk c' at c' ^ (j % 8))
SF_DEV uint32_t swz(int j, int c) {
  return (uint32_t)((c >> 3) * (CH * 128) + j * 128 + (((c & 7) ^ (j & 7)) << 4));
}
SF_DEV void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

struct Item {
  int b, kvh, qt, seg, c0, c1, nseg;  // chunks [c0, c1) of segment seg (of nseg) of group (b, kvh, qt)
};

}  // namespace

// item = (b * Hkv + kvh) * ntiles + qt. Warps 0..3 compute, warp 4 produces.
__global__ void __launch_bounds__(160, 1) attn_fd_kernel(const __grid_constant__ CUtensorMap tmK,
                                                        const __grid_constant__ CUtensorMap tmV,
                                                        const __grid_constant__ CUtensorMap tmK4,
                                                        const __grid_constant__ CUtensorMap tmV4, AttnParams p,
                                                        int ntiles, int nseg_max, int seg_keys, int n_items) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  const uint32_t raw = smem_u32(sm_raw);
  uint8_t* sm = sm_raw + (((raw + 1023u) & ~1023u) - raw);
  const uint32_t sbase = smem_u32(sm);
  float* mrg = reinterpret_cast<float*>(sm + NST * STAGE_BYTES);  // [4][16][HD] O, then [4][16] m, l
  float* mrg_m = mrg + 4 * 16 * HD;
  float* mrg_l = mrg_m + 4 * 16;
  uint64_t* full = reinterpret_cast<uint64_t*>(mrg_l + 4 * 16);
  uint64_t* empty = full + NST;
  int* mrg_flag = reinterpret_cast<int*>(empty + NST);

  KtScope kt_(KT_ATTN, (uint32_t)p.q_len);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int G = p.Hq / p.Hkv;
  const int R = p.q_len * G;

  // segment-major item order: consecutive CTAs take different groups' segment s, so the long
  // (full) and short (tail) segments spread evenly over the persistent CTAs
  const int n_groups = p.B * p.Hkv * ntiles;
  const int seg_ch = seg_keys / CH;
  auto item_of = [&](int idx, Item& it) {
    int r = idx % n_groups;
    it.seg = idx / n_groups;
    it.qt = r % ntiles;
    r /= ntiles;
    it.kvh = r % p.Hkv;
    it.b = r / p.Hkv;
    const int r0 = it.qt * 16;
    const int nr = min(16, R - r0);
    const int kmax = min(p.pos0[it.b] + min(p.q_len - 1, (r0 + nr - 1) / G), p.max_key - 1);
    const int nch = kmax / CH + 1;
    it.nseg = (nch + seg_ch - 1) / seg_ch;
    it.c0 = it.seg * seg_ch;
    it.c1 = min(nch, it.c0 + seg_ch);  // empty when seg >= nseg
    return kmax;
  };

  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);  // one arrival per compute warp
    }
    fence_barrier_init();
  }
  // pages past a sequence's last key are not loaded; their (masked, p = 0) V rows must be finite
  for (int i = tid; i < NST * STAGE_BYTES / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0u, 0u, 0u, 0u);
  fence_proxy_async();
  __syncthreads();
  pdl_wait();  // queries, lengths and the new KV rows come from the previous kernels
  kt_.mark();
  pdl_trigger();

  if (warp == 4) {
    // ---- TMA producer
    int seq = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      Item it;
      const int kmax = item_of(item, it);
      for (int c = it.c0; c < it.c1; ++c, ++seq) {
        const int st = seq % NST;
        mbar_wait(&empty[st], ((uint32_t)(seq / NST) & 1u) ^ 1u);
        const int kstart = c * CH;
        const int npages = (min(CH, kmax + 1 - kstart) + 15) / 16;
        const int pg = (lane < npages) ? p.block_table[it.b * p.pages_per_seq + kstart / 16 + lane] : 0;
        const int pg0 = __shfl_sync(0xffffffffu, pg, 0);
        // the chunk's pages are consecutive in the pool (the identity page table, and any run of a
        // permuted one): 4 TMA boxes of 8 pages x 16 keys x 64 dims instead of 32 one-page boxes
        // (pages past the sequence's last key are masked; the pool is zero-initialised, so they are finite)
        const bool run = __all_sync(0xffffffffu, lane >= npages || pg == pg0 + lane);
        if (run) {
          if (lane == 0) {
            mbar_arrive_expect_tx(&full[st], (uint32_t)(4 * 8 * 16 * 128));
            uint8_t* kb = sm + st * STAGE_BYTES;
            uint8_t* vb = kb + KV_BYTES;
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              tma_load_4d(kb + hf * (CH * 128), &tmK4, &full[st], hf * 64, 0, it.kvh, pg0, kEvictFirst);
              tma_load_4d(vb + hf * (CH * 128), &tmV4, &full[st], hf * 64, 0, it.kvh, pg0, kEvictFirst);
            }
          }
          __syncwarp();
          continue;
        }
        if (lane == 0) mbar_arrive_expect_tx(&full[st], (uint32_t)(npages * 4 * 16 * 128));
        __syncwarp();
        for (int i = 0; i < npages; ++i) {
          const int blk = __shfl_sync(0xffffffffu, pg, i);
          if (lane == 0) {
            const int row = (blk * p.Hkv + it.kvh) * 16;
            uint8_t* kb = sm + st * STAGE_BYTES;
            uint8_t* vb = kb + KV_BYTES;
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              tma_load_2d(kb + hf * (CH * 128) + i * 16 * 128, &tmK, &full[st], hf * 64, row, kEvictFirst);
              tma_load_2d(vb + hf * (CH * 128) + i * 16 * 128, &tmV, &full[st], hf * 64, row, kEvictFirst);
            }
          }
        }
        __syncwarp();
      }
    }
    return;
  }

  // ---- compute warps
  const float scale_log2 = 0.08838834764831845f * 1.4426950408889634f;  // log2(e) / sqrt(128)
  int seq = 0;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    Item it;
    item_of(item, it);
    if (it.c0 >= it.c1) continue;  // segment beyond this group's keys
    const unsigned long long ti0 = g_kt.rec ? kt_now() : 0ull;
    const int r0 = it.qt * 16;
    const int nr = min(16, R - r0);
    const int base = p.pos0[it.b];
    // Q fragments (rows g, g+8 of the tile) from the fp32 rotated queries
    uint32_t qa[8][4];
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
      const int r = g + 8 * hr;
      const bool ok = r < nr;
      const int rr = r0 + (ok ? r : 0), qi = rr / G, h = it.kvh * G + rr % G;
      // bf16 rotated queries (rope_append rounded them RNE)
      const uint32_t* qrow = reinterpret_cast<const uint32_t*>(reinterpret_cast<const __nv_bfloat16*>(p.q) +
                                                               ((size_t)(it.b * p.q_len + qi) * p.Hq + h) * HD);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int d0 = kk * 16 + 2 * t4;
        qa[kk][hr] = ok ? qrow[d0 / 2] : 0u;
        qa[kk][2 + hr] = ok ? qrow[(d0 + 8) / 2] : 0u;
      }
    }
    const int pos_lo = base + (r0 + g) / G, pos_hi = base + (r0 + g + 8) / G;
    const bool row_lo = g < nr, row_hi = g + 8 < nr;
    float m_lo = -INFINITY, m_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;  // log2-domain running max
    float o[16][4];
#pragma unroll
    for (int nt = 0; nt < 16; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) o[nt][i] = 0.f;

    for (int c = it.c0; c < it.c1; ++c, ++seq) {
      const int st = seq % NST;
      mbar_wait(&full[st], (uint32_t)(seq / NST) & 1u);
      const uint32_t kb = sbase + st * STAGE_BYTES, vb = kb + KV_BYTES;
      const int kstart = c * CH + warp * 32;
      // S = Q K_w^T for this warp's 32 keys
      float s[4][4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) s[nt][i] = 0.f;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int key = warp * 32 + nt * 8 + (lane & 7);
#pragma unroll
        for (int kp = 0; kp < 4; ++kp) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4(kb + swz(key, kp * 4 + (lane >> 3)), b0, b1, b2, b3);
          mma16816(s[nt], qa[2 * kp], b0, b1);
          mma16816(s[nt], qa[2 * kp + 1], b2, b3);
        }
      }
      // mask, new running max (exact; masked entries excluded)
      float cm_lo = -INFINITY, cm_hi = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int key = kstart + nt * 8 + 2 * t4 + (i & 1);
          const bool hi = i >= 2;
          const bool vis = hi ? (row_hi && key <= pos_hi) : (row_lo && key <= pos_lo);
          const float v = vis ? s[nt][i] * scale_log2 : -INFINITY;
          s[nt][i] = v;
          if (hi) cm_hi = fmaxf(cm_hi, v); else cm_lo = fmaxf(cm_lo, v);
        }
#pragma unroll
      for (int off = 1; off <= 2; off <<= 1) {
        cm_lo = fmaxf(cm_lo, __shfl_xor_sync(0xffffffffu, cm_lo, off));
        cm_hi = fmaxf(cm_hi, __shfl_xor_sync(0xffffffffu, cm_hi, off));
      }
      const float mn_lo = fmaxf(m_lo, cm_lo), mn_hi = fmaxf(m_hi, cm_hi);
      const float a_lo = (mn_lo == -INFINITY) ? 1.f : exp2f(m_lo - mn_lo);
      const float a_hi = (mn_hi == -INFINITY) ? 1.f : exp2f(m_hi - mn_hi);
      m_lo = mn_lo;
      m_hi = mn_hi;
      // P (bf16 A fragments straight from the S accumulators) and its row sums
      uint32_t pa[2][4];
      float ps_lo = 0.f, ps_hi = 0.f;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        float e[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float M = i >= 2 ? mn_hi : mn_lo;
          e[i] = (s[nt][i] == -INFINITY) ? 0.f : exp2f(s[nt][i] - M);
        }
        ps_lo += e[0] + e[1];
        ps_hi += e[2] + e[3];
        // k-step kk = nt/2 (16 keys): a0,a1 = n-tile 2kk (rows g, g+8); a2,a3 = n-tile 2kk+1
        pa[nt >> 1][(nt & 1) * 2 + 0] = pack_bf16(e[0], e[1]);
        pa[nt >> 1][(nt & 1) * 2 + 1] = pack_bf16(e[2], e[3]);
      }
#pragma unroll
      for (int off = 1; off <= 2; off <<= 1) {
        ps_lo += __shfl_xor_sync(0xffffffffu, ps_lo, off);
        ps_hi += __shfl_xor_sync(0xffffffffu, ps_hi, off);
      }
      l_lo = l_lo * a_lo + ps_lo;
      l_hi = l_hi * a_hi + ps_hi;
#pragma unroll
      for (int nt = 0; nt < 16; ++nt) {
        o[nt][0] *= a_lo;
        o[nt][1] *= a_lo;
        o[nt][2] *= a_hi;
        o[nt][3] *= a_hi;
      }
      // O += P V_w: 2 k-steps (this warp's 32 keys) x 16 n-tiles (128 dims)
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const uint32_t a[4] = {pa[kk][0], pa[kk][1], pa[kk][2], pa[kk][3]};
#pragma unroll
        for (int np = 0; np < 8; ++np) {
          const int mi = lane >> 3, ri = lane & 7;
          const int key = warp * 32 + kk * 16 + (mi & 1) * 8 + ri;
          const int chunk = np * 2 + (mi >> 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(vb + swz(key, chunk), b0, b1, b2, b3);
          mma16816(o[2 * np], a, b0, b1);
          mma16816(o[2 * np + 1], a, b2, b3);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);  // this warp is done with the stage
    }
    const unsigned long long ti1 = g_kt.rec ? kt_now() : 0ull;
    // ---- merge the 4 warp states in fixed order and normalise
    if (g < nr) {  // (rows of the tile past the block's rows are never read)
#pragma unroll
      for (int nt = 0; nt < 16; ++nt)
        *reinterpret_cast<float2*>(mrg + (warp * 16 + g) * HD + nt * 8 + 2 * t4) = make_float2(o[nt][0], o[nt][1]);
    }
    if (g + 8 < nr) {
#pragma unroll
      for (int nt = 0; nt < 16; ++nt)
        *reinterpret_cast<float2*>(mrg + (warp * 16 + g + 8) * HD + nt * 8 + 2 * t4) = make_float2(o[nt][2], o[nt][3]);
    }
    if (t4 == 0) {
      mrg_m[warp * 16 + g] = m_lo;
      mrg_m[warp * 16 + g + 8] = m_hi;
      mrg_l[warp * 16 + g] = l_lo;
      mrg_l[warp * 16 + g + 8] = l_hi;
    }
    named_bar(1, 128);
    // per-row merge factors once (row r: thread r): M = max_w m_w, f_w = 2^(m_w - M), L = sum_w l_w f_w
    // (same values and order as forming them per element)
    if (tid < nr) {
      const int r = tid;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < 4; ++w) M = fmaxf(M, mrg_m[w * 16 + r]);
      float L = 0.f;
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const float f = (mrg_m[w * 16 + r] == -INFINITY) ? 0.f : exp2f(mrg_m[w * 16 + r] - M);
        L += mrg_l[w * 16 + r] * f;
        mrg_m[w * 16 + r] = f;
      }
      mrg_l[r] = L;
      mrg_l[16 + r] = M;
    }
    named_bar(1, 128);
    const int group = (it.b * p.Hkv + it.kvh) * ntiles + it.qt;
    for (int e = tid; e < nr * HD; e += 128) {
      const int r = e / HD, d = e % HD;
      float acc = 0.f;
#pragma unroll
      for (int w = 0; w < 4; ++w) acc += mrg[(w * 16 + r) * HD + d] * mrg_m[w * 16 + r];
      const float L = mrg_l[r];
      const int rr = r0 + r, qi = rr / G, h = it.kvh * G + rr % G;
      const int t = it.b * p.q_len + qi;
      if (it.nseg == 1) {
        reinterpret_cast<__nv_bfloat16*>(p.out)[((size_t)t * p.Hq + h) * HD + d] = __float2bfloat16_rn(acc / L);
      } else {
        const size_t slot = ((size_t)t * p.Hq + h) * p.nchunk_max + it.seg;
        p.part_o[slot * HD + d] = acc;
        if (d == 0) {
          p.part_ml[2 * slot] = mrg_l[16 + r];
          p.part_ml[2 * slot + 1] = L;
        }
      }
    }
    if (it.nseg > 1) {
      // one gpu-scope release per item (cumulative over the compute warps' partial writes, which
      // the CTA barrier orders before it) instead of a fence in every thread
      named_bar(1, 128);
      if (tid == 0) {
        int prev;
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(prev) : "l"(p.seg_cnt + group) : "memory");
        mrg_flag[0] = prev == it.nseg - 1;
      }
      named_bar(1, 128);
      if (mrg_flag[0]) {  // every segment of the group has landed: merge them in segment order
        for (int e = tid; e < nr * HD; e += 128) {
          const int r = e / HD, d = e % HD;
          const int rr = r0 + r, qi = rr / G, h = it.kvh * G + rr % G;
          const int t = it.b * p.q_len + qi;
          const size_t s0 = ((size_t)t * p.Hq + h) * p.nchunk_max;
          float M = -INFINITY;
          for (int sg = 0; sg < it.nseg; ++sg) M = fmaxf(M, __ldcg(&p.part_ml[2 * (s0 + sg)]));
          float L = 0.f, acc = 0.f;
          for (int sg = 0; sg < it.nseg; ++sg) {
            const float ms = __ldcg(&p.part_ml[2 * (s0 + sg)]);
            const float f = (ms == -INFINITY) ? 0.f : exp2f(ms - M);
            L += __ldcg(&p.part_ml[2 * (s0 + sg) + 1]) * f;
            acc += __ldcg(&p.part_o[(s0 + sg) * HD + d]) * f;
          }
          reinterpret_cast<__nv_bfloat16*>(p.out)[((size_t)t * p.Hq + h) * HD + d] = __float2bfloat16_rn(acc / L);
        }
        if (tid == 0) p.seg_cnt[group] = 0;  // re-arm for the next launch
      }
    }
    named_bar(1, 128);
    if (tid == 0 && g_kt.rec) kt_item((uint32_t)(it.seg | (it.nseg << 8) | ((it.c1 - it.c0) << 16)), ti0, ti1, kt_now());
  }
}

static bool encode_kv_map(CUtensorMap* m, const void* base, long long rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t dims[2] = {(cuuint64_t)HD, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)HD * 2};
  cuuint32_t box[2] = {64, 16};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the pool as [pages][Hkv][16 keys][hd]: box = 8 consecutive pages x 16 keys x 1 head x 64 dims
static bool encode_kv_map4(CUtensorMap* m, const void* base, int Hkv, long long n_pages) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t dims[4] = {(cuuint64_t)HD, 16, (cuuint64_t)Hkv, (cuuint64_t)n_pages};
  cuuint64_t strides[3] = {(cuuint64_t)HD * 2, (cuuint64_t)16 * HD * 2, (cuuint64_t)Hkv * 16 * HD * 2};
  cuuint32_t box[4] = {64, 16, 1, 8};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t launch_attention_fd(const AttnParams& p, cudaStream_t s) {
  static bool attr = false;
  static int num_sms = 148;
  if (!attr) {
    cudaFuncSetAttribute(attn_fd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    attr = true;
  }
  const int G = p.Hq / p.Hkv;
  const int ntiles = (p.q_len * G + 15) / 16;
  // segment size override (tests exercise the multi-segment fold at short contexts; read per launch)
  const int env_seg = getenv("SF_ATTN_SEG") ? atoi(getenv("SF_ATTN_SEG")) : 0;
  const int seg_keys = (env_seg >= CH && env_seg % CH == 0) ? env_seg : kAttnSeg;
  const int nseg_max = (p.max_key + seg_keys - 1) / seg_keys;
  if (nseg_max > p.nchunk_max || !p.seg_cnt) return cudaErrorInvalidValue;
  const int n_items = p.B * p.Hkv * ntiles * nseg_max;
  const int grid = std::min(n_items, num_sms);
  CUtensorMap mk, mv;
  const long long rows = (long long)p.n_pages * p.Hkv * 16;
  CUtensorMap mk4, mv4;
  if (!encode_kv_map(&mk, p.Kp, rows) || !encode_kv_map(&mv, p.Vp, rows)) return cudaErrorInvalidValue;
  if (!encode_kv_map4(&mk4, p.Kp, p.Hkv, p.n_pages) || !encode_kv_map4(&mv4, p.Vp, p.Hkv, p.n_pages))
    return cudaErrorInvalidValue;
  launch_k(attn_fd_kernel, dim3(grid), dim3(160), SMEM, s, mk, mv, mk4, mv4, p, ntiles, nseg_max, seg_keys, n_items);
  return cudaGetLastError();
}

cudaError_t kt_setup_attn_fd(void* rec, unsigned* cnt, unsigned cap) {
  KtBuf b;
  b.rec = reinterpret_cast<KtRec*>(rec);
  b.cnt = cnt;
  b.cap = cap;
  return kt_setup_tu(b);
}

}  // namespace sf
