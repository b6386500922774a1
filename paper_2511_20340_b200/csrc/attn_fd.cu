// attn_fd.cu -- bf16 hybrid-mask paged decode attention (mode CAUSAL_PREFIX), flash-decoding form.
//
// Work: (sequence b, kv head, 16-row query tile) groups. Keys are cut into fixed SEG-key segments
// (absolute positions) and the arithmetic is defined segment-wise:
//   per segment s and warp w: an online softmax over w's 32-key slice of each of the segment's
//     128-key chunks, starting fresh -> (m, l, O)_{s,w}   (S = Q K^T and O += P V by mma.sync bf16,
//     masked keys excluded, P kept in registers);
//   per warp: fold the segment states in order s = 0, 1, ...: M = max, f = 2^(m - M),
//     l = l_a f_a + l_b f_b, O = O_a f_a + O_b f_b (explicitly rounded products);
//   across warps: the same merge in the fixed order w = 0..3, then out = acc / L.
// Two schedules compute exactly this (bit-identical results): a CTA per group walking all its
// segments (folds in registers; large batches), or a CTA per (group, segment) for small batches,
// which publishes its four warp states; the CTA completing a group's last segment (arrival
// counter) folds them and merges. A producer warp streams the chunks with TMA into a 3-stage ring.
// Every row's arithmetic depends only on its own keys (batch invariance, C23).
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
                                                        int ntiles, int nseg_max, int seg_keys, int n_items,
                                                        int split_arg) {
  const int split = split_arg & 1;
  const bool probe = (split_arg & 2) != 0;  // (SF_ATTN_PROBE, measurement only: stream the chunks, no math)
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
    it.seg = split ? idx / n_groups : 0;
    it.qt = r % ntiles;
    r /= ntiles;
    it.kvh = r % p.Hkv;
    it.b = r / p.Hkv;
    const int r0 = it.qt * 16;
    const int nr = min(16, R - r0);
    const int kmax = min(p.pos0[it.b] + attn_row_last(p, min(p.q_len - 1, (r0 + nr - 1) / G)), p.max_key - 1);
    const int nch = kmax / CH + 1;
    it.nseg = (nch + seg_ch - 1) / seg_ch;
    it.c0 = split ? it.seg * seg_ch : 0;
    it.c1 = split ? min(nch, it.c0 + seg_ch) : nch;  // empty when seg >= nseg
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
    const int pos_lo = base + attn_row_last(p, (r0 + g) / G), pos_hi = base + attn_row_last(p, (r0 + g + 8) / G);
    const bool row_lo = g < nr, row_hi = g + 8 < nr;
    float m_lo = -INFINITY, m_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;  // log2-domain running max
    float o[16][4];
#pragma unroll
    for (int nt = 0; nt < 16; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) o[nt][i] = 0.f;
    // this warp's fold of its finished segments (starts empty: fold(empty, x) == x exactly)
    float tm_lo = -INFINITY, tm_hi = -INFINITY, tl_lo = 0.f, tl_hi = 0.f;
    float to[16][4];
#pragma unroll
    for (int nt = 0; nt < 16; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) to[nt][i] = 0.f;
    auto fold_segment = [&]() {
      const float M_lo = fmaxf(tm_lo, m_lo), M_hi = fmaxf(tm_hi, m_hi);
      const float ft_lo = (tm_lo == -INFINITY) ? 0.f : exp2f(tm_lo - M_lo);
      const float fc_lo = (m_lo == -INFINITY) ? 0.f : exp2f(m_lo - M_lo);
      const float ft_hi = (tm_hi == -INFINITY) ? 0.f : exp2f(tm_hi - M_hi);
      const float fc_hi = (m_hi == -INFINITY) ? 0.f : exp2f(m_hi - M_hi);
      tl_lo = __fadd_rn(__fmul_rn(tl_lo, ft_lo), __fmul_rn(l_lo, fc_lo));
      tl_hi = __fadd_rn(__fmul_rn(tl_hi, ft_hi), __fmul_rn(l_hi, fc_hi));
#pragma unroll
      for (int nt = 0; nt < 16; ++nt) {
        to[nt][0] = __fadd_rn(__fmul_rn(to[nt][0], ft_lo), __fmul_rn(o[nt][0], fc_lo));
        to[nt][1] = __fadd_rn(__fmul_rn(to[nt][1], ft_lo), __fmul_rn(o[nt][1], fc_lo));
        to[nt][2] = __fadd_rn(__fmul_rn(to[nt][2], ft_hi), __fmul_rn(o[nt][2], fc_hi));
        to[nt][3] = __fadd_rn(__fmul_rn(to[nt][3], ft_hi), __fmul_rn(o[nt][3], fc_hi));
      }
      tm_lo = M_lo;
      tm_hi = M_hi;
      m_lo = m_hi = -INFINITY;
      l_lo = l_hi = 0.f;
#pragma unroll
      for (int nt = 0; nt < 16; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) o[nt][i] = 0.f;
    };

    for (int c = it.c0; c < it.c1; ++c, ++seq) {
      if (c != it.c0 && c % seg_ch == 0) fold_segment();  // segment boundary (group schedule)
      const int st = seq % NST;
      mbar_wait(&full[st], (uint32_t)(seq / NST) & 1u);
      if (probe) {  // (finite output: a state of one unit-weight zero row)
        m_lo = m_hi = 0.f;
        l_lo = l_hi = 1.f;
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        continue;
      }
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
      // (no row of the warp raised its max: every factor is exactly 1 and the rescale is the identity)
      if (!__all_sync(0xffffffffu, a_lo == 1.f && a_hi == 1.f)) {
#pragma unroll
        for (int nt = 0; nt < 16; ++nt) {
          o[nt][0] *= a_lo;
          o[nt][1] *= a_lo;
          o[nt][2] *= a_hi;
          o[nt][3] *= a_hi;
        }
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
    fold_segment();
    const int group = (it.b * p.Hkv + it.kvh) * ntiles + it.qt;
    auto row_slot = [&](int r) {  // (token, head) of tile row r
      const int rr = r0 + r, qi = rr / G, h = it.kvh * G + rr % G;
      return (size_t)(it.b * p.q_len + qi) * p.Hq + h;
    };
    if (split && it.nseg > 1) {
      // ---- segment schedule: publish this segment's four warp states
      auto pub = [&](int r, int hsel) {
        const size_t base = (row_slot(r) * p.nchunk_max + it.seg) * 4 + warp;
#pragma unroll
        for (int nt = 0; nt < 16; ++nt)
          *reinterpret_cast<float2*>(p.part_o + base * HD + nt * 8 + 2 * t4) =
              make_float2(to[nt][2 * hsel], to[nt][2 * hsel + 1]);
        if (t4 == 0) {
          p.part_ml[2 * base] = hsel ? tm_hi : tm_lo;
          p.part_ml[2 * base + 1] = hsel ? tl_hi : tl_lo;
        }
      };
      if (g < nr) pub(g, 0);
      if (g + 8 < nr) pub(g + 8, 1);
      named_bar(1, 128);
      if (tid == 0) {
        int prev;
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(prev) : "l"(p.seg_cnt + group) : "memory");
        mrg_flag[0] = prev == it.nseg - 1;
        if (prev == it.nseg - 1) p.seg_cnt[group] = 0;  // re-arm for the next launch
      }
      named_bar(1, 128);
      if (!mrg_flag[0]) continue;
      // the group's last segment: fold every warp slot's segment states in segment order (the same
      // operations as the in-register fold). Step factors per (warp, row) first (one thread each),
      // then every thread (one dimension) streams the O values, all segments of 4 (warp, row)
      // pairs in flight at a time.
      constexpr int SMAX = 8;
      float* fa_s = mrg;                   // [4][16][SMAX] factor of the running state, then
      float* fb_s = mrg + 4 * 16 * SMAX;   // of segment s; the O fold overwrites mrg[] afterwards
      const int nsg = min(it.nseg, SMAX);
      if (tid < 4 * nr) {
        const int w = tid / nr, r = tid % nr;
        const size_t s0 = row_slot(r) * p.nchunk_max;
        float m = -INFINITY, l = 0.f;
        for (int sg = 0; sg < nsg; ++sg) {
          const size_t bs = (s0 + sg) * 4 + w;
          const float ms = __ldcg(&p.part_ml[2 * bs]), ls = __ldcg(&p.part_ml[2 * bs + 1]);
          const float M = fmaxf(m, ms);
          const float fa = (m == -INFINITY) ? 0.f : exp2f(m - M);
          const float fb = (ms == -INFINITY) ? 0.f : exp2f(ms - M);
          l = __fadd_rn(__fmul_rn(l, fa), __fmul_rn(ls, fb));
          m = M;
          fa_s[(w * 16 + r) * SMAX + sg] = fa;
          fb_s[(w * 16 + r) * SMAX + sg] = fb;
        }
        mrg_m[w * 16 + r] = m;
        mrg_l[w * 16 + r] = l;
      }
      named_bar(1, 128);
      float Ofold[64];  // (warp, row) pairs x this thread's dimension d = tid
      for (int q0 = 0; q0 < 4 * nr; q0 += 4) {
        float Os[4][SMAX];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int q = min(q0 + j, 4 * nr - 1), w = q / nr, r = q % nr;
          const size_t s0 = row_slot(r) * p.nchunk_max;
#pragma unroll
          for (int sg = 0; sg < SMAX; ++sg)
            Os[j][sg] = (sg < nsg) ? __ldcg(&p.part_o[((s0 + sg) * 4 + w) * HD + tid]) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int q = min(q0 + j, 4 * nr - 1), w = q / nr, r = q % nr;
          float O = 0.f;
#pragma unroll
          for (int sg = 0; sg < SMAX; ++sg)
            if (sg < nsg)
              O = __fadd_rn(__fmul_rn(O, fa_s[(w * 16 + r) * SMAX + sg]), __fmul_rn(Os[j][sg], fb_s[(w * 16 + r) * SMAX + sg]));
          if (q0 + j < 4 * nr) Ofold[q0 + j] = O;
        }
      }
      named_bar(1, 128);  // factors consumed before mrg[] is overwritten
      for (int q = 0; q < 4 * nr; ++q) {
        const int w = q / nr, r = q % nr;
        mrg[(w * 16 + r) * HD + tid] = Ofold[q];
      }
    } else {
      // ---- merge the 4 warp states in fixed order and normalise
      if (g < nr) {  // (rows of the tile past the block's rows are never read)
#pragma unroll
        for (int nt = 0; nt < 16; ++nt)
          *reinterpret_cast<float2*>(mrg + (warp * 16 + g) * HD + nt * 8 + 2 * t4) = make_float2(to[nt][0], to[nt][1]);
      }
      if (g + 8 < nr) {
#pragma unroll
        for (int nt = 0; nt < 16; ++nt)
          *reinterpret_cast<float2*>(mrg + (warp * 16 + g + 8) * HD + nt * 8 + 2 * t4) =
              make_float2(to[nt][2], to[nt][3]);
      }
      if (t4 == 0) {
        mrg_m[warp * 16 + g] = tm_lo;
        mrg_m[warp * 16 + g + 8] = tm_hi;
        mrg_l[warp * 16 + g] = tl_lo;
        mrg_l[warp * 16 + g + 8] = tl_hi;
      }
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
    for (int e = tid; e < nr * HD; e += 128) {
      const int r = e / HD, d = e % HD;
      float acc = 0.f;
#pragma unroll
      for (int w = 0; w < 4; ++w) acc += mrg[(w * 16 + r) * HD + d] * mrg_m[w * 16 + r];
      reinterpret_cast<__nv_bfloat16*>(p.out)[row_slot(r) * HD + d] = __float2bfloat16_rn(acc / mrg_l[r]);
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
  return encode_tmap_cached(enc, m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                            CU_TENSOR_MAP_SWIZZLE_128B) == CUDA_SUCCESS;
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
  return encode_tmap_cached(enc, m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box,
                            CU_TENSOR_MAP_SWIZZLE_128B) == CUDA_SUCCESS;
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
  // schedule (the arithmetic is the same): a CTA per (group, segment) when the groups alone would
  // leave most SMs idle, else a CTA per group folding its segments in registers
  const int n_groups = p.B * p.Hkv * ntiles;
  const char* env_split = getenv("SF_ATTN_SPLIT");  // tests force either schedule
  const int split = (nseg_max > 1 && nseg_max <= 8) &&  // (the publishing fold holds <= 8 segments)
                    (env_split ? atoi(env_split) > 0 : 2 * n_groups <= num_sms);
  const int n_items = split ? n_groups * nseg_max : n_groups;
  const int grid = std::min(n_items, num_sms);
  CUtensorMap mk, mv;
  const long long rows = (long long)p.n_pages * p.Hkv * 16;
  CUtensorMap mk4, mv4;
  if (!encode_kv_map(&mk, p.Kp, rows) || !encode_kv_map(&mv, p.Vp, rows)) return cudaErrorInvalidValue;
  if (!encode_kv_map4(&mk4, p.Kp, p.Hkv, p.n_pages) || !encode_kv_map4(&mv4, p.Vp, p.Hkv, p.n_pages))
    return cudaErrorInvalidValue;
  static const int env_probe = getenv("SF_ATTN_PROBE") ? atoi(getenv("SF_ATTN_PROBE")) : 0;
  launch_k(attn_fd_kernel, dim3(grid), dim3(160), SMEM, s, mk, mv, mk4, mv4, p, ntiles, nseg_max, seg_keys, n_items,
           split | (env_probe ? 2 : 0));
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
