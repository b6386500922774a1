// attn_fd.cu -- bf16 hybrid-mask paged decode attention (mode CAUSAL_PREFIX), flash-decoding form.
//
// Work: (sequence b, kv head, 16-row query tile) groups. Keys are cut into fixed SEG-key segments
// (absolute positions) and the arithmetic is defined segment-wise:
//   per segment s and warp w: an online softmax over w's 32-key slice of each of the segment's
//     128-key chunks, starting fresh -> (m, l, O)_{s,w}   (S^T = K Q^T and O^T += V^T P^T by mma.sync
//     bf16 with the keys as MMA rows and the tile's query rows as one or two 8-column n-tiles -- a
//     decode block of <= 8 rows costs half the MMAs of a 16-row M tile; masked keys excluded, P^T
//     transposed into the PV operand in registers with movmatrix);
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
#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"

namespace sf {
namespace {

constexpr int HD = 128;
constexpr int CH = 128;
constexpr int NST = 3;
constexpr int KV_BYTES = CH * HD * 2;      // 32 KB
constexpr int STAGE_BYTES = 2 * KV_BYTES;  // 64 KB
constexpr int NW = kAttnWarps;      // compute warps
constexpr int KPW = CH / NW;         // keys per warp slice of a chunk (one 16-key m-tile)
constexpr int TR = kAttnTileRows;    // query rows per tile (one 8-column n-tile)
constexpr int NTHR = (NW + 1) * 32;  // + the TMA producer warp
static_assert(KPW == 16 && TR == 8, "one m-tile of keys and one n-tile of queries per warp");
constexpr int MERGE_BYTES = NW * TR * (HD + 2) * 4;  // per-warp O, m, l for the final merge
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
// transpose of an 8x8 b16 matrix held as the mma fragment layout (thread (g, t4): row g, columns 2 t4, +1)
SF_DEV uint32_t movmatrix_trans(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
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

// item = (b * Hkv + kvh) * ntiles + qt. Warps 0..NW-1 compute, warp NW produces.
__global__ void __launch_bounds__(NTHR, 1) attn_fd_kernel(const __grid_constant__ CUtensorMap tmK,
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
  float* mrg = reinterpret_cast<float*>(sm + NST * STAGE_BYTES);  // [NW][TR][HD] O, then [NW][TR] m, l
  float* mrg_m = mrg + NW * TR * HD;
  float* mrg_l = mrg_m + NW * TR;
  uint64_t* full = reinterpret_cast<uint64_t*>(mrg_l + NW * TR);
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
    const int r0 = it.qt * TR;
    const int nr = min(TR, R - r0);
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
      mbar_init(&empty[s], NW);  // one arrival per compute warp
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

  if (warp == NW) {
    // ---- TMA producer
    int seq = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      Item it;
      const int kmax = item_of(item, it);
      for (int c = it.c0; c < it.c1; ++c, ++seq) {
        const int st = seq % NST;
        const int kstart = c * CH;
        const int npages = (min(CH, kmax + 1 - kstart) + 15) / 16;
        // the chunk's page-table entries are requested before waiting for the slot (the load's latency
        // hides behind the wait instead of delaying the TMA issue once the slot is free)
        const int pg = (lane < npages) ? p.block_table[it.b * p.pages_per_seq + kstart / 16 + lane] : 0;
        mbar_wait(&empty[st], ((uint32_t)(seq / NST) & 1u) ^ 1u);
        const int pg0 = __shfl_sync(0xffffffffu, pg, 0);
        // a full chunk whose pages are consecutive in the pool (the identity page table, and any run of a
        // permuted one): 4 TMA boxes of 8 pages x 16 keys x 64 dims instead of 32 one-page boxes. A tail
        // chunk loads just its npages pages: boxes past the last key would be HBM bytes the math masks away
        // (~16% of the KV stream at a 512-key prompt); the stale rows left in the slot are finite
        const bool run = npages == 8 && __all_sync(0xffffffffu, lane >= npages || pg == pg0 + lane);
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

  // ---- compute warps. Keys are the MMA rows (S^T = K Q^T, O^T += V^T P^T): warp w's 16 keys of a chunk
  // are one m-tile, the tile's <= 8 query rows one 8-column n-tile. A column's arithmetic never depends
  // on the other columns or on the tile's row count (batch invariance, C23).
  const float scale_log2 = 0.08838834764831845f * 1.4426950408889634f;  // log2(e) / sqrt(128)
  const int mi = lane >> 3, ri = lane & 7;
  int seq = 0;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    Item it;
    item_of(item, it);
    if (it.c0 >= it.c1) continue;  // segment beyond this group's keys
    const unsigned long long ti0 = g_kt.rec ? kt_now() : 0ull;
    const int r0 = it.qt * TR;
    const int nr = min(TR, R - r0);
    const int base = p.pos0[it.b];
    // Q^T B fragments: query column q = g, dims kk*16 + 2 t4 (+1) and + 8 (bf16, rope_append's RNE)
    uint32_t qb[8][2];
    {
      const bool ok = g < nr;
      const int rr = r0 + (ok ? g : 0), qi = rr / G, h = it.kvh * G + rr % G;
      const uint32_t* qrow = reinterpret_cast<const uint32_t*>(reinterpret_cast<const __nv_bfloat16*>(p.q) +
                                                               ((size_t)(it.b * p.q_len + qi) * p.Hq + h) * HD);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int d0 = kk * 16 + 2 * t4;
        qb[kk][0] = ok ? qrow[d0 / 2] : 0u;
        qb[kk][1] = ok ? qrow[(d0 + 8) / 2] : 0u;
      }
    }
    // this thread's query columns q = 2 t4 + j: visibility bound (last visible key)
    int posq[2];
    bool okq[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int q = 2 * t4 + j;
      okq[j] = q < nr;
      posq[j] = base + attn_row_last(p, (r0 + min(q, nr - 1)) / G);
    }
    // the last key any column of the tile sees: a warp slice past it is fully masked, and its chunk step
    // would leave (m, l, O) unchanged -- the warp skips it
    int wlast = max(okq[0] ? posq[0] : -1, okq[1] ? posq[1] : -1);
#pragma unroll
    for (int off = 1; off <= 16; off <<= 1) wlast = max(wlast, __shfl_xor_sync(0xffffffffu, wlast, off));
    float m[2], l[2], tm[2], tl[2];  // per column: running max (log2 domain), sum; folded
#pragma unroll
    for (int j = 0; j < 2; ++j) m[j] = tm[j] = -INFINITY, l[j] = tl[j] = 0.f;
    // O^T accumulators: m-tile md = dims md*16 .. +15; [c]: (dim g | g+8, column 2 t4 | +1)
    float o[8][4], to[8][4];
#pragma unroll
    for (int md = 0; md < 8; ++md)
#pragma unroll
      for (int i = 0; i < 4; ++i) o[md][i] = to[md][i] = 0.f;
    // this warp's fold of its finished segments (starts empty: fold(empty, x) == x exactly)
    auto fold_segment = [&]() {
      float ft[2], fc[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const float M = fmaxf(tm[j], m[j]);
        ft[j] = (tm[j] == -INFINITY) ? 0.f : exp2f(tm[j] - M);
        fc[j] = (m[j] == -INFINITY) ? 0.f : exp2f(m[j] - M);
        tl[j] = __fadd_rn(__fmul_rn(tl[j], ft[j]), __fmul_rn(l[j], fc[j]));
        tm[j] = M;
        m[j] = -INFINITY;
        l[j] = 0.f;
      }
#pragma unroll
      for (int md = 0; md < 8; ++md)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          to[md][i] = __fadd_rn(__fmul_rn(to[md][i], ft[i & 1]), __fmul_rn(o[md][i], fc[i & 1]));
          o[md][i] = 0.f;
        }
    };

    for (int c = it.c0; c < it.c1; ++c, ++seq) {
      if (c != it.c0 && c % seg_ch == 0) fold_segment();  // segment boundary (group schedule)
      const int st = seq % NST;
      mbar_wait(&full[st], (uint32_t)(seq / NST) & 1u);
      const int kstart = c * CH + warp * KPW;
      if (probe) {  // (finite output: a state of one unit-weight zero row)
#pragma unroll
        for (int j = 0; j < 2; ++j) m[j] = 0.f, l[j] = 1.f;
      } else if (kstart <= wlast) {  // (warp-uniform)
        const uint32_t kb = sbase + st * STAGE_BYTES, vb = kb + KV_BYTES;
        // S^T = K_w Q^T: 16 keys x 8 columns, 8 k-steps of 16 dims (two independent accumulator chains)
        float s[4] = {0.f, 0.f, 0.f, 0.f}, s2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int kk = 0; kk < 8; kk += 2) {
          uint32_t a[4], a2[4];
          ldsm_x4(kb + swz(warp * KPW + (mi & 1) * 8 + ri, kk * 2 + (mi >> 1)), a[0], a[1], a[2], a[3]);
          ldsm_x4(kb + swz(warp * KPW + (mi & 1) * 8 + ri, kk * 2 + 2 + (mi >> 1)), a2[0], a2[1], a2[2], a2[3]);
          mma16816(s, a, qb[kk][0], qb[kk][1]);
          mma16816(s2, a2, qb[kk + 1][0], qb[kk + 1][1]);
        }
        // mask, new running max per column (exact; masked entries excluded)
        float cm[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int key = kstart + g + 8 * (i >> 1), j = i & 1;
          const bool vis = okq[j] && key <= posq[j];
          const float v = vis ? (s[i] + s2[i]) * scale_log2 : -INFINITY;
          s[i] = v;
          cm[j] = fmaxf(cm[j], v);
        }
        float af[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
#pragma unroll
          for (int off = 4; off <= 16; off <<= 1) cm[j] = fmaxf(cm[j], __shfl_xor_sync(0xffffffffu, cm[j], off));
          const float mn = fmaxf(m[j], cm[j]);
          af[j] = (mn == -INFINITY) ? 1.f : exp2f(m[j] - mn);
          m[j] = mn;
        }
        // P^T and its column sums; P^T's 8x8 blocks transposed in registers into the PV B fragments
        float e[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) e[i] = (s[i] == -INFINITY) ? 0.f : exp2f(s[i] - m[i & 1]);
        float ps[2] = {e[0] + e[2], e[1] + e[3]};
        const uint32_t pb0 = movmatrix_trans(pack_bf16(e[0], e[1]));  // keys 0..7 of the slice
        const uint32_t pb1 = movmatrix_trans(pack_bf16(e[2], e[3]));  // keys 8..15
#pragma unroll
        for (int j = 0; j < 2; ++j) {
#pragma unroll
          for (int off = 4; off <= 16; off <<= 1) ps[j] += __shfl_xor_sync(0xffffffffu, ps[j], off);
          l[j] = l[j] * af[j] + ps[j];
        }
        // (no column of the warp raised its max: every factor is exactly 1 and the rescale is the identity)
        if (!__all_sync(0xffffffffu, af[0] == 1.f && af[1] == 1.f)) {
#pragma unroll
          for (int md = 0; md < 8; ++md)
#pragma unroll
            for (int i = 0; i < 4; ++i) o[md][i] *= af[i & 1];
        }
        // O^T += V_w^T P^T: m-tiles md (16 dims), one k-step (the slice's 16 keys)
#pragma unroll
        for (int md = 0; md < 8; ++md) {
          uint32_t a[4];
          ldsm_x4_t(vb + swz(warp * KPW + (mi >> 1) * 8 + ri, md * 2 + (mi & 1)), a[0], a[1], a[2], a[3]);
          mma16816(o[md], a, pb0, pb1);
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
      // ---- segment schedule: publish this segment's warp states
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int q = 2 * t4 + j;
        if (q >= nr) continue;
        const size_t bq = (row_slot(q) * p.nchunk_max + it.seg) * NW + warp;
#pragma unroll
        for (int md = 0; md < 8; ++md) {
          p.part_o[bq * HD + md * 16 + g] = to[md][j];
          p.part_o[bq * HD + md * 16 + g + 8] = to[md][2 + j];
        }
        if (g == 0) {
          p.part_ml[2 * bq] = tm[j];
          p.part_ml[2 * bq + 1] = tl[j];
        }
      }
      named_bar(1, NW * 32);
      if (tid == 0) {
        int prev;
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(prev) : "l"(p.seg_cnt + group) : "memory");
        mrg_flag[0] = prev == it.nseg - 1;
        if (prev == it.nseg - 1) p.seg_cnt[group] = 0;  // re-arm for the next launch
      }
      named_bar(1, NW * 32);
      if (!mrg_flag[0]) continue;
      // the group's last segment: fold every warp slot's segment states in segment order (the same
      // operations as the in-register fold). Step factors per (warp, row) first (one thread each),
      // then every thread (one dimension, one parity of the (warp, row) pairs) streams the O values,
      // all segments of 4 pairs in flight at a time.
      constexpr int SMAX = 8;
      float* fa_s = mrg;                    // [NW][TR][SMAX] factor of the running state, then
      float* fb_s = mrg + NW * TR * SMAX;   // of segment s; the O fold overwrites mrg[] afterwards
      const int nsg = min(it.nseg, SMAX);
      if (tid < NW * nr) {
        const int w = tid / nr, r = tid % nr;
        const size_t s0 = row_slot(r) * p.nchunk_max;
        float m = -INFINITY, l = 0.f;
        for (int sg = 0; sg < nsg; ++sg) {
          const size_t bs = (s0 + sg) * NW + w;
          const float ms = __ldcg(&p.part_ml[2 * bs]), ls = __ldcg(&p.part_ml[2 * bs + 1]);
          const float M = fmaxf(m, ms);
          const float fa = (m == -INFINITY) ? 0.f : exp2f(m - M);
          const float fb = (ms == -INFINITY) ? 0.f : exp2f(ms - M);
          l = __fadd_rn(__fmul_rn(l, fa), __fmul_rn(ls, fb));
          m = M;
          fa_s[(w * TR + r) * SMAX + sg] = fa;
          fb_s[(w * TR + r) * SMAX + sg] = fb;
        }
        mrg_m[w * TR + r] = m;
        mrg_l[w * TR + r] = l;
      }
      named_bar(1, NW * 32);
      const int d = tid & (HD - 1), par = tid >> 7;  // dimension, pair parity
      const int npair = NW * nr;                      // (warp, row) pairs q = w nr + r
      float Ofold[NW * TR / 2];
      for (int i0 = 0; 2 * i0 < npair; i0 += 4) {
        float Os[4][SMAX];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int q = min(2 * (i0 + j) + par, npair - 1), w = q / nr, r = q % nr;
          const size_t s0 = row_slot(r) * p.nchunk_max;
#pragma unroll
          for (int sg = 0; sg < SMAX; ++sg)
            Os[j][sg] = (sg < nsg) ? __ldcg(&p.part_o[((s0 + sg) * NW + w) * HD + d]) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int q = min(2 * (i0 + j) + par, npair - 1), w = q / nr, r = q % nr;
          float O = 0.f;
#pragma unroll
          for (int sg = 0; sg < SMAX; ++sg)
            if (sg < nsg)
              O = __fadd_rn(__fmul_rn(O, fa_s[(w * TR + r) * SMAX + sg]), __fmul_rn(Os[j][sg], fb_s[(w * TR + r) * SMAX + sg]));
          if (i0 + j < NW * TR / 2) Ofold[i0 + j] = O;
        }
      }
      named_bar(1, NW * 32);  // factors consumed before mrg[] is overwritten
      for (int i = 0; 2 * i + par < npair; ++i) {
        const int q = 2 * i + par, w = q / nr, r = q % nr;
        mrg[(w * TR + r) * HD + d] = Ofold[i];
      }
    } else {
      // ---- the warp states, for the merge in fixed order
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int q = 2 * t4 + j;
        if (q < nr) {  // (rows of the tile past the block's rows are never read)
#pragma unroll
          for (int md = 0; md < 8; ++md) {
            mrg[(warp * TR + q) * HD + md * 16 + g] = to[md][j];
            mrg[(warp * TR + q) * HD + md * 16 + g + 8] = to[md][2 + j];
          }
          if (g == 0) {
            mrg_m[warp * TR + q] = tm[j];
            mrg_l[warp * TR + q] = tl[j];
          }
        }
      }
    }
    named_bar(1, NW * 32);
    // per-row merge factors once (row r: thread r): M = max_w m_w, f_w = 2^(m_w - M), L = sum_w l_w f_w
    // (same values and order as forming them per element)
    if (tid < nr) {
      const int r = tid;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < NW; ++w) M = fmaxf(M, mrg_m[w * TR + r]);
      float L = 0.f;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const float f = (mrg_m[w * TR + r] == -INFINITY) ? 0.f : exp2f(mrg_m[w * TR + r] - M);
        L += mrg_l[w * TR + r] * f;
        mrg_m[w * TR + r] = f;
      }
      mrg_l[r] = L;
    }
    named_bar(1, NW * 32);
    for (int e = tid; e < nr * HD; e += NW * 32) {
      const int r = e / HD, d = e % HD;
      float acc = 0.f;
#pragma unroll
      for (int w = 0; w < NW; ++w) acc += mrg[(w * TR + r) * HD + d] * mrg_m[w * TR + r];
      reinterpret_cast<__nv_bfloat16*>(p.out)[row_slot(r) * HD + d] = __float2bfloat16_rn(acc / mrg_l[r]);
    }
    named_bar(1, NW * 32);
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
  const int ntiles = (p.q_len * G + TR - 1) / TR;
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
  launch_k(attn_fd_kernel, dim3(grid), dim3(NTHR), SMEM, s, mk, mv, mk4, mv4, p, ntiles, nseg_max, seg_keys, n_items,
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
