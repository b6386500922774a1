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
constexpr int NTHR = (NW + 1) * 32;  // + the TMA producer warp
static_assert(KPW == 16, "one m-tile of keys per warp");
constexpr int kFoldSeg = 64;  // key segments one row can span (the fold's factor table in the merge buffer)
constexpr int MERGE_BYTES = NW * 8 * (HD + 2) * 4;  // per-warp O, m, l of 8 rows for the final merge
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

// item = (b * Hkv + kvh) * ntiles + qt. Warps 0..NW-1 compute, warp NW produces. NQ: 8-column n-tiles per
// query tile (tiles of 8 NQ rows; 2 when a sequence's (query, head) rows exceed 8, so each (sequence, kv
// head) streams its keys once for up to 16 rows)
template <int NQ>
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
  constexpr int TT = 8 * NQ;  // query rows per tile
  float* mrg = reinterpret_cast<float*>(sm + NST * STAGE_BYTES);  // [NW][8][HD] O, then [NW][8] m, l
  float* mrg_m = mrg + NW * 8 * HD;
  float* mrg_l = mrg_m + NW * 8;
  uint64_t* full = reinterpret_cast<uint64_t*>(mrg_l + NW * 8);
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
    const int r0 = it.qt * TT;
    const int nr = min(TT, R - r0);
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

  if (warp == NW) {
    // ---- TMA producer. Chunk c of item it into ring slot st (sequence number sq of this CTA's chunks)
    auto issue = [&](const Item& it, int kmax, int c, int sq, bool wait_slot) {
      const int st = sq % NST;
      const int kstart = c * CH;
      const int npages = (min(CH, kmax + 1 - kstart) + 15) / 16;
      // the chunk's page-table entries are requested before waiting for the slot (the load's latency
      // hides behind the wait instead of delaying the TMA issue once the slot is free)
      const int pg = (lane < npages) ? p.block_table[it.b * p.pages_per_seq + kstart / 16 + lane] : 0;
      if (wait_slot) mbar_wait(&empty[st], ((uint32_t)(sq / NST) & 1u) ^ 1u);
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
        return;
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
    };
    // Before the grid dependency resolves: the first item's leading chunks whose keys all precede its
    // sequence's first new row. They hold only KV rows written by earlier steps; the previous kernel (the
    // RoPE / append step) writes rows pos0 .. only. pos0 and the page table come from launches at least two
    // back, complete once this kernel runs (PDL: the previous kernel passed its own dependency wait).
    int pre = 0;
    if ((int)blockIdx.x < n_items) {
      Item it;
      const int kmax = item_of(blockIdx.x, it);
      const int base = p.pos0[it.b];
      for (int c = it.c0; c < it.c1 && pre < NST && (c + 1) * CH <= base; ++c, ++pre) issue(it, kmax, c, pre, false);
    }
    pdl_wait();  // the new KV rows (and, for the compute warps, the queries) come from the previous kernel
    kt_.mark();
    pdl_trigger();
    int seq = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      Item it;
      const int kmax = item_of(item, it);
      for (int c = it.c0; c < it.c1; ++c, ++seq)
        if (seq >= pre) issue(it, kmax, c, seq, true);
    }
    return;
  }
  pdl_wait();  // queries, lengths and the new KV rows come from the previous kernels
  kt_.mark();
  pdl_trigger();

  // ---- compute warps. Keys are the MMA rows (S^T = K Q^T, O^T += V^T P^T): warp w's 16 keys of a chunk
  // are one m-tile, the tile's query rows one (NQ = 1) or two (NQ = 2) 8-column n-tiles sharing the K / V
  // fragments. A column's arithmetic never depends on the other columns, the n-tile count or the tile's
  // row count (batch invariance, C23; the same bits for 8- and 16-row tiles).
  const float scale_log2 = 0.08838834764831845f * 1.4426950408889634f;  // log2(e) / sqrt(128)
  const int mi = lane >> 3, ri = lane & 7;
  int seq = 0;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    Item it;
    item_of(item, it);
    if (it.c0 >= it.c1) continue;  // segment beyond this group's keys
    const unsigned long long ti0 = g_kt.rec ? kt_now() : 0ull;
    const int r0 = it.qt * TT;
    const int nr = min(TT, R - r0);
    const bool two = NQ == 2 && nr > 8;  // (warp-uniform) the second n-tile holds rows
    const int base = p.pos0[it.b];
    // Q^T B fragments: query column q = nq*8 + g, dims kk*16 + 2 t4 (+1) and + 8 (bf16, rope_append's RNE)
    uint32_t qb[NQ][8][2];
#pragma unroll
    for (int nq = 0; nq < NQ; ++nq) {
      const int r = nq * 8 + g;
      const bool ok = r < nr;
      const int rr = r0 + (ok ? r : 0), qi = rr / G, h = it.kvh * G + rr % G;
      const uint32_t* qrow = reinterpret_cast<const uint32_t*>(reinterpret_cast<const __nv_bfloat16*>(p.q) +
                                                               ((size_t)(it.b * p.q_len + qi) * p.Hq + h) * HD);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int d0 = kk * 16 + 2 * t4;
        qb[nq][kk][0] = ok ? qrow[d0 / 2] : 0u;
        qb[nq][kk][1] = ok ? qrow[(d0 + 8) / 2] : 0u;
      }
    }
    // this thread's query columns q = nq*8 + 2 t4 + j: visibility bound (last visible key)
    int posq[NQ][2];
    bool okq[NQ][2];
    int wlast = -1;  // the last key any column of the tile sees: a warp slice past it is skipped (its
                     // chunk step would leave (m, l, O) unchanged)
#pragma unroll
    for (int nq = 0; nq < NQ; ++nq)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int q = nq * 8 + 2 * t4 + j;
        okq[nq][j] = q < nr;
        posq[nq][j] = base + attn_row_last(p, (r0 + min(q, nr - 1)) / G);
        if (okq[nq][j]) wlast = max(wlast, posq[nq][j]);
      }
#pragma unroll
    for (int off = 1; off <= 16; off <<= 1) wlast = max(wlast, __shfl_xor_sync(0xffffffffu, wlast, off));
    float m[NQ][2], l[NQ][2];  // per column: running max (log2 domain), sum
#pragma unroll
    for (int nq = 0; nq < NQ; ++nq)
#pragma unroll
      for (int j = 0; j < 2; ++j) m[nq][j] = -INFINITY, l[nq][j] = 0.f;
    // O^T accumulators: m-tile md = dims md*16 .. +15, n-tile nq; [c]: (dim g | g+8, column 2 t4 | +1)
    float o[8][NQ][4];
#pragma unroll
    for (int md = 0; md < 8; ++md)
#pragma unroll
      for (int nq = 0; nq < NQ; ++nq)
#pragma unroll
        for (int i = 0; i < 4; ++i) o[md][nq][i] = 0.f;
    const auto row_slot = [&](int r) {  // (token, head) of tile row r
      const int rr = r0 + r, qi = rr / G, h = it.kvh * G + rr % G;
      return (size_t)(it.b * p.q_len + qi) * p.Hq + h;
    };
    // a finished key segment's warp state -> the partial buffer (folded in segment order at the end), and a
    // fresh state for the next segment
    auto publish_segment = [&](int sgi) {
#pragma unroll
      for (int nq = 0; nq < NQ; ++nq)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int q = nq * 8 + 2 * t4 + j;
          if (q < nr) {
            const size_t bq = (row_slot(q) * p.nchunk_max + sgi) * NW + warp;
#pragma unroll
            for (int md = 0; md < 8; ++md) {
              p.part_o[bq * HD + md * 16 + g] = o[md][nq][j];
              p.part_o[bq * HD + md * 16 + g + 8] = o[md][nq][2 + j];
            }
            if (g == 0) {
              p.part_ml[2 * bq] = m[nq][j];
              p.part_ml[2 * bq + 1] = l[nq][j];
            }
          }
          m[nq][j] = -INFINITY;
          l[nq][j] = 0.f;
        }
#pragma unroll
      for (int md = 0; md < 8; ++md)
#pragma unroll
        for (int nq = 0; nq < NQ; ++nq)
#pragma unroll
          for (int i = 0; i < 4; ++i) o[md][nq][i] = 0.f;
    };

    for (int c = it.c0; c < it.c1; ++c, ++seq) {
      if (c != it.c0 && c % seg_ch == 0) publish_segment(c / seg_ch - 1);  // segment boundary (group schedule)
      const int st = seq % NST;
      mbar_wait(&full[st], (uint32_t)(seq / NST) & 1u);
      const int kstart = c * CH + warp * KPW;
      if (probe) {  // (finite output: a state of one unit-weight zero row)
#pragma unroll
        for (int nq = 0; nq < NQ; ++nq)
#pragma unroll
          for (int j = 0; j < 2; ++j) m[nq][j] = 0.f, l[nq][j] = 1.f;
      } else if (kstart <= wlast) {  // (warp-uniform)
        const uint32_t kb = sbase + st * STAGE_BYTES, vb = kb + KV_BYTES;
        // S^T = K_w Q^T: 16 keys x 8 columns per n-tile, 8 k-steps of 16 dims (two accumulator chains)
        float s[NQ][4], s2[NQ][4];
#pragma unroll
        for (int nq = 0; nq < NQ; ++nq)
#pragma unroll
          for (int i = 0; i < 4; ++i) s[nq][i] = s2[nq][i] = 0.f;
#pragma unroll
        for (int kk = 0; kk < 8; kk += 2) {
          uint32_t a[4], a2[4];
          ldsm_x4(kb + swz(warp * KPW + (mi & 1) * 8 + ri, kk * 2 + (mi >> 1)), a[0], a[1], a[2], a[3]);
          ldsm_x4(kb + swz(warp * KPW + (mi & 1) * 8 + ri, kk * 2 + 2 + (mi >> 1)), a2[0], a2[1], a2[2], a2[3]);
#pragma unroll
          for (int nq = 0; nq < NQ; ++nq) {
            if (nq == 1 && !two) break;
            mma16816(s[nq], a, qb[nq][kk][0], qb[nq][kk][1]);
            mma16816(s2[nq], a2, qb[nq][kk + 1][0], qb[nq][kk + 1][1]);
          }
        }
        uint32_t pb[NQ][2];
        bool resc = false;  // some column of the warp raised its max
#pragma unroll
        for (int nq = 0; nq < NQ; ++nq) {
          if (nq == 1 && !two) break;
          // mask, new running max per column (exact; masked entries excluded)
          float cm[2] = {-INFINITY, -INFINITY};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int key = kstart + g + 8 * (i >> 1), j = i & 1;
            const bool vis = okq[nq][j] && key <= posq[nq][j];
            const float v = vis ? (s[nq][i] + s2[nq][i]) * scale_log2 : -INFINITY;
            s[nq][i] = v;
            cm[j] = fmaxf(cm[j], v);
          }
          float af[2];
#pragma unroll
          for (int j = 0; j < 2; ++j) {
#pragma unroll
            for (int off = 4; off <= 16; off <<= 1) cm[j] = fmaxf(cm[j], __shfl_xor_sync(0xffffffffu, cm[j], off));
            const float mn = fmaxf(m[nq][j], cm[j]);
            af[j] = (mn == -INFINITY) ? 1.f : exp2f(m[nq][j] - mn);
            m[nq][j] = mn;
          }
          // P^T and its column sums; P^T's 8x8 blocks transposed in registers into the PV B fragments
          float e[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) e[i] = (s[nq][i] == -INFINITY) ? 0.f : exp2f(s[nq][i] - m[nq][i & 1]);
          float ps[2] = {e[0] + e[2], e[1] + e[3]};
          pb[nq][0] = movmatrix_trans(pack_bf16(e[0], e[1]));  // keys 0..7 of the slice
          pb[nq][1] = movmatrix_trans(pack_bf16(e[2], e[3]));  // keys 8..15
#pragma unroll
          for (int j = 0; j < 2; ++j) {
#pragma unroll
            for (int off = 4; off <= 16; off <<= 1) ps[j] += __shfl_xor_sync(0xffffffffu, ps[j], off);
            l[nq][j] = l[nq][j] * af[j] + ps[j];
          }
          // (no column of the warp raised its max: every factor is exactly 1 and the rescale is the identity)
          if (!__all_sync(0xffffffffu, af[0] == 1.f && af[1] == 1.f)) {
            resc = true;
#pragma unroll
            for (int md = 0; md < 8; ++md)
#pragma unroll
              for (int i = 0; i < 4; ++i) o[md][nq][i] *= af[i & 1];
          }
        }
        (void)resc;
        // O^T += V_w^T P^T: m-tiles md (16 dims), one k-step (the slice's 16 keys), n-tiles nq
#pragma unroll
        for (int md = 0; md < 8; ++md) {
          uint32_t a[4];
          ldsm_x4_t(vb + swz(warp * KPW + (mi >> 1) * 8 + ri, md * 2 + (mi & 1)), a[0], a[1], a[2], a[3]);
#pragma unroll
          for (int nq = 0; nq < NQ; ++nq) {
            if (nq == 1 && !two) break;
            mma16816(o[md][nq], a, pb[nq][0], pb[nq][1]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);  // this warp is done with the stage
    }
    const unsigned long long ti1 = g_kt.rec ? kt_now() : 0ull;
    const int group = (it.b * p.Hkv + it.kvh) * ntiles + it.qt;
    // several segments: each one's warp states are in the partial buffer, folded below in segment order
    // (the split schedule's CTA that completes the group, or the group's own CTA)
    const bool multi = it.nseg > 1;
    if (multi) {
      publish_segment(split ? it.seg : it.nseg - 1);
      if (split) {
        named_bar(1, NW * 32);
        if (tid == 0) {
          int prev;
          asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(prev) : "l"(p.seg_cnt + group) : "memory");
          mrg_flag[0] = prev == it.nseg - 1;
          if (prev == it.nseg - 1) p.seg_cnt[group] = 0;  // re-arm for the next launch
        }
        named_bar(1, NW * 32);
        if (!mrg_flag[0]) continue;
      } else {
        __threadfence();
        named_bar(1, NW * 32);
      }
    }
    // ---- the merge, one 8-row half of the tile at a time through the 8-row merge buffer: the warp
    // states (or, for the group's last segment, every warp slot's segment states folded in segment
    // order -- the same operations as the in-register fold), then the fixed-order merge and normalise
#pragma unroll
    for (int hf = 0; hf < NQ; ++hf) {
      if (hf == 1 && !two) break;
      const int rb = hf * 8, nh = min(8, nr - rb);  // rows [rb, rb + nh) of the tile
      if (multi) {
        // step factors per (warp, row) first (one thread each), then every thread (one dimension, one
        // parity of the (warp, row) pairs) folds the O values of 4 pairs, 8 segments' loads in flight
        float* fa_s = mrg;                   // [NW][8][kFoldSeg] factor of the running state, then
        float* fb_s = mrg + NW * 8 * kFoldSeg;  // of segment s; the O fold overwrites mrg[] afterwards
        const int nsg = it.nseg;
        if (tid < NW * nh) {
          const int w = tid / nh, r = tid % nh;
          const size_t s0 = row_slot(rb + r) * p.nchunk_max;
          float m_ = -INFINITY, l_ = 0.f;
          for (int sg = 0; sg < nsg; ++sg) {
            const size_t bs = (s0 + sg) * NW + w;
            const float ms = __ldcg(&p.part_ml[2 * bs]), ls = __ldcg(&p.part_ml[2 * bs + 1]);
            const float M = fmaxf(m_, ms);
            const float fa = (m_ == -INFINITY) ? 0.f : exp2f(m_ - M);
            const float fb = (ms == -INFINITY) ? 0.f : exp2f(ms - M);
            l_ = __fadd_rn(__fmul_rn(l_, fa), __fmul_rn(ls, fb));
            m_ = M;
            fa_s[(w * 8 + r) * kFoldSeg + sg] = fa;
            fb_s[(w * 8 + r) * kFoldSeg + sg] = fb;
          }
          mrg_m[w * 8 + r] = m_;
          mrg_l[w * 8 + r] = l_;
        }
        named_bar(1, NW * 32);
        const int d = tid & (HD - 1), par = tid >> 7;  // dimension, pair parity
        const int npair = NW * nh;                      // (warp, row) pairs q = w nh + r
        float Ofold[NW * 8 / 2];
        for (int i0 = 0; 2 * i0 < npair; i0 += 4) {
          float O[4] = {0.f, 0.f, 0.f, 0.f};
          for (int sg0 = 0; sg0 < nsg; sg0 += 8) {
            float Os[4][8];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int q = min(2 * (i0 + j) + par, npair - 1), w = q / nh, r = q % nh;
              const size_t s0 = row_slot(rb + r) * p.nchunk_max;
#pragma unroll
              for (int sg = 0; sg < 8; ++sg)
                Os[j][sg] = (sg0 + sg < nsg) ? __ldcg(&p.part_o[((s0 + sg0 + sg) * NW + w) * HD + d]) : 0.f;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int q = min(2 * (i0 + j) + par, npair - 1), w = q / nh, r = q % nh;
              const float* fa = fa_s + (w * 8 + r) * kFoldSeg + sg0;
              const float* fb = fb_s + (w * 8 + r) * kFoldSeg + sg0;
#pragma unroll
              for (int sg = 0; sg < 8; ++sg)
                if (sg0 + sg < nsg) O[j] = __fadd_rn(__fmul_rn(O[j], fa[sg]), __fmul_rn(Os[j][sg], fb[sg]));
            }
          }
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (i0 + j < NW * 8 / 2) Ofold[i0 + j] = O[j];
        }
        named_bar(1, NW * 32);  // factors consumed before mrg[] is overwritten
        for (int i = 0; 2 * i + par < npair; ++i) {
          const int q = 2 * i + par, w = q / nh, r = q % nh;
          mrg[(w * 8 + r) * HD + d] = Ofold[i];
        }
      } else {
        // this warp's states of the half's rows (one segment: a fold from the empty state is the identity)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int q = 2 * t4 + j;
          if (q < nh) {  // (rows of the tile past the block's rows are never read)
#pragma unroll
            for (int md = 0; md < 8; ++md) {
              mrg[(warp * 8 + q) * HD + md * 16 + g] = o[md][hf][j];
              mrg[(warp * 8 + q) * HD + md * 16 + g + 8] = o[md][hf][2 + j];
            }
            if (g == 0) {
              mrg_m[warp * 8 + q] = m[hf][j];
              mrg_l[warp * 8 + q] = l[hf][j];
            }
          }
        }
      }
      named_bar(1, NW * 32);
      // warp r merges row r (the 8 compute warps <-> the half's <= 8 rows): lanes 0..NW-1 hold warp slot
      // w's m / l and form f_w = 2^(m_w - M), M = max_w m_w; L = sum_w l_w f_w and every output dimension
      // acc = sum_w O_w f_w are accumulated in the fixed order w = 0, 1, .. (lane l: dims 4l .. 4l + 3)
      if (warp < nh) {
        const int r = warp;
        const float mw = lane < NW ? mrg_m[lane * 8 + r] : -INFINITY;
        float M = mw;
#pragma unroll
        for (int off = 1; off < NW; off <<= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
        const float f = (lane < NW && mw != -INFINITY) ? exp2f(mw - M) : 0.f;
        const float lw = lane < NW ? mrg_l[lane * 8 + r] : 0.f;
        float L = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const float fw = __shfl_sync(0xffffffffu, f, w);
          L += __shfl_sync(0xffffffffu, lw, w) * fw;
          const float4 v = *reinterpret_cast<const float4*>(mrg + (w * 8 + r) * HD + 4 * lane);
          acc[0] += v.x * fw;
          acc[1] += v.y * fw;
          acc[2] += v.z * fw;
          acc[3] += v.w * fw;
        }
        const __nv_bfloat162 lo = __floats2bfloat162_rn(acc[0] / L, acc[1] / L);
        const __nv_bfloat162 hi = __floats2bfloat162_rn(acc[2] / L, acc[3] / L);
        uint2 pk;
        pk.x = *reinterpret_cast<const uint32_t*>(&lo);
        pk.y = *reinterpret_cast<const uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.out) + row_slot(rb + r) * HD + 4 * lane) = pk;
      }
      named_bar(1, NW * 32);
    }
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
    cudaFuncSetAttribute(attn_fd_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    cudaFuncSetAttribute(attn_fd_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    attr = true;
  }
  const int G = p.Hq / p.Hkv;
  // 16-row tiles (two n-tiles) when a sequence's (query, head) rows exceed 8 -- 13B at k = 8, GQA -- so
  // its keys are streamed once per 16 rows; the same per-column arithmetic either way (bit-identical).
  // SF_ATTN_NQ=1 forces 8-row tiles (tests)
  const int env_nq = getenv("SF_ATTN_NQ") ? atoi(getenv("SF_ATTN_NQ")) : 0;  // (read per launch: tests compare)
  const int NQ = (p.q_len * G > 8 && env_nq != 1) ? 2 : 1;
  const int ntiles = (p.q_len * G + 8 * NQ - 1) / (8 * NQ);
  // segment size override (tests exercise the multi-segment fold at short contexts; read per launch)
  const int env_seg = getenv("SF_ATTN_SEG") ? atoi(getenv("SF_ATTN_SEG")) : 0;
  const int seg_keys = (env_seg >= CH && env_seg % CH == 0) ? env_seg : kAttnSeg;
  const int nseg_max = (p.max_key + seg_keys - 1) / seg_keys;
  if (nseg_max > p.nchunk_max || nseg_max > kFoldSeg || !p.seg_cnt) return cudaErrorInvalidValue;
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
  launch_k(NQ == 2 ? attn_fd_kernel<2> : attn_fd_kernel<1>, dim3(grid), dim3(NTHR), SMEM, s, mk, mv, mk4, mv4, p, ntiles, nseg_max, seg_keys, n_items,
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
