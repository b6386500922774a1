// attn_mma.cu -- bf16 hybrid-mask paged decode attention (mode CAUSAL_PREFIX), tensor-core version.
//
// Same split-KV semantics as the SIMT kernel in kernels.cu (fixed absolute 128-key chunks, one
// unnormalised partial (m, l, acc) per (row, head, chunk), merged in chunk order by
// attn_combine_kernel), so every row's result is independent of batch size, block length and
// split count (batch invariance, reading C23).
//
// Persistent CTAs walk a static list of (sequence, kv head, query tile, chunk range) items. A
// producer warp streams each 128-key K/V chunk (64 KB) with TMA: one 2-D box per (16-key page,
// 64-dim half) of the paged cache, 128-byte swizzled (conflict-free ldmatrix), into a 3-stage
// mbarrier ring, while 4 compute warps work on the previous chunk:
//   S = Q K^T   : warp w owns keys 32w..32w+31, mma.sync m16n8k16 bf16 -> fp32
//   chunk softmax: row max / sum across the 4 warps in fixed order (exact zeros for masked keys)
//   O = P V     : P (bf16) exchanged through smem, warp w owns output dims 32w..32w+31
#include <cudaTypedefs.h>

#include <algorithm>
#include <cfloat>
#include <cmath>

#include "common.cuh"
#include "kernels.cuh"

namespace sf {

namespace {

constexpr int HD = 128;
constexpr int CH = kAttnChunk;   // 128 keys
constexpr int NST = 3;           // pipeline stages
constexpr int KV_BYTES = CH * HD * 2;            // one of K or V per stage: 32 KB
constexpr int STAGE_BYTES = 2 * KV_BYTES;        // 64 KB
constexpr int PLD = CH + 8;                      // padded P row (bf16 elements)
constexpr int SMEM = NST * STAGE_BYTES + 16 * PLD * 2 + 2 * 4 * 16 * 4 + 2 * NST * 8 + 1024 + 64;

SF_DEV void cp_async16_zfill(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
SF_DEV void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
SF_DEV void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
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
// byte offset of 16-byte chunk c (0..15) of key row j in a [2 halves][128 keys][128 B] tile, each
// 128-byte row 128B-swizzled exactly as TMA SWIZZLE_128B writes it (chunk c' at c' ^ (j % 8))
SF_DEV uint32_t swz(int j, int c) {
  return (uint32_t)((c >> 3) * (CH * 128) + j * 128 + (((c & 7) ^ (j & 7)) << 4));
}
SF_DEV void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

struct Item {
  int b, kvh, qt, c0, c1;
};

}  // namespace

// Work list is implicit: item = ((b * Hkv + kvh) * ntiles + qt) * nsplit + split.
// Warps 0..3 compute, warp 4 produces (TMA).
__global__ void __launch_bounds__(160, 1) attn_mma_kernel(const __grid_constant__ CUtensorMap tmK,
                                                         const __grid_constant__ CUtensorMap tmV, AttnParams p,
                                                         int ntiles, int nsplit, int n_items) {
  KtScope kt_(KT_ATTN, (uint32_t)(1));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  const uint32_t raw = smem_u32(sm_raw);
  uint8_t* sm = sm_raw + (((raw + 1023u) & ~1023u) - raw);
  const uint32_t sbase = smem_u32(sm);
  __nv_bfloat16* Ps = reinterpret_cast<__nv_bfloat16*>(sm + NST * STAGE_BYTES);
  float* red_m = reinterpret_cast<float*>(sm + NST * STAGE_BYTES + 16 * PLD * 2);
  float* red_l = red_m + 4 * 16;
  uint64_t* full = reinterpret_cast<uint64_t*>(red_l + 4 * 16);
  uint64_t* empty = full + NST;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int G = p.Hq / p.Hkv;
  const int R = p.q_len * G;

  auto item_of = [&](int idx, Item& it) -> bool {
    int r = idx;
    const int split = r % nsplit;
    r /= nsplit;
    it.qt = r % ntiles;
    r /= ntiles;
    it.kvh = r % p.Hkv;
    it.b = r / p.Hkv;
    const int r0 = it.qt * 16;
    const int nr = min(16, R - r0);
    const int kmax = min(p.pos0[it.b] + min(p.q_len - 1, (r0 + nr - 1) / G), p.max_key - 1);
    const int nch = kmax / CH + 1;
    const int per = (nch + nsplit - 1) / nsplit;
    it.c0 = split * per;
    it.c1 = min(nch, it.c0 + per);
    return it.c0 < it.c1;
  };

  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);  // one arrival per compute warp
    }
    fence_barrier_init();
  }
  // Pages past a sequence's last key are not loaded: their (masked, p = 0) V rows must still be
  // finite, so the ring starts zeroed; afterwards it only ever holds real (finite) K/V values.
  for (int i = tid; i < NST * STAGE_BYTES / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0u, 0u, 0u, 0u);
  fence_proxy_async();
  __syncthreads();

  if (warp == 4) {
    // ---- TMA producer
    int seq = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      Item it;
      if (!item_of(item, it)) continue;
      const int r0 = it.qt * 16;
      const int nr = min(16, R - r0);
      const int kmax = min(p.pos0[it.b] + min(p.q_len - 1, (r0 + nr - 1) / G), p.max_key - 1);
      for (int c = it.c0; c < it.c1; ++c, ++seq) {
        const int st = seq % NST;
        mbar_wait(&empty[st], ((uint32_t)(seq / NST) & 1u) ^ 1u);
        const int kstart = c * CH;
        const int npages = (min(CH, kmax + 1 - kstart) + 15) / 16;
        const int pg = (lane < npages) ? p.block_table[it.b * p.pages_per_seq + kstart / 16 + lane] : 0;
        if (lane == 0) mbar_arrive_expect_tx(&full[st], (uint32_t)(npages * 4 * 16 * 128));
        __syncwarp();
        // page ids broadcast warp-wide, then the elected lane issues the boxes
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

  int cur_item = blockIdx.x;
  Item cur{};
  while (cur_item < n_items && !item_of(cur_item, cur)) cur_item += gridDim.x;
  int use_seq = 0;
  uint32_t qa[8][4];  // Q A-fragments (bf16) for 8 k-steps of 16 dims
  int q_item = -1;
  while (cur_item < n_items) {
    const int r0 = cur.qt * 16;
    const int nr = min(16, R - r0);
    const int base = p.pos0[cur.b];
    if (q_item != cur_item) {
      // load Q rows g and g+8 of this tile (fp32 rotated queries -> bf16 fragments)
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const int r = g + 8 * hr;
        const bool ok = r < nr;
        const int rr = r0 + r, qi = rr / G, h = cur.kvh * G + rr % G;
        const float* qrow = p.q + ((size_t)(cur.b * p.q_len + qi) * p.Hq + h) * HD;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const int d0 = kk * 16 + 2 * t4;
          float2 x0 = ok ? *reinterpret_cast<const float2*>(qrow + d0) : make_float2(0.f, 0.f);
          float2 x1 = ok ? *reinterpret_cast<const float2*>(qrow + d0 + 8) : make_float2(0.f, 0.f);
          qa[kk][hr] = pack_bf16(x0.x, x0.y);
          qa[kk][2 + hr] = pack_bf16(x1.x, x1.y);
        }
      }
      q_item = cur_item;
    }
    for (int c = cur.c0; c < cur.c1; ++c) {
      const int stage = use_seq % NST;
      mbar_wait(&full[stage], (uint32_t)(use_seq / NST) & 1u);  // this chunk's K/V landed
      const uint32_t kb = sbase + stage * STAGE_BYTES, vb = kb + KV_BYTES;
      const int kstart = c * CH;
      // ---- S = Q K^T over this warp's 32 keys
      float s[4][4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) s[nt][i] = 0.f;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int key = warp * 32 + nt * 8 + (lane & 7);
#pragma unroll
        for (int kp = 0; kp < 4; ++kp) {  // pairs of k-steps (32 dims)
          uint32_t b0, b1, b2, b3;
          ldsm_x4(kb + swz(key, kp * 4 + (lane >> 3)), b0, b1, b2, b3);
          mma16816(s[nt], qa[2 * kp], b0, b1);
          mma16816(s[nt], qa[2 * kp + 1], b2, b3);
        }
      }
      // ---- mask + chunk max (rows g, g+8)
      const float scale = 0.08838834764831845f;  // 1/sqrt(128)
      const int pos_lo = base + (r0 + g) / G, pos_hi = base + (r0 + g + 8) / G;
      const bool row_lo = g < nr, row_hi = g + 8 < nr;
      float mlo = -INFINITY, mhi = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int key = kstart + warp * 32 + nt * 8 + 2 * t4 + (i & 1);
          const bool hi = i >= 2;
          const bool vis = hi ? (row_hi && key <= pos_hi) : (row_lo && key <= pos_lo);
          const float v = vis ? s[nt][i] * scale : -INFINITY;
          s[nt][i] = v;
          if (hi) mhi = fmaxf(mhi, v); else mlo = fmaxf(mlo, v);
        }
      }
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        mlo = fmaxf(mlo, __shfl_xor_sync(0xffffffffu, mlo, o));
        mhi = fmaxf(mhi, __shfl_xor_sync(0xffffffffu, mhi, o));
      }
      if (t4 == 0) {
        red_m[warp * 16 + g] = mlo;
        red_m[warp * 16 + g + 8] = mhi;
      }
      named_bar(1, 128);
      const float Mlo = fmaxf(fmaxf(red_m[g], red_m[16 + g]), fmaxf(red_m[32 + g], red_m[48 + g]));
      const float Mhi =
          fmaxf(fmaxf(red_m[8 + g], red_m[24 + g]), fmaxf(red_m[40 + g], red_m[56 + g]));
      float llo = 0.f, lhi = 0.f;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        float e[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float M = i >= 2 ? Mhi : Mlo;
          e[i] = (s[nt][i] == -INFINITY) ? 0.f : expf(s[nt][i] - M);
        }
        llo += e[0] + e[1];
        lhi += e[2] + e[3];
        const int col = warp * 32 + nt * 8 + 2 * t4;
        *reinterpret_cast<uint32_t*>(Ps + g * PLD + col) = pack_bf16(e[0], e[1]);
        *reinterpret_cast<uint32_t*>(Ps + (g + 8) * PLD + col) = pack_bf16(e[2], e[3]);
      }
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        llo += __shfl_xor_sync(0xffffffffu, llo, o);
        lhi += __shfl_xor_sync(0xffffffffu, lhi, o);
      }
      if (t4 == 0) {
        red_l[warp * 16 + g] = llo;
        red_l[warp * 16 + g + 8] = lhi;
      }
      named_bar(1, 128);
      // ---- O = P V for this warp's 32 output dims (n-tiles 4w..4w+3)
      float o[4][4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) o[nt][i] = 0.f;
      const uint32_t pbase = smem_u32(Ps);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        uint32_t a[4];
        {
          const int mi = lane >> 3, ri = lane & 7;
          const int row = (mi & 1) * 8 + ri, col = kk * 16 + (mi >> 1) * 8;
          ldsm_x4(pbase + (row * PLD + col) * 2, a[0], a[1], a[2], a[3]);
        }
#pragma unroll
        for (int np = 0; np < 2; ++np) {
          const int mi = lane >> 3, ri = lane & 7;
          const int key = kk * 16 + (mi & 1) * 8 + ri;
          const int chunk = warp * 4 + np * 2 + (mi >> 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(vb + swz(key, chunk), b0, b1, b2, b3);
          mma16816(o[2 * np], a, b0, b1);
          mma16816(o[2 * np + 1], a, b2, b3);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);  // this warp is done reading the stage
      // ---- write the chunk partial
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const int r = g + 8 * hr;
        if (r < nr) {
          const int rr = r0 + r, qi = rr / G, h = cur.kvh * G + rr % G;
          const int t = cur.b * p.q_len + qi;
          const size_t ob = ((size_t)t * p.Hq + h) * p.nchunk_max + c;
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) {
            const int d = warp * 32 + nt * 8 + 2 * t4;
            *reinterpret_cast<float2*>(p.part_o + ob * HD + d) = make_float2(o[nt][2 * hr], o[nt][2 * hr + 1]);
          }
          if (warp == 0 && t4 == 0) {
            const float M = hr ? Mhi : Mlo;
            const float L = ((red_l[r] + red_l[16 + r]) + red_l[32 + r]) + red_l[48 + r];
            p.part_ml[2 * ob] = M;
            p.part_ml[2 * ob + 1] = L;
          }
        }
      }
      ++use_seq;
      named_bar(1, 128);  // Ps + red buffers free for reuse
    }
    do {
      cur_item += gridDim.x;
    } while (cur_item < n_items && !item_of(cur_item, cur));
  }
}

static int g_num_sms = 0;

// 2-D view of one layer's paged K (or V) pool: [n_pages * Hkv * 16 rows, 128 dims] bf16; a box is
// one 16-key page x 64 dims (128 B rows), 128B-swizzled.
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

cudaError_t launch_attention_mma(const AttnParams& p, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    attr = true;
  }
  const int G = p.Hq / p.Hkv;
  const int ntiles = (p.q_len * G + 15) / 16;
  const int nch = (p.max_key + CH - 1) / CH;
  const int pairs = p.B * p.Hkv * ntiles;
  // split the key range only when there are too few (sequence, head) pairs to fill the GPU
  int nsplit = 1;
  while (nsplit < nch && pairs * nsplit < 2 * g_num_sms) ++nsplit;
  const int n_items = pairs * nsplit;
  const int grid = std::min(n_items, g_num_sms);
  CUtensorMap mk, mv;
  const long long rows = (long long)p.n_pages * p.Hkv * 16;
  if (!encode_kv_map(&mk, p.Kp, rows) || !encode_kv_map(&mv, p.Vp, rows)) return cudaErrorInvalidValue;
  launch_k(attn_mma_kernel, dim3(grid), dim3(160), SMEM, s, mk, mv, p, ntiles, nsplit, n_items);
  return cudaGetLastError();
}

cudaError_t kt_setup_attn_mma(void* rec, unsigned* cnt, unsigned cap) {
  KtBuf b;
  b.rec = reinterpret_cast<KtRec*>(rec);
  b.cnt = cnt;
  b.cap = cap;
  return kt_setup_tu(b);
}

}  // namespace sf
