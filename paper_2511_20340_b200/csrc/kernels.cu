// kernels.cu -- element-wise, normalisation, RoPE/paged-KV append, hybrid-mask attention and
// accept kernels of the SpecFormer decode step. Every reduction uses a fixed order that depends
// only on the row's own data and position (batch invariance, reading C23), so GPU SD == GPU AR
// bit for bit.
#include <algorithm>
#include <cfloat>
#include <cmath>

#include "common.cuh"
#include "kernels.cuh"

namespace sf {

// ------------------------------------------------------------------------ RoPE table
// cos/sin(pos * theta^(-2i/hd)) evaluated in double, stored fp32 (reading C5).
__global__ void rope_table_kernel(float2* tab, int max_seq, int hd, float theta) {
  KtScope kt_(KT_MISC, (uint32_t)(4));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  const int half = hd / 2;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= max_seq * half) return;
  const int pos = idx / half, i = idx % half;
  const double inv = pow((double)theta, -2.0 * i / hd);
  double s, c;
  sincos((double)pos * inv, &s, &c);
  tab[idx] = make_float2((float)c, (float)s);
}

// ------------------------------------------------------------------------ row builders
__global__ void build_verify_rows_kernel(int B, int k, const int* last_token, const int* draft, int* tok) {
  KtScope kt_(KT_ROWS, (uint32_t)(0));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= B * (k + 1)) return;
  const int b = r / (k + 1), i = r % (k + 1);
  tok[r] = (i == 0) ? last_token[b] : draft[b * k + i - 1];
}
__global__ void build_prefill_rows_kernel(int B, int P, int c0, int C, const int* tokens, int* tok, int* pos0) {
  KtScope kt_(KT_ROWS, (uint32_t)(1));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < B) pos0[r] = c0;
  if (r >= B * C) return;
  const int b = r / C, i = r % C;
  tok[r] = tokens[(size_t)b * P + c0 + i];
}

// ------------------------------------------------------------------------ embedding (HS[0])
template <typename TW>
__global__ void embed_kernel(const int* tok, const TW* emb, int d, int vocab, float* resid, float* tap0) {
  KtScope kt_(KT_EMBED, (uint32_t)(d));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  const int t = blockIdx.x;
  int id = tok[t];
  id = min(max(id, 0), vocab - 1);
  const TW* src = emb + (size_t)id * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const float v = Elt<TW>::to_f(src[i]);
    resid[(size_t)t * d + i] = v;
    if (tap0) tap0[(size_t)t * d + i] = v;
  }
}

// ------------------------------------------------------------------------ RMSNorm
// y = x / sqrt(mean(x^2) + eps) * g, fp32 statistics, one CTA (256 threads) per row.
template <typename TO>
__global__ void __launch_bounds__(256) rmsnorm_kernel(const float* in, int in_ld, const float* g, float eps, int d,
                                                      TO* out, int out_ld) {
  KtScope kt_(KT_RMSNORM, (uint32_t)(d));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  __shared__ float red[8];
  const int t = blockIdx.x;
  const float* x = in + (size_t)t * in_ld;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += 256) ss = fmaf(x[i], x[i], ss);
  ss = block_sum<256>(ss, red);
  const float r = 1.0f / sqrtf(ss / (float)d + eps);
  TO* y = out + (size_t)t * out_ld;
  for (int i = threadIdx.x; i < d; i += 256) y[i] = Elt<TO>::from_f(x[i] * r * g[i]);
}

// Grouped RMS Norm + concat (Eq.8 I_Cat; the paper's Triton kernel KP1, P330-332):
// out[t, g*d + i] = taps[g][t][i] / rms_g * s[g][i]
template <typename TO>
__global__ void __launch_bounds__(256) group_rms_kernel(const float* taps, int64_t tap_stride, const float* sc,
                                                        float eps, int d, TO* out) {
  KtScope kt_(KT_GROUP_RMS, (uint32_t)(d));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  __shared__ float red[8];
  const int t = blockIdx.x;
  for (int g = 0; g < 4; ++g) {
    const float* x = taps + g * tap_stride + (size_t)t * d;
    float ss = 0.f;
    for (int i = threadIdx.x; i < d; i += 256) ss = fmaf(x[i], x[i], ss);
    ss = block_sum<256>(ss, red);
    const float r = 1.0f / sqrtf(ss / (float)d + eps);
    TO* y = out + (size_t)t * 4 * d + (size_t)g * d;
    for (int i = threadIdx.x; i < d; i += 256) y[i] = Elt<TO>::from_f(x[i] * r * sc[g * d + i]);
  }
}

// ------------------------------------------------------------------------ vectorised row kernels
// bf16 path, d % 128 == 0: one CTA of d / (4 NG) threads per row, thread t owns the float4 groups
// 4t + 4 nthr j (j < NG): every load / store is 16 bytes and even a 5-row step spreads over
// thousands of threads.
static int row_ng(int d) {
  for (int ng = 1; ng <= 4; ++ng)
    if (d % (128 * ng) == 0 && d / (4 * ng) <= 1024) return ng;
  return 0;
}
SF_DEV void st_bf16x4(__nv_bfloat16* p, float a, float b, float c, float d) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, d);
  uint2 pk;
  pk.x = *reinterpret_cast<uint32_t*>(&lo);
  pk.y = *reinterpret_cast<uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(p) = pk;
}
// y = x / sqrt(mean(x^2) + eps) * g  (grid.y > 1: grouped form, group g = blockIdx.y reads taps
// + g * x_stride, scales g_ + g * d, writes columns [g d, (g+1) d) of a [T, 4d] row -- Eq.8 I_Cat)
template <int NG>
__global__ void __launch_bounds__(1024) rms_rows_kernel(const float* x_, int64_t x_stride, int in_ld, const float* g_,
                                                        float eps, int d, __nv_bfloat16* out, int out_ld) {
  KtScope kt_(gridDim.y > 1 ? KT_GROUP_RMS : KT_RMSNORM, (uint32_t)(d));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  __shared__ float red[32];
  const int t = blockIdx.x, grp = blockIdx.y, nthr = blockDim.x;
  const float* x = x_ + grp * x_stride + (size_t)t * in_ld;
  const float* gm = g_ + (size_t)grp * d;
  float4 v[NG];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < NG; ++j) {
    v[j] = *reinterpret_cast<const float4*>(x + 4 * threadIdx.x + 4 * nthr * j);
    ss = fmaf(v[j].x, v[j].x, ss);
    ss = fmaf(v[j].y, v[j].y, ss);
    ss = fmaf(v[j].z, v[j].z, ss);
    ss = fmaf(v[j].w, v[j].w, ss);
  }
  ss = block_sum_dyn(ss, red);
  const float r = 1.0f / sqrtf(ss / (float)d + eps);
  __nv_bfloat16* y = out + (size_t)t * out_ld + (size_t)grp * d;
#pragma unroll
  for (int j = 0; j < NG; ++j) {
    const int i = 4 * threadIdx.x + 4 * nthr * j;
    const float4 gg = *reinterpret_cast<const float4*>(gm + i);
    st_bf16x4(y + i, v[j].x * r * gg.x, v[j].y * r * gg.y, v[j].z * r * gg.z, v[j].w * r * gg.w);
  }
}
// embedding rows (bf16 table) -> fp32 residual stream (+ tap HS[0]), 8 elements per thread
__global__ void __launch_bounds__(1024) embed_v_kernel(const int* tok, const __nv_bfloat16* emb, int d, int vocab,
                                                       float* resid, float* tap0) {
  KtScope kt_(KT_EMBED, (uint32_t)(d));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  const int t = blockIdx.x;
  const int id = min(max(tok[t], 0), vocab - 1);
  for (int i = 8 * threadIdx.x; i < d; i += 8 * blockDim.x) {
    const uint4 raw = *reinterpret_cast<const uint4*>(emb + (size_t)id * d + i);
    const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
    const float2 a = __bfloat1622float2(h2[0]), b = __bfloat1622float2(h2[1]), c = __bfloat1622float2(h2[2]),
                 e = __bfloat1622float2(h2[3]);
    const float4 lo = make_float4(a.x, a.y, b.x, b.y), hi = make_float4(c.x, c.y, e.x, e.y);
    *reinterpret_cast<float4*>(resid + (size_t)t * d + i) = lo;
    *reinterpret_cast<float4*>(resid + (size_t)t * d + i + 4) = hi;
    if (tap0) {
      *reinterpret_cast<float4*>(tap0 + (size_t)t * d + i) = lo;
      *reinterpret_cast<float4*>(tap0 + (size_t)t * d + i + 4) = hi;
    }
  }
}

// ------------------------------------------------------------------------ RoPE + paged KV append
// qkv row = [q (Hq*hd) | k (Hkv*hd) | v (Hkv*hd)]. Queries rotated -> q_out fp32;
// keys rotated and values copied into the sequence's pages at their absolute positions.
// One warp per (row, head slot) -- grid (T, ceil((Hq + 2 Hkv) / 4)), 4 warps per CTA -- so even a
// 5-row verify block spreads over hundreds of warps; lane l owns the rotate-half pairs
// (i, i + hd/2) for i = VEC l .. VEC l + VEC - 1 (+ 32 VEC j), VEC = 2 when hd/2 is a multiple of 64.
template <typename TA, int VEC, bool QB>
__global__ void __launch_bounds__(256) rope_append_kernel(const TA* qkv, int q_len, const int* pos0,
                                                          const float2* rope, int Hq, int Hkv, int hd,
                                                          const int* bt, int pps, TA* Kp, TA* Vp, void* q_out,
                                                          int hpw) {
  KtScope kt_(KT_ROPE, (uint32_t)(Hq));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  const int t = blockIdx.x;
  const int lane = threadIdx.x & 31;
  for (int hh = 0; hh < hpw; ++hh) {
  const int h = (blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5)) * hpw + hh;
  if (h >= Hq + 2 * Hkv) return;
  const int b = t / q_len, qi = t % q_len;
  const int pos = pos0[b] + qi;
  const int half = hd / 2;
  const int W = (Hq + 2 * Hkv) * hd;
  const TA* row = qkv + (size_t)t * W + (size_t)h * hd;
  const int blk = bt[b * pps + pos / 16], slot = pos % 16;
  if (h >= Hq + Hkv) {  // value head: plain copy into the page
    TA* dst = Vp + (((size_t)blk * Hkv + (h - Hq - Hkv)) * 16 + slot) * hd;
    for (int i = lane * VEC; i < hd; i += 32 * VEC) {
      if constexpr (VEC == 2 && sizeof(TA) == 2) {
        *reinterpret_cast<__nv_bfloat162*>(dst + i) = *reinterpret_cast<const __nv_bfloat162*>(row + i);
      } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) dst[i + v] = row[i + v];
      }
    }
    continue;
  }
  const float2* cs = rope + (size_t)pos * half;
  for (int i = lane * VEC; i < half; i += 32 * VEC) {
    float x1[VEC], x2[VEC], y1[VEC], y2[VEC];
    float2 c[VEC];
    if constexpr (VEC == 2 && sizeof(TA) == 2) {
      const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(row + i));
      const float2 bb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(row + i + half));
      const float4 cc = *reinterpret_cast<const float4*>(cs + i);
      x1[0] = a.x, x1[1] = a.y, x2[0] = bb.x, x2[1] = bb.y;
      c[0] = make_float2(cc.x, cc.y), c[1] = make_float2(cc.z, cc.w);
    } else {
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        c[v] = cs[i + v];
        x1[v] = Elt<TA>::to_f(row[i + v]);
        x2[v] = Elt<TA>::to_f(row[i + v + half]);
      }
    }
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      y1[v] = rope_y1(x1[v], x2[v], c[v].x, c[v].y);
      y2[v] = rope_y2(x1[v], x2[v], c[v].x, c[v].y);
    }
    if (h < Hq) {
      if constexpr (QB) {  // bf16 queries (RNE: the same bits the attention kernel would round to)
        __nv_bfloat16* qb = reinterpret_cast<__nv_bfloat16*>(q_out) + ((size_t)t * Hq + h) * hd;
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          qb[i + v] = __float2bfloat16_rn(y1[v]);
          qb[i + v + half] = __float2bfloat16_rn(y2[v]);
        }
        continue;
      }
      float* q = reinterpret_cast<float*>(q_out) + ((size_t)t * Hq + h) * hd;
      if constexpr (VEC == 2) {
        *reinterpret_cast<float2*>(q + i) = make_float2(y1[0], y1[1]);
        *reinterpret_cast<float2*>(q + i + half) = make_float2(y2[0], y2[1]);
      } else {
        q[i] = y1[0];
        q[i + half] = y2[0];
      }
    } else {
      TA* dst = Kp + (((size_t)blk * Hkv + (h - Hq)) * 16 + slot) * hd;
      if constexpr (VEC == 2 && sizeof(TA) == 2) {
        *reinterpret_cast<__nv_bfloat162*>(dst + i) = __floats2bfloat162_rn(y1[0], y1[1]);
        *reinterpret_cast<__nv_bfloat162*>(dst + i + half) = __floats2bfloat162_rn(y2[0], y2[1]);
      } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          dst[i + v] = Elt<TA>::from_f(y1[v]);
          dst[i + v + half] = Elt<TA>::from_f(y2[v]);
        }
      }
    }
  }
  }  // heads of this warp
}

// bf16, hd = 128, bf16 queries (the flash-decoding path; the QKV weight rows are pair-interleaved
// per head, so its output is too): persistent warps walk the (row, head) items two at a time
// (loads of both in flight), lane l owns the rotate-half pairs (2l, 2l+64) and (2l+1, 2l+65).
// A few hundred resident CTAs instead of T x heads / 8 short ones.
__global__ void __launch_bounds__(256) rope_append128_kernel(const __nv_bfloat16* qkv, int T, int q_len,
                                                             const int* pos0, const float2* rope, int Hq, int Hkv,
                                                             const int* bt, int pps, __nv_bfloat16* Kp,
                                                             __nv_bfloat16* Vp, __nv_bfloat16* q_out) {
  KtScope kt_(KT_ROPE, (uint32_t)(Hq));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  const int H = Hq + 2 * Hkv, W = H * 128;
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
      // pair-interleaved head rows (include/specformer.h): position 2d holds dim d, 2d+1 dim d + 64;
      // lane l reads positions 4l..4l+3 = dims (2l, 2l+64, 2l+1, 2l+65)
      const __nv_bfloat16* row = qkv + (size_t)t[u] * W + (size_t)h[u] * 128;
      const uint2 raw = *reinterpret_cast<const uint2*>(row + 4 * lane);
      const __nv_bfloat162 p0 = *reinterpret_cast<const __nv_bfloat162*>(&raw.x);  // (2l, 2l+64)
      const __nv_bfloat162 p1 = *reinterpret_cast<const __nv_bfloat162*>(&raw.y);  // (2l+1, 2l+65)
      const __nv_bfloat162 lo = __halves2bfloat162(__low2bfloat16(p0), __low2bfloat16(p1));
      const __nv_bfloat162 hi = __halves2bfloat162(__high2bfloat16(p0), __high2bfloat16(p1));
      a[u] = *reinterpret_cast<const uint32_t*>(&lo);   // dims 2l, 2l+1
      bb[u] = *reinterpret_cast<const uint32_t*>(&hi);  // dims 2l+64, 2l+65
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

// ------------------------------------------------------------------------ paged attention
// Hybrid-mask decode attention, mode CAUSAL_PREFIX: query row i of sequence b (absolute position
// p = pos0[b] + i) attends keys 0..p of its pages. Split-KV over FIXED absolute 128-key chunks:
// CTA (chunk c, kv head, query tile, b) writes an unnormalised partial (m, l, acc); the combine
// kernel merges chunks in order c = 0, 1, ... . Shared-memory staged K/V via 16-byte cp.async.
constexpr int QT = 16;  // query rows per CTA

SF_DEV void cp_async16(void* smem, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(g) : "memory");
}
SF_DEV void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

template <typename TKV, int HD>
__global__ void __launch_bounds__(128) attn_partial_kernel(AttnParams p) {
  KtScope kt_(KT_ATTN_PART, (uint32_t)(HD));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  constexpr int VEC = 16 / sizeof(TKV);     // elements per 16-byte vector
  constexpr int KLD = HD + VEC;             // padded K row (bank-conflict-free per-key reads)
  extern __shared__ __align__(16) uint8_t sm[];
  TKV* Ks = reinterpret_cast<TKV*>(sm);
  TKV* Vs = Ks + kAttnChunk * KLD;
  float* Qs = reinterpret_cast<float*>(Vs + kAttnChunk * HD);
  float* S = Qs + QT * HD;

  const int c = blockIdx.x, b = blockIdx.z;
  const int G = p.Hq / p.Hkv;
  const int ntiles = (p.q_len * G + QT - 1) / QT;
  const int kvh = blockIdx.y / ntiles, qt = blockIdx.y % ntiles;
  const int R = p.q_len * G;
  const int r0 = qt * QT;
  const int nr = min(QT, R - r0);
  const int base = p.pos0[b];
  const int kstart = c * kAttnChunk;
  const int kmax = base + attn_row_last(p, min(p.q_len - 1, (r0 + nr - 1) / G));  // largest visible key of the tile
  if (kstart > kmax) return;
  const int nk = min(kAttnChunk, kmax + 1 - kstart);
  const int tid = threadIdx.x;

  // stage K, V chunk
  const TKV* Kg = reinterpret_cast<const TKV*>(p.Kp);
  const TKV* Vg = reinterpret_cast<const TKV*>(p.Vp);
  for (int e = tid; e < nk * (HD / VEC); e += 128) {
    const int j = e / (HD / VEC), part = e % (HD / VEC);
    const int key = kstart + j;
    const int blk = p.block_table[b * p.pages_per_seq + key / 16];
    const size_t off = (((size_t)blk * p.Hkv + kvh) * 16 + (key % 16)) * HD + part * VEC;
    cp_async16(Ks + j * KLD + part * VEC, Kg + off);
    cp_async16(Vs + j * HD + part * VEC, Vg + off);
  }
  // queries
  for (int e = tid; e < nr * HD; e += 128) {
    const int r = e / HD, dd = e % HD;
    const int rr = r0 + r, qi = rr / G, h = kvh * G + rr % G;
    const int t = b * p.q_len + qi;
    Qs[r * HD + dd] = p.q[((size_t)t * p.Hq + h) * HD + dd];
  }
  cp_async_wait_all();
  __syncthreads();

  const float scale = rsqrtf((float)HD);
  // ---- scores: thread <-> key
  {
    const int j = tid;
    float acc[QT];
#pragma unroll
    for (int r = 0; r < QT; ++r) acc[r] = 0.f;
    if (j < nk) {
#pragma unroll 4
      for (int d0 = 0; d0 < HD; d0 += VEC) {
        float kv[VEC];
        if constexpr (sizeof(TKV) == 2) {
          const uint4 raw = *reinterpret_cast<const uint4*>(Ks + j * KLD + d0);
          const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float2 f = __bfloat1622float2(h2[u]);
            kv[2 * u] = f.x;
            kv[2 * u + 1] = f.y;
          }
        } else {
          const float4 raw = *reinterpret_cast<const float4*>(Ks + j * KLD + d0);
          kv[0] = raw.x; kv[1] = raw.y; kv[2] = raw.z; kv[3] = raw.w;
        }
#pragma unroll
        for (int r = 0; r < QT; ++r) {
          if (r < nr) {
#pragma unroll
            for (int u = 0; u < VEC; ++u) acc[r] = fmaf(Qs[r * HD + d0 + u], kv[u], acc[r]);
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < QT; ++r) {
      if (r < nr) {
        const int pos = base + attn_row_last(p, (r0 + r) / G);
        const bool vis = (j < nk) && (kstart + j <= pos);
        S[r * kAttnChunk + j] = vis ? acc[r] * scale : -INFINITY;
      }
    }
  }
  __syncthreads();
  // ---- chunk softmax (unnormalised): warp per row
  const int warp = tid >> 5, lane = tid & 31;
  float* ML = S + QT * kAttnChunk;
  for (int r = warp; r < nr; r += 4) {
    float v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = S[r * kAttnChunk + lane + 32 * i];
    float mx = fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3]));
    mx = warp_max(mx);
    float l = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float e = (mx == -INFINITY || v[i] == -INFINITY) ? 0.f : expf(v[i] - mx);
      S[r * kAttnChunk + lane + 32 * i] = e;
      l += e;
    }
    l = warp_sum(l);
    if (lane == 0) {
      ML[2 * r] = mx;
      ML[2 * r + 1] = l;
    }
  }
  __syncthreads();
  // ---- P V: thread <-> (dim, row group)
  {
    constexpr int RG = 128 / HD;
    const int dd = tid % HD, rg = tid / HD;
    float acc[QT / RG > 0 ? QT / RG : 1];
#pragma unroll
    for (int i = 0; i < QT / RG; ++i) acc[i] = 0.f;
    for (int j = 0; j < nk; ++j) {
      const float v = Elt<TKV>::to_f(Vs[j * HD + dd]);
#pragma unroll
      for (int i = 0; i < QT / RG; ++i) {
        const int r = rg + i * RG;
        if (r < nr) acc[i] = fmaf(S[r * kAttnChunk + j], v, acc[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < QT / RG; ++i) {
      const int r = rg + i * RG;
      if (r < nr) {
        const int rr = r0 + r, qi = rr / G, h = kvh * G + rr % G;
        const int t = b * p.q_len + qi;
        const size_t o = ((size_t)t * p.Hq + h) * p.nchunk_max + c;
        p.part_o[o * HD + dd] = acc[i];
        if (dd == 0) {
          p.part_ml[2 * o] = ML[2 * r];
          p.part_ml[2 * o + 1] = ML[2 * r + 1];
        }
      }
    }
  }
}

// combine chunks 0..pos/128 in order: M = max m_c; out = sum_c acc_c e^(m_c - M) / sum_c l_c e^(m_c - M)
template <typename TA>
__global__ void attn_combine_kernel(AttnParams p) {
  KtScope kt_(KT_ATTN_COMB, (uint32_t)(0));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  const int t = blockIdx.x, h = blockIdx.y;
  const int b = t / p.q_len, qi = t % p.q_len;
  const int pos = p.pos0[b] + attn_row_last(p, qi);
  const int nc = pos / kAttnChunk + 1;
  const size_t o0 = ((size_t)t * p.Hq + h) * p.nchunk_max;
  float M = -INFINITY;
  for (int c = 0; c < nc; ++c) M = fmaxf(M, p.part_ml[2 * (o0 + c)]);
  float L = 0.f;
  for (int c = 0; c < nc; ++c) L += p.part_ml[2 * (o0 + c) + 1] * expf(p.part_ml[2 * (o0 + c)] - M);
  for (int dd = threadIdx.x; dd < p.hd; dd += blockDim.x) {
    float acc = 0.f;
    for (int c = 0; c < nc; ++c) acc += p.part_o[(o0 + c) * p.hd + dd] * expf(p.part_ml[2 * (o0 + c)] - M);
    reinterpret_cast<TA*>(p.out)[((size_t)t * p.Hq + h) * p.hd + dd] = Elt<TA>::from_f(acc / L);
  }
}

// ------------------------------------------------------------------------ draft bidirectional SA
// Eq.10 / P204: self-attention along the k draft slots of one context row, unmasked
// (BIDIR_LOCAL), no RoPE; effective batch B. One CTA per (b, head); warp w takes query slots
// i = w, w + 4, ...: scores by lane-parallel dot products + warp sums, softmax over the k slots in
// registers, then each lane forms hd/32 output dimensions.
template <typename TA>
__global__ void __launch_bounds__(128) bidir_attn_kernel(const TA* qkv, int k, int Hq, int Hkv, int hd, int causal,
                                                         TA* out) {
  KtScope kt_(KT_BIDIR, (uint32_t)(k));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  extern __shared__ float fs[];
  const int b = blockIdx.x, h = blockIdx.y;
  const int G = Hq / Hkv, kh = h / G;
  const int W = (Hq + 2 * Hkv) * hd;
  float* q = fs;
  float* kk = q + k * hd;
  float* vv = kk + k * hd;
  if constexpr (sizeof(TA) == 2) {  // bf16: four elements per 8-byte load (hd % 4 == 0)
    for (int e = 4 * threadIdx.x; e < k * hd; e += 4 * blockDim.x) {
      const int i = e / hd, dd = e % hd;
      const TA* row = qkv + (size_t)(b * k + i) * W;
      const uint2 a = *reinterpret_cast<const uint2*>(row + h * hd + dd);
      const uint2 c = *reinterpret_cast<const uint2*>(row + (Hq + kh) * hd + dd);
      const uint2 v = *reinterpret_cast<const uint2*>(row + (Hq + Hkv + kh) * hd + dd);
      const uint32_t w3[3][2] = {{a.x, a.y}, {c.x, c.y}, {v.x, v.y}};
      float* dsts[3] = {q, kk, vv};
#pragma unroll
      for (int t = 0; t < 3; ++t)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w3[t][u]));
          dsts[t][e + 2 * u] = f.x;
          dsts[t][e + 2 * u + 1] = f.y;
        }
    }
  } else {
    for (int e = threadIdx.x; e < k * hd; e += blockDim.x) {
      const int i = e / hd, dd = e % hd;
      const TA* row = qkv + (size_t)(b * k + i) * W;
      q[e] = Elt<TA>::to_f(row[h * hd + dd]);
      kk[e] = Elt<TA>::to_f(row[(Hq + kh) * hd + dd]);
      vv[e] = Elt<TA>::to_f(row[(Hq + Hkv + kh) * hd + dd]);
    }
  }
  __syncthreads();
  const float scale = rsqrtf((float)hd);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int i = warp; i < k; i += nw) {
    float sc[16];
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (j >= k) break;
      float a = 0.f;
      for (int dd = lane; dd < hd; dd += 32) a = fmaf(q[i * hd + dd], kk[j * hd + dd], a);
      a = warp_sum(a) * scale;
      sc[j] = (causal && j > i) ? -INFINITY : a;
      mx = fmaxf(mx, sc[j]);
    }
    float l = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (j >= k) break;
      sc[j] = (sc[j] == -INFINITY) ? 0.f : expf(sc[j] - mx);
      l += sc[j];
    }
    for (int dd = lane; dd < hd; dd += 32) {
      float a = 0.f;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j >= k) break;
        a = fmaf(sc[j] / l, vv[j * hd + dd], a);  // (the same quotient every dd: hoisted by the compiler)
      }
      out[(size_t)(b * k + i) * Hq * hd + h * hd + dd] = Elt<TA>::from_f(a);
    }
  }
}

// ------------------------------------------------------------------------ gather
// "-Pos" (T4 ablation, DESIGN.md §3 reading): every draft slot gets the normalised context row plus its
// own position vector. One CTA per sequence; fixed reduction tree (blockDim 256).
__global__ void __launch_bounds__(256) pos_broadcast_kernel(const float* src, const float* gamma, const float* bias,
                                                            int k, int d, float eps, float* D) {
  KtScope kt_(KT_GATHER, (uint32_t)(d));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  __shared__ float red[32];
  const int b = blockIdx.x;
  const float* x = src + (size_t)b * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) ss = fmaf(x[i], x[i], ss);
  ss = block_sum_dyn(ss, red);
  const float r = 1.0f / sqrtf(ss / (float)d + eps);
  for (int j = 0; j < k; ++j)
    for (int i = threadIdx.x; i < d; i += blockDim.x)
      D[((size_t)b * k + j) * d + i] = x[i] * r * gamma[i] + bias[(size_t)j * d + i];
}
cudaError_t launch_pos_broadcast(const float* src, const float* gamma, const float* bias, int B, int k, int d, float eps,
                                 float* D, cudaStream_t s) {
  launch_k(pos_broadcast_kernel, dim3(B), dim3(256), 0, s, src, gamma, bias, k, d, eps, D);
  return cudaGetLastError();
}

__global__ void gather_rows_kernel(const float* src, int q_len, const int* idx, int const_idx, int d, float* dst) {
  KtScope kt_(KT_GATHER, (uint32_t)(d));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  const int b = blockIdx.x;
  const int r = idx ? idx[b] : const_idx;
  const float* sr = src + ((size_t)b * q_len + r) * d;
  if (d % 4 == 0) {
    for (int i = 4 * threadIdx.x; i < d; i += 4 * blockDim.x)
      *reinterpret_cast<float4*>(dst + (size_t)b * d + i) = *reinterpret_cast<const float4*>(sr + i);
  } else {
    for (int i = threadIdx.x; i < d; i += blockDim.x) dst[(size_t)b * d + i] = sr[i];
  }
}

// ------------------------------------------------------------------------ argmax (lowest id on ties)
constexpr int kArgmaxSlice = 2048;
int argmax_splits(int V) { return (V + kArgmaxSlice - 1) / kArgmaxSlice; }

SF_DEV void better(float& bv, int& bi, float v, int i) {
  if (v > bv || (v == bv && i < bi)) {
    bv = v;
    bi = i;
  }
}
__global__ void __launch_bounds__(256) argmax_partial_kernel(const float* logits, int V, int nsplit, float* pval,
                                                             int* pidx, int* err) {
  KtScope kt_(KT_ARGMAX_P, (uint32_t)(V));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  __shared__ float sv[8];
  __shared__ int si[8];
  const int row = blockIdx.y, sp = blockIdx.x;
  const int lo = sp * kArgmaxSlice, hi = min(V, lo + kArgmaxSlice);
  const float* x = logits + (size_t)row * V;
  float bv = -INFINITY;
  int bi = INT_MAX;
  bool bad = false;
  for (int i = lo + threadIdx.x; i < hi; i += 256) {
    const float v = x[i];
    if (!isfinite(v)) bad = true;
    better(bv, bi, v, i);
  }
  if (bad) atomicOr(err, 1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    better(bv, bi, ov, oi);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sv[w] = bv;
    si[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 1; j < 8; ++j) better(bv, bi, sv[j], si[j]);
    pval[row * nsplit + sp] = bv;
    pidx[row * nsplit + sp] = bi;
  }
}
__global__ void argmax_final_kernel(const float* pval, const int* pidx, int R, int nsplit, int* out) {
  KtScope kt_(KT_ARGMAX_F, (uint32_t)(nsplit));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= R) return;
  float bv = -INFINITY;
  int bi = INT_MAX;
  for (int s = 0; s < nsplit; ++s) better(bv, bi, pval[row * nsplit + s], pidx[row * nsplit + s]);
  out[row] = (bi == INT_MAX) ? 0 : bi;
}

// Tensor parallelism (vocabulary-sharded LM head): each rank packs its rows' best (logit, id) as
// key = orderable(logit) << 32 | (0xFFFFFFFF - (v0 + id)), the ranks max-reduce the keys (largest
// logit, lowest id on ties -- the same rule as above over the whole vocabulary), and the winner's id
// is unpacked.
SF_DEV unsigned long long argmax_key(float v, unsigned id) {
  unsigned u = __float_as_uint(v == 0.f ? 0.f : v);  // (-0 == +0, as in better())
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);  // order-preserving map of the finite floats
  return ((unsigned long long)u << 32) | (0xFFFFFFFFu - id);
}
__global__ void argmax_key_kernel(const float* pval, const int* pidx, int R, int nsplit, int v0,
                                  unsigned long long* keys) {
  KtScope kt_(KT_ARGMAX_F, (uint32_t)(nsplit));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= R) return;
  float bv = -INFINITY;
  int bi = INT_MAX;
  for (int s = 0; s < nsplit; ++s) better(bv, bi, pval[row * nsplit + s], pidx[row * nsplit + s]);
  keys[row] = (bi == INT_MAX) ? 0ull : argmax_key(bv, (unsigned)(v0 + bi));
}
__global__ void argmax_unkey_kernel(unsigned long long* keys, int R, int* out, int reset) {
  KtScope kt_(KT_ARGMAX_F, 0u);
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= R) return;
  const unsigned long long k = keys[row];
  out[row] = k ? (int)(0xFFFFFFFFu - (unsigned)(k & 0xFFFFFFFFull)) : 0;
  if (reset) keys[row] = 0ull;  // ready for the next fused-argmax launch
}

// ------------------------------------------------------------------------ accept + commit
// P25: accept only drafts equal to the base model's greedy outputs. Single CTA (B <= 1024).
// ------------------------------------------------------------------------ KV page pool (NEXT-4)
// A stack of free page ids (pool[0..*top)) shared by the handle's sequences; sequence b's logical page i
// is bt[b pps + i] for i < alloc_cnt[b]. Pages are taken just before positions are written: up to
// position need_pos - 1 (prefill: P + k + 1; after each commit: seq_len + k + 1, the next verify's
// block). An empty pool sets the sticky capacity bit (err |= 2) and leaves the sequence short.
SF_DEV void page_take(int b, int need_pos, const PagePool& pp) {
  const int need = min(pp.pps, (need_pos + 15) / 16);
  int have = pp.alloc_cnt[b];
  while (have < need) {
    const int t = atomicSub(pp.top, 1) - 1;
    if (t < 0) {
      atomicAdd(pp.top, 1);
      atomicOr(pp.err, 2);
      break;
    }
    pp.bt[b * pp.pps + have] = pp.pool[t];
    ++have;
  }
  pp.alloc_cnt[b] = have;
}
__global__ void page_take_kernel(int b0, int nb, const int* seq_len, int extra, PagePool pp) {
  KtScope kt_(KT_MISC, (uint32_t)(6));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nb) page_take(b0 + i, (seq_len ? seq_len[b0 + i] : 0) + extra, pp);
}
__global__ void page_release_kernel(int b0, int nb, PagePool pp) {
  KtScope kt_(KT_MISC, (uint32_t)(7));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nb) return;
  const int b = b0 + i, cnt = pp.alloc_cnt[b];
  const int t = atomicAdd(pp.top, cnt);
  for (int j = 0; j < cnt; ++j) pp.pool[t + j] = pp.bt[b * pp.pps + j];
  pp.alloc_cnt[b] = 0;
}
__global__ void page_reset_kernel(int n_pages, int B, PagePool pp) {
  KtScope kt_(KT_MISC, (uint32_t)(8));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_pages) pp.pool[i] = n_pages - 1 - i;  // (the stack hands out pages 0, 1, 2, ... first)
  if (i < B) pp.alloc_cnt[i] = 0;
  if (i == 0) *pp.top = n_pages;
}
cudaError_t launch_page_take(int b0, int nb, const int* seq_len, int extra, const PagePool& pp, cudaStream_t s) {
  launch_k(page_take_kernel, dim3((nb + 127) / 128), dim3(128), 0, s, b0, nb, seq_len, extra, pp);
  return cudaGetLastError();
}
cudaError_t launch_page_release(int b0, int nb, const PagePool& pp, cudaStream_t s) {
  launch_k(page_release_kernel, dim3((nb + 127) / 128), dim3(128), 0, s, b0, nb, pp);
  return cudaGetLastError();
}
cudaError_t launch_page_reset(int n_pages, int B, const PagePool& pp, cudaStream_t s) {
  launch_k(page_reset_kernel, dim3((std::max(n_pages, B) + 255) / 256), dim3(256), 0, s, n_pages, B, pp);
  return cudaGetLastError();
}

__global__ void accept_kernel(int B, int k, const int* draft, const int* greedy, int* seq_len, int* n_prev,
                              int* last_token, int* r_b, int* accept_len, int* emitted, int* step_counter,
                              int* accept_log, int* emitted_log, const int* log_cap_dev, PagePool pp) {
  KtScope kt_(KT_ACCEPT, (uint32_t)(k));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  const int b = threadIdx.x;
  const int step = step_counter ? *step_counter : 0;
  const int log_cap = (accept_log || emitted_log) && log_cap_dev ? *log_cap_dev : 0;
  if (b < B) {
    const int* g = greedy + b * (k + 1);
    int m = 0;
    while (m < k && draft[b * k + m] == g[m]) ++m;
    for (int i = 0; i <= k; ++i) {
      const int e = (i <= m) ? g[i] : -1;
      emitted[b * (k + 1) + i] = e;
      if (emitted_log && step < log_cap) emitted_log[((size_t)step * B + b) * (k + 1) + i] = e;
    }
    accept_len[b] = m;
    if (accept_log && step < log_cap) accept_log[(size_t)step * B + b] = m;
    n_prev[b] = seq_len[b];
    seq_len[b] += m + 1;
    last_token[b] = g[m];
    r_b[b] = m;
    if (pp.pool) page_take(b, seq_len[b] + k + 1, pp);  // pages for the next verify block
  }
  __syncthreads();
  if (threadIdx.x == 0 && step_counter) *step_counter = step + 1;
}

__global__ void force_drafts_kernel(int B, int k, int V, const int* cont, int cont_len, const int* corrupt,
                                    int corrupt_steps, const int* seq_len, const int* prompt_len,
                                    const int* step_counter, int* draft) {
  KtScope kt_(KT_MISC, (uint32_t)(1));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int gidx = seq_len[b] - prompt_len[b];
  const int step = step_counter ? *step_counter : 0;
  const int cs = corrupt ? corrupt[(size_t)(step % corrupt_steps) * B + b] : k + 1;
  for (int j = 1; j <= k; ++j) {
    const int ci = min(gidx + j, cont_len - 1);
    int tok = cont[(size_t)b * cont_len + ci];
    if (j == cs) tok = (tok + 1) % V;
    draft[b * k + j - 1] = tok;
  }
}

__global__ void fill_kernel(int* p, int n, int v) {
  KtScope kt_(KT_MISC, (uint32_t)(2));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void prefill_finish_kernel(int B, int P, const int* greedy, int* seq_len, int* n_prev, int* last_token,
                                      int* r_b, int* prompt_len, int* first_out) {
  KtScope kt_(KT_MISC, (uint32_t)(3));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  seq_len[b] = P;
  n_prev[b] = P;
  last_token[b] = greedy[b];
  r_b[b] = 0;
  prompt_len[b] = P;
  if (first_out) first_out[b] = greedy[b];
}

// ======================================================================== launchers
#define SF_GRID(n, t) (((n) + (t)-1) / (t))

cudaError_t launch_rope_table(float2* table, int max_seq, int hd, float theta, cudaStream_t s) {
  const int n = max_seq * hd / 2;
  launch_k(rope_table_kernel, dim3(SF_GRID(n, 256)), dim3(256), 0, s, table, max_seq, hd, theta);
  return cudaGetLastError();
}
cudaError_t launch_build_verify_rows(int B, int k, const int* last_token, const int* draft, int* tok_rows,
                                     cudaStream_t s) {
  launch_k(build_verify_rows_kernel, dim3(SF_GRID(B * (k + 1), 128)), dim3(128), 0, s, B, k, last_token, draft, tok_rows);
  return cudaGetLastError();
}
cudaError_t launch_build_prefill_rows(int B, int P, int c0, int C, const int* tokens, int* tok_rows, int* pos0,
                                      cudaStream_t s) {
  launch_k(build_prefill_rows_kernel, dim3(SF_GRID(max(B * C, B), 128)), dim3(128), 0, s, B, P, c0, C, tokens, tok_rows, pos0);
  return cudaGetLastError();
}
cudaError_t launch_embed(bool bf, const int* tok, const void* embed, int T, int d, int vocab, float* resid,
                         float* tap0, cudaStream_t s) {
  if (bf && d % 8 == 0)
    return launch_k(embed_v_kernel, dim3(T), dim3(std::min(1024, d / 8)), 0, s, tok, (const __nv_bfloat16*)embed, d,
                    vocab, resid, tap0);
  if (bf)
    launch_k(embed_kernel<__nv_bfloat16>, dim3(T), dim3(256), 0, s, tok, (const __nv_bfloat16*)embed, d, vocab, resid, tap0);
  else
    launch_k(embed_kernel<float>, dim3(T), dim3(256), 0, s, tok, (const float*)embed, d, vocab, resid, tap0);
  return cudaGetLastError();
}
static cudaError_t launch_rms_rows(const float* x, int64_t x_stride, int in_ld, const float* g, float eps, int T,
                                   int groups, int d, __nv_bfloat16* out, int out_ld, cudaStream_t s) {
  const int ng = row_ng(d);
  const dim3 grid(T, groups), block(d / (4 * ng));
  switch (ng) {
    case 1: return launch_k(rms_rows_kernel<1>, grid, block, 0, s, x, x_stride, in_ld, g, eps, d, out, out_ld);
    case 2: return launch_k(rms_rows_kernel<2>, grid, block, 0, s, x, x_stride, in_ld, g, eps, d, out, out_ld);
    case 3: return launch_k(rms_rows_kernel<3>, grid, block, 0, s, x, x_stride, in_ld, g, eps, d, out, out_ld);
    default: return launch_k(rms_rows_kernel<4>, grid, block, 0, s, x, x_stride, in_ld, g, eps, d, out, out_ld);
  }
}
cudaError_t launch_rmsnorm(bool bf, const float* in, int in_ld, const float* gamma, float eps, int T, int d,
                           void* out, int out_ld, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  if (bf && row_ng(d) && in_ld % 4 == 0 && out_ld % 4 == 0)
    return launch_rms_rows(in, 0, in_ld, gamma, eps, T, 1, d, (__nv_bfloat16*)out, out_ld, s);
  if (bf)
    launch_k(rmsnorm_kernel<__nv_bfloat16>, dim3(T), dim3(256), 0, s, in, in_ld, gamma, eps, d, (__nv_bfloat16*)out, out_ld);
  else
    launch_k(rmsnorm_kernel<float>, dim3(T), dim3(256), 0, s, in, in_ld, gamma, eps, d, (float*)out, out_ld);
  return cudaGetLastError();
}
cudaError_t launch_group_rms(bool bf, const float* taps, int64_t tap_stride, const float* scales, float eps, int T,
                             int d, void* out, cudaStream_t s) {
  if (bf && row_ng(d) && tap_stride % 4 == 0)
    return launch_rms_rows(taps, tap_stride, d, scales, eps, T, 4, d, (__nv_bfloat16*)out, 4 * d, s);
  if (bf)
    launch_k(group_rms_kernel<__nv_bfloat16>, dim3(T), dim3(256), 0, s, taps, tap_stride, scales, eps, d, (__nv_bfloat16*)out);
  else
    launch_k(group_rms_kernel<float>, dim3(T), dim3(256), 0, s, taps, tap_stride, scales, eps, d, (float*)out);
  return cudaGetLastError();
}
cudaError_t launch_rope_append(bool bf, const void* qkv, int T, int q_len, const int* pos0, const float2* rope,
                               int Hq, int Hkv, int hd, const int* bt, int pps, void* Kp, void* Vp, void* q_out,
                               bool q_bf16, cudaStream_t s, bool pair_rows) {
  if (bf && q_bf16 && hd == 128 && pair_rows) {
    const int items = T * (Hq + 2 * Hkv);
    const int grid = std::max(1, std::min((items + 15) / 16, 148 * 4));
    return launch_k(rope_append128_kernel, dim3(grid), dim3(256), 0, s, (const __nv_bfloat16*)qkv, T, q_len, pos0, rope,
                    Hq, Hkv, bt, pps, (__nv_bfloat16*)Kp, (__nv_bfloat16*)Vp, (__nv_bfloat16*)q_out);
  }
  const int hpw = 1;                      // heads per warp
  const int wpc = T >= 64 ? 8 : 4;          // warps per CTA: fewer, fuller CTAs for long blocks
  const dim3 grid(T, (Hq + 2 * Hkv + wpc * hpw - 1) / (wpc * hpw));
  const bool v2 = (hd / 2) % 64 == 0;
  if (bf) {
    auto k = q_bf16 ? (v2 ? rope_append_kernel<__nv_bfloat16, 2, true> : rope_append_kernel<__nv_bfloat16, 1, true>)
                    : (v2 ? rope_append_kernel<__nv_bfloat16, 2, false> : rope_append_kernel<__nv_bfloat16, 1, false>);
    return launch_k(k, grid, dim3(32 * wpc), 0, s, (const __nv_bfloat16*)qkv, q_len, pos0, rope, Hq, Hkv, hd, bt, pps,
                    (__nv_bfloat16*)Kp, (__nv_bfloat16*)Vp, q_out, hpw);
  }
  auto k = v2 ? rope_append_kernel<float, 2, false> : rope_append_kernel<float, 1, false>;
  return launch_k(k, grid, dim3(32 * wpc), 0, s, (const float*)qkv, q_len, pos0, rope, Hq, Hkv, hd, bt, pps, (float*)Kp,
                  (float*)Vp, q_out, hpw);
}

template <typename TKV, int HD>
static cudaError_t attn_impl(const AttnParams& p, cudaStream_t s) {
  constexpr int VEC = 16 / sizeof(TKV);
  const size_t smem = (size_t)kAttnChunk * (HD + VEC) * sizeof(TKV) + (size_t)kAttnChunk * HD * sizeof(TKV) +
                      (size_t)QT * HD * 4 + (size_t)QT * kAttnChunk * 4 + QT * 2 * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_partial_kernel<TKV, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const int G = p.Hq / p.Hkv;
  const int ntiles = (p.q_len * G + QT - 1) / QT;
  const int nch = (p.max_key + kAttnChunk - 1) / kAttnChunk;
  dim3 grid(nch, p.Hkv * ntiles, p.B);
  launch_k(attn_partial_kernel<TKV, HD>, dim3(grid), dim3(128), smem, s, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  dim3 g2(p.B * p.q_len, p.Hq);
  if (sizeof(TKV) == 2)
    launch_k(attn_combine_kernel<__nv_bfloat16>, dim3(g2), dim3(min(HD, 128)), 0, s, p);
  else
    launch_k(attn_combine_kernel<float>, dim3(g2), dim3(min(HD, 128)), 0, s, p);
  return cudaGetLastError();
}
cudaError_t launch_attention(bool bf, const AttnParams& p, cudaStream_t s) {
  if (bf && p.hd == 128) return launch_attention_fd(p, s);  // flash-decoding, no split-KV partials
  if (bf) {
    switch (p.hd) {
      case 64: return attn_impl<__nv_bfloat16, 64>(p, s);
      case 128: return attn_impl<__nv_bfloat16, 128>(p, s);
      case 16: return attn_impl<__nv_bfloat16, 16>(p, s);
    }
  } else {
    switch (p.hd) {
      case 16: return attn_impl<float, 16>(p, s);
      case 64: return attn_impl<float, 64>(p, s);
      case 128: return attn_impl<float, 128>(p, s);
    }
  }
  return cudaErrorInvalidValue;
}
cudaError_t launch_bidir_attention(bool bf, const void* qkv, int B, int k, int Hq, int Hkv, int hd, bool causal,
                                   void* out, cudaStream_t s) {
  dim3 grid(B, Hq);
  const size_t smem = (size_t)(3 * k * hd) * 4;
  if (bf)
    launch_k(bidir_attn_kernel<__nv_bfloat16>, dim3(grid), dim3(128), smem, s, (const __nv_bfloat16*)qkv, k, Hq, Hkv, hd, causal,
                                                            (__nv_bfloat16*)out);
  else
    launch_k(bidir_attn_kernel<float>, dim3(grid), dim3(128), smem, s, (const float*)qkv, k, Hq, Hkv, hd, causal, (float*)out);
  return cudaGetLastError();
}
cudaError_t launch_gather_rows(const float* src, int q_len, const int* idx, int const_idx, int B, int d, float* dst,
                               cudaStream_t s) {
  launch_k(gather_rows_kernel, dim3(B), dim3(std::max(32, std::min(1024, d / 4 / 32 * 32))), 0, s, src, q_len, idx,
           const_idx, d, dst);
  return cudaGetLastError();
}
struct BufList {
  const void* p[8];
};
__global__ void reduce_bufs_kernel(BufList bl, int n, int64_t count, int max_u64, void* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    if (max_u64 == 1) {
      unsigned long long m = 0;
      for (int q = 0; q < n; ++q) m = max(m, reinterpret_cast<const unsigned long long*>(bl.p[q])[i]);
      reinterpret_cast<unsigned long long*>(out)[i] = m;
    } else if (max_u64 == 2) {  // bf16 sum, fp32 accumulation in rank order, one rounding
      float a = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(bl.p[0])[i]);
      for (int q = 1; q < n; ++q) a += __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(bl.p[q])[i]);
      reinterpret_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(a);
    } else {
      float a = reinterpret_cast<const float*>(bl.p[0])[i];
      for (int q = 1; q < n; ++q) a += reinterpret_cast<const float*>(bl.p[q])[i];  // buffer (rank) order
      reinterpret_cast<float*>(out)[i] = a;
    }
  }
}
cudaError_t launch_reduce_bufs(const void* const* bufs, int n, int64_t count, int mode, void* out, cudaStream_t s) {
  if (n < 1 || n > 8) return cudaErrorInvalidValue;
  BufList bl{};
  for (int q = 0; q < n; ++q) bl.p[q] = bufs[q];
  const int grid = (int)std::min<int64_t>(1184, (count + 255) / 256);
  reduce_bufs_kernel<<<std::max(grid, 1), 256, 0, s>>>(bl, n, count, mode, out);
  return cudaGetLastError();
}
// tensor parallelism, bf16 all-reduce (the default; SF_FLAG_TP_F32_REDUCE: fp32): the rank's fp32 row-parallel output
// rounded to bf16 (RNE) for the collective, and the reduced bf16 sum widened back
__global__ void cvt_f32_bf16_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out, int64_t n, int to_bf) {
  KtScope kt_(KT_MISC, (uint32_t)(9));
  pdl_wait();
  kt_.mark();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (to_bf) out[i] = __float2bfloat16_rn(in[i]);
    else const_cast<float*>(in)[i] = __bfloat162float(out[i]);
  }
}
cudaError_t launch_cvt_f32_bf16(float* f32, __nv_bfloat16* bf, int64_t n, bool to_bf, cudaStream_t s) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(1184, (n + 255) / 256));
  return launch_k(cvt_f32_bf16_kernel, dim3(grid), dim3(256), 0, s, (const float*)f32, bf, n, to_bf ? 1 : 0);
}

cudaError_t launch_argmax_key(const float* logits, int R, int V, int v0, float* pval, int* pidx,
                              unsigned long long* keys, int* err, cudaStream_t s) {
  const int ns = argmax_splits(V);
  const dim3 grid(ns, R);
  launch_k(argmax_partial_kernel, dim3(grid), dim3(256), 0, s, logits, V, ns, pval, pidx, err);
  return launch_k(argmax_key_kernel, dim3(SF_GRID(R, 128)), dim3(128), 0, s, pval, pidx, R, ns, v0, keys);
}
cudaError_t launch_argmax_unkey(unsigned long long* keys, int R, int* out, cudaStream_t s, bool reset) {
  return launch_k(argmax_unkey_kernel, dim3(SF_GRID(R, 128)), dim3(128), 0, s, keys, R, out, reset ? 1 : 0);
}

cudaError_t launch_argmax(const float* logits, int R, int V, float* pval, int* pidx, int* out, int* err,
                          cudaStream_t s) {
  const int ns = argmax_splits(V);
  dim3 grid(ns, R);
  launch_k(argmax_partial_kernel, dim3(grid), dim3(256), 0, s, logits, V, ns, pval, pidx, err);
  launch_k(argmax_final_kernel, dim3(SF_GRID(R, 128)), dim3(128), 0, s, pval, pidx, R, ns, out);
  return cudaGetLastError();
}
cudaError_t launch_accept(int B, int k, const int* draft, const int* greedy, int* seq_len, int* n_prev,
                          int* last_token, int* r_b, int* accept_len, int* emitted, int* step_counter,
                          int* accept_log, int* emitted_log, const int* log_cap, const PagePool& pp, cudaStream_t s) {
  const int th = ((B + 31) / 32) * 32;
  launch_k(accept_kernel, dim3(1), dim3(th), 0, s, B, k, draft, greedy, seq_len, n_prev, last_token, r_b, accept_len, emitted,
                                 step_counter, accept_log, emitted_log, log_cap, pp);
  return cudaGetLastError();
}
cudaError_t launch_force_drafts(int B, int k, int V, const int* cont, int cont_len, const int* corrupt,
                                int corrupt_steps, const int* seq_len, const int* prompt_len,
                                const int* step_counter, int* draft, cudaStream_t s) {
  launch_k(force_drafts_kernel, dim3(SF_GRID(B, 128)), dim3(128), 0, s, B, k, V, cont, cont_len, corrupt, corrupt_steps, seq_len,
                                                      prompt_len, step_counter, draft);
  return cudaGetLastError();
}
cudaError_t launch_fill(int* p, int n, int v, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  launch_k(fill_kernel, dim3(SF_GRID(n, 256)), dim3(256), 0, s, p, n, v);
  return cudaGetLastError();
}
cudaError_t launch_prefill_finish(int B, int P, const int* greedy, int* seq_len, int* n_prev, int* last_token,
                                  int* r_b, int* prompt_len, int* first_out, cudaStream_t s) {
  launch_k(prefill_finish_kernel, dim3(SF_GRID(B, 128)), dim3(128), 0, s, B, P, greedy, seq_len, n_prev, last_token, r_b,
                                                         prompt_len, first_out);
  return cudaGetLastError();
}

cudaError_t kt_setup_kernels(void* rec, unsigned* cnt, unsigned cap) {
  KtBuf b;
  b.rec = reinterpret_cast<KtRec*>(rec);
  b.cnt = cnt;
  b.cap = cap;
  return kt_setup_tu(b);
}

}  // namespace sf
