// gemm_seq.cuh -- the layer-sequence kernel (included by gemm.cu: one translation unit with the
// stream-K partition, the PTX wrappers and the host helpers it shares with gemm_sk_kernel).
//
// At small verify blocks (T = B(k+1) <= 80 rows: batch 1..16) a base layer is weight streaming
// (PAPER P72-86, Eq.1-2: AI_m = 1 at B = 1), and the separate launches of round 1 lost ~40% of it at
// the kernel boundaries: every GEMM launch paid ~4 us before its first MMA (CTA setup, first weight
// load) and ~6 us of range imbalance and fixup tail after its last one, during which the HBM idled.
// This kernel runs the part of a base layer between two attentions as ONE persistent launch:
//
//   O-proj (EPI_PARTIAL) -> residual + RMS_ffn (consumer) -> gate/up (SwiGLU) -> down (EPI_PARTIAL)
//   -> residual (+ hook tap) + next RMSNorm (consumer) -> next layer's QKV (fused RoPE / KV append,
//   or EPI_PARTIAL + the RoPE consumer at T >= 64)
//
// Every CTA pair keeps its own stream-K ranges of each GEMM phase -- the same partition, MMA shapes,
// k order and epilogue arithmetic as the standalone launches (so every output bit is the same and
// batch invariance across the T threshold holds, reading C23) -- but the TMA producer streams the
// weights of the NEXT phases into the smem ring as soon as slots free up, independently of the
// data dependencies; only the small activation tile of a stage waits until its phase's inputs are
// complete (a grid-wide completion counter per phase). The consumers (residual + RMSNorm, RoPE /
// append) run on the epilogue warps of the CTAs with the same per-element arithmetic as
// resid_norm_kernel / rope_partial_kernel (the norm's reduction tree is replayed exactly: virtual
// thread t of the 1024-thread row kernel = lane t % 32 of warp (t / 32) % 8 in round t / 256).
// Requires all CTAs co-resident (one per SM, grid = the co-resident CTA pairs, as the standalone
// kernel), which the cluster occupancy query guarantees.

struct SeqPhase {
  int kind;
  // GEMM phase: k-blocks, pair tiles, work groups (pairs), tile-entry cost, tensor-map slot, epilogue
  int mode, kb, n_tiles, G, drain, map;
  GemmEpi epi;
  // consumer phase: the producing GEMM's partial geometry (pairs, k-blocks, tile-entry cost, pair
  // tiles, slot row stride)
  int pG, pkb, pdrain, pntiles, Tslot;
  // SEQ_RESID_NORM: x = resid + partials; out = x; tap = x; xn = bf16(x rs gamma)
  const float* resid;
  float* out;
  float* tap;
  const float* gamma;
  __nv_bfloat16* xn;
  int d;
  float eps;
};

struct SeqParams {
  int T, Tp, NT, stages, nbuf, cgrp, npre, n_phases;
  uint32_t tmem_cols;
  float* partial;  // split-K partial slots (the standalone GEMMs' scratch)
  int* flags;      // per-CTA tail-piece flags (standalone layout)
  int* sync;       // kSeqSyncInts ints (zeroed once): launch epoch, exit counter, per-phase completion
                   // counters, per-(phase, CTA) and per-(phase, 128-row tile) flags -- all monotonic
                   // in the epoch, so nothing is re-armed between launches
  SeqPhase ph[kSeqMaxPhases];
};
struct SeqMaps {
  CUtensorMap w[kSeqMaxGemm];  // tile-contiguous weights ([N * K / 64, 64] view)
  CUtensorMap a[kSeqMaxGemm];  // activations [T, K], box NT / 2 rows
};
static_assert(sizeof(SeqParams) + sizeof(SeqMaps) <= 4000, "kernel parameter space");
// sync block layout
constexpr int kSeqRows = 128;  // T limit
SF_DEV int* seq_done(int* sy, int ph) { return sy + 8 + ph; }
// quarter task qq of row `row` has published its sums in this launch: flag == the launch's epoch mark
// (epoch-stamped, so rows a launch does not touch -- a shorter block -- need no re-arming)
SF_DEV int* seq_rowflag(int* sy, int ph, int row, int qq) { return sy + 64 + (ph * kSeqRows + row) * 4 + qq; }
SF_DEV float* seq_ss(int* sy, int ph, int row) {  // [32] per-virtual-warp sums of squares of a row
  return reinterpret_cast<float*>(sy + 64 + kSeqMaxPhases * kSeqRows * 4) + ((size_t)ph * kSeqRows + row) * 32;
}
static_assert(64 + kSeqMaxPhases * kSeqRows * (4 + 32) <= kSeqSyncInts, "sync block");

SF_DEV int rn_ng_dev(int d) {  // float4 groups per virtual thread (rn_ng, device copy)
  for (int ng = 1; ng <= 4; ++ng)
    if (d % (4 * ng * 32) == 0 && d / (4 * ng) <= 1024) return ng;
  return 0;
}
SF_DEV void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
SF_DEV bool mbar_test(uint64_t* bar, uint32_t phase) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return done != 0;
}

__global__ void __launch_bounds__(384, 1)
gemm_seq_kernel(const __grid_constant__ SeqMaps maps, const __grid_constant__ SeqParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_u32 + 1023u) & ~1023u) - raw_u32);
  const int a_rows = p.NT / 2;  // this CTA's half of the activation tile (CTA pair)
  const int stage_bytes = BM * BK * 2 + a_rows * BK * 2;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)p.stages * stage_bytes);
  uint64_t* empty = full + p.stages;
  uint64_t* accf = empty + p.stages;  // [2]
  uint64_t* acce = accf + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + 2);
  float* red = reinterpret_cast<float*>(tmem_slot + 4);  // [33] consumer reduction scratch
  int* seg_n = reinterpret_cast<int*>(red + 36);         // [kRnMaxTiles] consumer k-segment tables
  int* seg_off = seg_n + kRnMaxTiles;                    // [kRnMaxTiles][kRnMaxSeg] float offsets

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const uint32_t prank = rank & 1u, pbase = rank & ~1u;
  const int c = blockIdx.x >> 1;  // work group (CTA pair)
  KtScope kt_(KT_GEMM_SEQ, (uint32_t)p.n_phases, 128);

  // this group's stream-K range of GEMM phase ph (the standalone launch's partition)
  auto prange = [&](int ph, long long& u0, long long& u1) -> bool {
    const SeqPhase& P = p.ph[ph];
    if (P.kind != SEQ_GEMM || c >= P.G) {
      u0 = u1 = 0;
      return false;
    }
    u0 = sk_begin(c, P.G, P.n_tiles, P.kb, P.drain);
    u1 = sk_begin(c + 1, P.G, P.n_tiles, P.kb, P.drain);
    return u1 > u0;
  };

  if (threadIdx.x == 0) {
    for (int ph = 0; ph < p.n_phases; ++ph)
      if (p.ph[ph].kind == SEQ_GEMM) {
        prefetch_tmap(&maps.w[p.ph[ph].map]);
        prefetch_tmap(&maps.a[p.ph[ph].map]);
      }
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&accf[b], 1);
      mbar_init(&acce[b], 2);  // both CTAs' epilogues release the accumulator
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(p.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---- TMA producer: two cursors over the (phase, unit) sequence. The weight cursor runs ahead as
    // ring slots free up (weights never depend on earlier phases); the activation cursor issues a
    // stage's activation tile once its phase's inputs are complete (done[phase - 1] == #CTAs, or the
    // previous kernel for phase 0).
    // (int cursors advanced incrementally: no 64-bit division per unit on this single-warp path)
    // Plain scalar cursors (no lambdas over structs: they would live in local memory on this
    // per-unit path). w*: the weight cursor, a*: the activation cursor; (ph, u, u1, t, k, kb, map) of
    // the current phase range, ring slot s and pass parity par.
    const int stages = p.stages, cgrp = p.cgrp, n_ph = p.n_phases;
    int wph = 0, wu = 0, wu1 = 0, wt = 0, wk = 0, wkb = 1, wmap = 0, ws = 0, wpar = 0;
    int aph = 0, au = 0, au1 = 0, at = 0, ak = 0, akb = 1, amap = 0, as = 0;
#define SF_SEQ_SEEK(PH, U, U1, T_, K_, KB, MAP, FROM)         \
  do {                                                          \
    for (PH = (FROM); PH < n_ph; ++PH) {                        \
      long long a0_, a1_;                                       \
      if (prange(PH, a0_, a1_)) {                               \
        U = (int)a0_, U1 = (int)a1_, KB = p.ph[PH].kb;          \
        MAP = p.ph[PH].map, T_ = U / KB, K_ = U - T_ * KB;      \
        break;                                                  \
      }                                                         \
    }                                                           \
  } while (0)
    SF_SEQ_SEEK(wph, wu, wu1, wt, wk, wkb, wmap, 0);
    aph = wph, au = wu, au1 = wu1, at = wt, ak = wk, akb = wkb, amap = wmap;
    int pending = 0;  // units whose weights are issued but not their activations
#define SF_SEQ_ISSUE_W()                                                                                      \
  do {                                                                                                        \
    if (elect_one()) {                                                                                        \
      uint8_t* st_ = smem + (size_t)ws * stage_bytes;                                                         \
      /* the leader arms the barrier for both CTAs' bytes (weights + activations); a phase cannot complete    \
         before that arrival, so the peer's bytes may land first */                                           \
      if (prank == 0) mbar_arrive_expect_tx(&full[ws], (uint32_t)(2 * stage_bytes));                         \
      tma_load_2d_2sm(st_, &maps.w[wmap], &full[ws], 0, ((wt * 2 + (int)rank) * wkb + wk) * BM, kEvictFirst); \
    }                                                                                                         \
    __syncwarp();                                                                                             \
    ++pending;                                                                                                \
    if (++ws == stages) ws = 0, wpar ^= 1;                                                                    \
    if (++wk == wkb) wk = 0, ++wt;                                                                            \
    if (++wu == wu1) SF_SEQ_SEEK(wph, wu, wu1, wt, wk, wkb, wmap, wph + 1);                                  \
  } while (0)
    // the first weight stages before the grid dependency resolves (PDL)
    for (int i = 0; i < p.npre && wph < n_ph; ++i) SF_SEQ_ISSUE_W();
    pdl_wait();
    pdl_trigger();
    int E1 = 0;  // this launch's epoch mark
    if (lane == 0) E1 = ld_acquire(p.sync) + 1;
    E1 = __shfl_sync(0xffffffffu, E1, 0);
    int ready = 0;  // phases <= ready have all their inputs
    while (aph < n_ph) {
      if (pending > 0) {
        bool go = aph <= ready;
        if (!go) {
          int v = 0;
          if (lane == 0) v = ld_acquire(seq_done(p.sync, aph - 1));
          v = __shfl_sync(0xffffffffu, v, 0);
          if (v >= E1 * (int)gridDim.x) {
            ready = aph;
            go = true;
            fence_proxy_async_global();  // the producers' generic stores -> this TMA read
            if (lane == 0) {
              const unsigned long long tn = kt_now();
              kt_item(0x400000u | ((uint32_t)aph << 8) | (uint32_t)(blockIdx.x & 0xFF), tn, tn, tn);
            }
          }
        }
        if (go) {
          if (elect_one())
            tma_load_2d_2sm(smem + (size_t)as * stage_bytes + BM * BK * 2, &maps.a[amap], &full[as], ak * BK,
                            (int)rank * a_rows, kEvictLast);
          __syncwarp();
          --pending;
          if (++as == stages) as = 0;
          if (++ak == akb) ak = 0, ++at;
          if (++au == au1) SF_SEQ_SEEK(aph, au, au1, at, ak, akb, amap, aph + 1);
          continue;
        }
      }
      if (wph < n_ph) {
        const int gl = ws / cgrp * cgrp + cgrp - 1;  // slots are released in groups of cgrp
        if (pending == 0 && wph <= ready) {
          // steady state inside a ready phase: wait for the slot (hardware-suspended try_wait) and issue
          // the stage's weight and activation tiles together, exactly as the standalone producer does
          mbar_wait(&empty[gl], (uint32_t)wpar ^ 1u);
          if (elect_one()) {
            uint8_t* st_ = smem + (size_t)ws * stage_bytes;
            if (prank == 0) mbar_arrive_expect_tx(&full[ws], (uint32_t)(2 * stage_bytes));
            tma_load_2d_2sm(st_, &maps.w[wmap], &full[ws], 0, ((wt * 2 + (int)rank) * wkb + wk) * BM, kEvictFirst);
            tma_load_2d_2sm(st_ + BM * BK * 2, &maps.a[wmap], &full[ws], wk * BK, (int)rank * a_rows, kEvictLast);
          }
          __syncwarp();
          if (++ws == stages) ws = 0, wpar ^= 1;
          if (++wk == wkb) wk = 0, ++wt;
          as = ws, ak = wk, at = wt;
          if (++wu == wu1) {
            SF_SEQ_SEEK(wph, wu, wu1, wt, wk, wkb, wmap, wph + 1);
            aph = wph, au = wu, au1 = wu1, at = wt, ak = wk, akb = wkb, amap = wmap;
          } else {
            au = wu;
          }
          continue;
        }
        if (pending == 0) {
          mbar_wait(&empty[gl], (uint32_t)wpar ^ 1u);
          SF_SEQ_ISSUE_W();
          continue;
        }
        if (mbar_test(&empty[gl], (uint32_t)wpar ^ 1u)) {
          SF_SEQ_ISSUE_W();
          continue;
        }
      }
      __nanosleep(64);  // an activation waits on its phase's inputs and the ring is full
    }
#undef SF_SEQ_ISSUE_W
#undef SF_SEQ_SEEK
  } else if (warp == 1 && prank == 0) {
    // ---- MMA issuer (pair leader), over every segment of every GEMM phase in order
    const uint32_t idesc = idesc_bf16_f32(2 * BM, p.NT);
    const uint32_t a_off = (uint32_t)(BM * BK * 2) >> 4;
    const int stages = p.stages, cgrp = p.cgrp, nbuf = p.nbuf, NT = p.NT;
    int s = 0, gcnt = 0, gseg = 0;
    uint32_t ph = 0;
    for (int pi = 0; pi < p.n_phases; ++pi) {
      long long u0, u1;
      if (!prange(pi, u0, u1)) continue;
      const int kb = p.ph[pi].kb;
      for (long long lo = u0; lo < u1; ++gseg) {
        const long long hi = min(u1, (lo / kb + 1) * kb);
        const int b = gseg % nbuf;
        mbar_wait(&acce[b], ((uint32_t)(gseg / nbuf) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t dacc = tmem + (uint32_t)(b * NT);
        unsigned long long kf0 = 0;
        for (long long uu = lo; uu < hi; ++uu) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          if (uu == lo && lane == 0) kf0 = kt_now();
          if (elect_one()) {
            const uint64_t dw = sw128_kmajor_desc(smem_u32(smem + (size_t)s * stage_bytes));
            const uint64_t da = dw + a_off;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
              umma_bf16_2sm(dacc, dw + (uint64_t)(kk * 2), da + (uint64_t)(kk * 2), idesc, (uu > lo || kk > 0) ? 1u : 0u);
            if (++gcnt == cgrp) umma_commit_2sm(&empty[s], (uint16_t)(3u << pbase));
          }
          __syncwarp();
          if (gcnt == cgrp) gcnt = 0;
          if (++s == stages) {
            s = 0;
            ph ^= 1u;
          }
        }
        if (elect_one()) umma_commit_2sm(&accf[b], (uint16_t)(3u << pbase));
        __syncwarp();
        if (lane == 0) {
          const unsigned long long tn = kt_now();
          kt_item(0x200000u | ((uint32_t)pi << 8) | (uint32_t)min(255ll, hi - lo), kf0, kf0, tn);
        }
        lo = hi;
      }
    }
  } else if (warp >= 4) {
    // ---- epilogue warps 4..11 (two groups of four, one warp per TMEM lane quadrant): the GEMM
    // phases' segment epilogues in order, and the consumer phases
    pdl_wait();  // partial slots / flags / outputs may still be in use by the previous kernel
    kt_.mark();
    const int quad = warp & 3, m = quad * 32 + lane, gid = (warp - 4) >> 2, ew = warp - 4;
    const bool lead = threadIdx.x == 128;
    const int E1 = *reinterpret_cast<volatile int*>(p.sync) + 1;  // this launch's epoch mark
    const int T = p.T;
    int total_segs = 0;
    for (int pi = 0; pi < p.n_phases; ++pi) {
      long long u0, u1;
      if (prange(pi, u0, u1)) total_segs += (int)((u1 - 1) / p.ph[pi].kb - u0 / p.ph[pi].kb + 1);
    }

    // (QKV RoPE) token c0 + lane's position and destination row, resolved while the MMA still runs
    int pre_pos = 0, pre_c0 = -1, pre_vt = -1;
    unsigned long long pre_row = 0;
    auto rope_dst_row = [&](const RopeEpi& R, int tl, int vt_) -> __nv_bfloat16* {
      const int t = tl + R.t0;
      const int b = t / R.q_len, pos = R.pos0[b] + t % R.q_len;
      if (vt_ < R.Hq) return reinterpret_cast<__nv_bfloat16*>(R.q_out) + ((size_t)t * R.Hq + vt_) * 128;
      const bool isk = vt_ < R.Hq + R.Hkv;
      const int kvh = isk ? vt_ - R.Hq : vt_ - R.Hq - R.Hkv;
      const int blk = R.bt[b * R.pps + pos / 16];
      return reinterpret_cast<__nv_bfloat16*>(isk ? R.Kp : R.Vp) + (((size_t)blk * R.Hkv + kvh) * 16 + pos % 16) * 128;
    };
    auto rope_prefetch = [&](const RopeEpi& R, int c0, int vt_) {
      const int nq = min(32, T - c0);
      pre_c0 = c0;
      pre_vt = vt_;
      if (lane < nq) {
        const int t = c0 + lane + R.t0;
        pre_pos = R.pos0[t / R.q_len] + t % R.q_len;
        pre_row = reinterpret_cast<unsigned long long>(rope_dst_row(R, c0 + lane, vt_));
      }
      if (vt_ < R.Hq + R.Hkv)
        for (int q = 0; q < nq; ++q) {
          const int pq = __shfl_sync(0xffffffffu, pre_pos, q);
          asm volatile("prefetch.global.L1 [%0];" ::"l"(R.table + (size_t)pq * 64 + (m >> 1)));
        }
    };
    // output of one 32-token chunk of this thread's row m (gemm_sk_kernel's direct_store)
    auto direct_store = [&](const SeqPhase& P, float (&v)[32], int c0, int nq, int vt_) {
      if (P.mode == EPI_QKV_ROPE) {
        // lane pair (2i, 2i+1) holds dims (i, i + 64) of the head (pair-interleaved rows); the
        // accumulator is rounded to bf16 first, as the unfused path does
        const RopeEpi& R = P.epi.rope;
        const bool odd = lane & 1;
        const int i = m >> 1, dim = odd ? 64 + i : i;
        const bool rot = vt_ < R.Hq + R.Hkv;
        int my_pos = pre_pos;
        unsigned long long my_row = pre_row;
        if (lane < nq && (c0 != pre_c0 || vt_ != pre_vt)) {
          const int t = c0 + lane + R.t0;
          my_pos = R.pos0[t / R.q_len] + t % R.q_len;
          my_row = reinterpret_cast<unsigned long long>(rope_dst_row(R, c0 + lane, vt_));
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
          reinterpret_cast<__nv_bfloat16*>(row)[dim] = __float2bfloat16_rn(y);
        }
        return;
      }
      // SwiGLU: lane 2i holds gate_i, lane 2i+1 up_i (row-interleaved weight)
      const size_t ldo = (size_t)P.epi.ldo;
      const int f = vt_ * 64 + (m >> 1);
      __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(P.epi.out) + (size_t)c0 * ldo + f;
      swiglu_pair(v, nq, lane, [&](int q, float y) { o[q * ldo] = __float2bfloat16_rn(y); });
    };

    constexpr int kPreT = 8;  // (small T) head pieces with one or two partners: partials loaded early
    float pf1[kPreT], pf2[kPreT];
    bool pre_fix = false;

    auto segment_epilogue = [&](const SeqPhase& P, int pi_cur, long long u, int t, long long se, int b, long long u0) {
      const int kb = P.kb;
      const long long ts = (long long)t * kb, te = ts + kb;
      const uint32_t t_row = tmem + (uint32_t)(b * p.NT) + ((uint32_t)(quad * 32) << 16);
      const int vt = t * 2 + (int)rank;  // 128-row tile of this CTA's rows
      const bool is_full = (u == ts) && (se == te);
      const bool is_head = (u == ts) && !is_full;
      if (P.mode == EPI_PARTIAL || (!is_full && !is_head)) {
        // EPI_PARTIAL: slot 2 group + (first segment of the range ? 0 : 1), summed in k order by the
        // consumer; a tail of a tile owned by another group: this CTA's slot, then its flag
        const bool tail = P.mode != EPI_PARTIAL;
        float* dst = tail ? p.partial + (size_t)blockIdx.x * p.Tp * BM
                          : p.partial + ((size_t)(2 * c + (u == u0 ? 0 : 1)) * 2 + rank) * T * BM;
        for (int c0 = gid * 32; c0 < T; c0 += 64) {
          uint32_t r[32];
          tmem_ld32_async(t_row + (uint32_t)c0, r);
          tmem_ld_wait();
#pragma unroll
          for (int cc = 0; cc < 32; ++cc)
            if (c0 + cc < T) dst[(size_t)(c0 + cc) * BM + m] = __uint_as_float(r[cc]);
        }
        if (tail) {
          // (the CTA barrier orders every thread's stores before the lead's cumulative release; a
          // per-thread __threadfence -- MEMBAR.SC.GPU -- would wait for this SM's in-flight TMA loads)
          named_sync(1, 256);
          if (lead) st_release(&p.flags[blockIdx.x], 1);
        }
        return;
      }
      // head or full tile: the other groups' k segments of this tile, in k order, then the output
      int c_lo = c + 1, c_hi = c;
      if (is_head) c_hi = sk_group_of((int)(te - 1), P.G, P.n_tiles, kb, P.drain);
      if (is_head && !pre_fix) {
        if (lead)
          for (int cc = c_lo; cc <= c_hi; ++cc)
            while (ld_acquire(&p.flags[cc * 2 + (int)rank]) == 0) __nanosleep(64);
        named_sync(1, 256);
      }
      for (int c0 = gid * 32; c0 < T; c0 += 64) {
        uint32_t r[32];
        tmem_ld32_async(t_row + (uint32_t)c0, r);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = __uint_as_float(r[q]);
        if (pre_fix) {  // fixed k order
#pragma unroll
          for (int q = 0; q < kPreT; ++q) v[q] += pf1[q];
          if (c_hi - c_lo + 1 == 2) {
#pragma unroll
            for (int q = 0; q < kPreT; ++q) v[q] += pf2[q];
          }
        } else {
          for (int cc = c_lo; cc <= c_hi; cc += 2) {  // fixed k order; two segments' loads in flight
            const float* s0 = p.partial + (size_t)(cc * 2 + (int)rank) * p.Tp * BM + m;
            const bool two = cc + 1 <= c_hi;
            const float* s1 = s0 + (two ? (size_t)2 * p.Tp * BM : 0);
            float a0[32], a1[32];
#pragma unroll
            for (int q = 0; q < 32; ++q) a0[q] = (c0 + q < T) ? __ldcg(&s0[(size_t)(c0 + q) * BM]) : 0.f;
            if (two) {
#pragma unroll
              for (int q = 0; q < 32; ++q) a1[q] = (c0 + q < T) ? __ldcg(&s1[(size_t)(c0 + q) * BM]) : 0.f;
            }
#pragma unroll
            for (int q = 0; q < 32; ++q) v[q] += a0[q];
            if (two) {
#pragma unroll
              for (int q = 0; q < 32; ++q) v[q] += a1[q];
            }
          }
        }
        direct_store(P, v, c0, min(32, T - c0), vt);
      }
      if (is_head) {
        named_sync(1, 256);
        if (lead)
          for (int cc = c_lo; cc <= c_hi; ++cc) p.flags[cc * 2 + (int)rank] = 0;  // re-arm
      }
    };

    // residual + partial sum + RMSNorm of row r: resid_norm_kernel's arithmetic and reduction tree. The
    // row kernel's virtual thread vt (d / 4 NG of them, 32-lane virtual warps vw) is lane vt % 32 of warp
    // vw % 8 of the quarter task vw / 8; the quarter tasks of a row run on different CTAs (one load
    // round trip each), publish their virtual warps' sums, and each replays the row kernel's final
    // 32-value warp reduction on the published sums (the same values in the same order -> same bits)
    auto rn_task = [&](const SeqPhase& P, int pi_rn, int r, int qq) {
      const int d = P.d, NG = rn_ng_dev(d), nthr = d / (4 * NG), nvw = nthr >> 5, nq = (nvw + 7) / 8;
      const int vw = qq * 8 + ew;
      const bool act = vw < nvw;  // (warp-uniform)
      float4 x[2];
      if (act) {
        const int vt = vw * 32 + lane;
        float ss = 0.f;
        for (int j = 0; j < NG; ++j) {
          const int i = 4 * vt + 4 * nthr * j;
          float4 xx = *reinterpret_cast<const float4*>(P.resid + (size_t)r * d + i);
          const int tile = i / BM, mm = i % BM;
          const int ns = seg_n[tile];
          const int* so = seg_off + tile * kRnMaxSeg;
          const float* bp = p.partial + (size_t)r * BM + mm;
          for (int q0 = 0; q0 < ns; q0 += 8) {  // k order; eight loads in flight
            float4 pv[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (q0 + q < ns) pv[q] = __ldcg(reinterpret_cast<const float4*>(bp + so[q0 + q]));
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (q0 + q < ns) {
                xx.x += pv[q].x;
                xx.y += pv[q].y;
                xx.z += pv[q].z;
                xx.w += pv[q].w;
              }
          }
          *reinterpret_cast<float4*>(P.out + (size_t)r * d + i) = xx;
          if (P.tap) *reinterpret_cast<float4*>(P.tap + (size_t)r * d + i) = xx;
          ss = fmaf(xx.x, xx.x, ss);
          ss = fmaf(xx.y, xx.y, ss);
          ss = fmaf(xx.z, xx.z, ss);
          ss = fmaf(xx.w, xx.w, ss);
          x[j & 1] = xx;
        }
        ss = warp_sum(ss);
        if (lane == 0) seq_ss(p.sync, pi_rn, r)[vw] = ss;
      }
      named_sync(1, 256);
      if (lead) st_release(seq_rowflag(p.sync, pi_rn, r, qq), E1);
      if (!P.gamma) return;
      if (lead)
        for (int q2 = 0; q2 < nq; ++q2)
          while (ld_acquire(seq_rowflag(p.sync, pi_rn, r, q2)) < E1) __nanosleep(32);
      named_sync(1, 256);
      if (ew == 0) {
        float v = (lane < nvw) ? __ldcg(seq_ss(p.sync, pi_rn, r) + lane) : 0.f;
        v = warp_sum(v);
        if (lane == 0) red[32] = v;
      }
      named_sync(1, 256);
      const float rs = 1.0f / sqrtf(red[32] / (float)d + P.eps);
      if (act) {
        const int vt = vw * 32 + lane;
        for (int j = 0; j < NG; ++j) {
          const int i = 4 * vt + 4 * nthr * j;
          const float4 xx = x[j & 1];
          const float4 gg = *reinterpret_cast<const float4*>(P.gamma + i);
          __nv_bfloat162 lo = __floats2bfloat162_rn(xx.x * rs * gg.x, xx.y * rs * gg.y);
          __nv_bfloat162 hi = __floats2bfloat162_rn(xx.z * rs * gg.z, xx.w * rs * gg.w);
          uint2 pk;
          pk.x = *reinterpret_cast<uint32_t*>(&lo);
          pk.y = *reinterpret_cast<uint32_t*>(&hi);
          *reinterpret_cast<uint2*>(P.xn + (size_t)r * d + i) = pk;
        }
      }
      named_sync(1, 256);  // red is reused by the next task
    };

    int gseg = 0;
    for (int pi = 0; pi < p.n_phases; ++pi) {
      const SeqPhase& P = p.ph[pi];
      const unsigned long long kt0 = lead ? kt_now() : 0ull;  // (timeline items: tools/ktrace.py)
      unsigned long long ktw = kt0;
      if (P.kind == SEQ_GEMM) {
        long long u0, u1;
        if (prange(pi, u0, u1)) {
          const int kb = P.kb;
          for (long long lo = u0; lo < u1; ++gseg) {
            const long long hi = min(u1, (lo / kb + 1) * kb);
            const int t = (int)(lo / kb);
            const int b = gseg % p.nbuf;
            if (P.mode == EPI_QKV_ROPE && lo == (long long)t * kb && gid * 32 < T)
              rope_prefetch(P.epi.rope, gid * 32, t * 2 + (int)rank);
            // small T, a head piece with one or two partner segments: wait for the partners' flags
            // and load their partials now, off the critical path after the last MMA
            pre_fix = false;
            if (P.mode != EPI_PARTIAL && T <= kPreT && lo == (long long)t * kb && hi < (long long)(t + 1) * kb) {
              const int c_hi = sk_group_of(t * kb + kb - 1, P.G, P.n_tiles, kb, P.drain);
              const int n_o = c_hi - c;
              if (n_o >= 1 && n_o <= 2) {
                // one thread polls, with back-off (a partner publishes its tail piece only once its
                // own epilogue reaches this phase; 256 spinning threads per CTA would load the L2)
                if (lead)
                  for (int cc = c + 1; cc <= c_hi; ++cc)
                    while (ld_acquire(&p.flags[cc * 2 + (int)rank]) == 0) __nanosleep(128);
                named_sync(1, 256);
                if (gid == 0) {
                  const float* s0 = p.partial + (size_t)((c + 1) * 2 + (int)rank) * p.Tp * BM + m;
                  const float* s1 = s0 + (size_t)2 * p.Tp * BM;
#pragma unroll
                  for (int q = 0; q < kPreT; ++q) pf1[q] = q < T ? __ldcg(&s0[(size_t)q * BM]) : 0.f;
                  if (n_o == 2) {
#pragma unroll
                    for (int q = 0; q < kPreT; ++q) pf2[q] = q < T ? __ldcg(&s1[(size_t)q * BM]) : 0.f;
                  }
                }
                pre_fix = true;
              }
            }
            const unsigned long long ks0 = lead ? kt_now() : 0ull;
            mbar_wait_sleep(&accf[b], (uint32_t)(gseg / p.nbuf) & 1u);
            tc_fence_after();
            const unsigned long long ks1 = lead ? kt_now() : 0ull;
            segment_epilogue(P, pi, lo, t, hi, b, u0);
            if (lead)
              kt_item(0x100000u | ((uint32_t)pi << 8) | (uint32_t)((lo == (long long)t * kb ? 1 : 0) | (hi == (long long)(t + 1) * kb ? 2 : 0)),
                      ks0, ks1, kt_now());
            tc_fence_before();
            named_sync(1, 256);
            if (lead && gseg < total_segs - 1) {  // (the MMA never waits for the last buffer)
              if (prank == 0) mbar_arrive(&acce[b]);
              else mbar_arrive_remote(&acce[b], pbase);
            }
            lo = hi;
          }
        }
      } else {
        // consumer phase: once every CTA has published the producing GEMM's partials
        if (lead)
          while (ld_acquire(seq_done(p.sync, pi - 1)) < E1 * (int)gridDim.x) __nanosleep(64);
        // the producing GEMM's k-segment table per 128-column tile (launch_resid_norm's)
        {
          const int n128 = P.pntiles * 2;
          for (int vt = threadIdx.x - 128; vt < n128; vt += 256) {
            const int ns = pseg_count(vt, P.pG, P.pntiles, P.pkb, P.pdrain, 2);
            seg_n[vt] = ns;
            for (int q = 0; q < ns && q < kRnMaxSeg; ++q)
              seg_off[vt * kRnMaxSeg + q] = (int)pseg_off(vt, q, P.pG, P.pntiles, P.pkb, P.pdrain, 2, P.Tslot);
          }
        }
        named_sync(1, 256);
        if (lead) ktw = kt_now();
        if (P.kind == SEQ_RESID_NORM) {
          const int d = P.d, nq = (d / (4 * rn_ng_dev(d)) / 32 + 7) / 8;
          for (int tau = blockIdx.x; tau < T * nq; tau += gridDim.x) rn_task(P, pi, tau / nq, tau % nq);
        } else {
          const RopeEpi& R = P.epi.rope;
          const int H = R.Hq + 2 * R.Hkv;
          for (int it = blockIdx.x * 8 + ew; it < T * H; it += gridDim.x * 8) {
            const int t = it / H, h = it % H;
            const int* so = seg_off + h * kRnMaxSeg;
            rope_partial_item(p.partial, t, h, seg_n[h], [&](int q) { return (size_t)so[q]; }, R.q_len, R.pos0, R.table,
                              R.Hq, R.Hkv, R.bt, R.pps, reinterpret_cast<__nv_bfloat16*>(R.Kp),
                              reinterpret_cast<__nv_bfloat16*>(R.Vp), reinterpret_cast<__nv_bfloat16*>(R.q_out));
          }
        }
        named_sync(1, 256);  // (the table is rebuilt by the next consumer phase)
      }
      // this CTA's part of phase pi is in memory (barrier, then the lead's cumulative release)
      named_sync(1, 256);
      if (lead) {
        red_release_add(seq_done(p.sync, pi), 1);
        kt_item(0x800000u | ((uint32_t)pi << 8) | (uint32_t)(blockIdx.x & 0xFF), kt0, ktw, kt_now());
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {  // the last CTA out advances the epoch (every CTA has read it by now)
    const int E1x = *reinterpret_cast<volatile int*>(p.sync) + 1;
    int prev;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(prev) : "l"(p.sync + 1) : "memory");
    if (prev == E1x * (int)gridDim.x - 1) st_release(p.sync, E1x);
  }
  cluster_sync();
  tc_fence_after();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols) : "memory");
}

// ------------------------------------------------------------------------ host side
bool gemm_seq_supported(int T, const SeqStep* st, int n) {
  if (T < 1 || T > 128 || n < 1 || n > kSeqMaxPhases) return false;
  int n_gemm = 0, prev_mode = -1, prevN = 0;
  for (int i = 0; i < n; ++i) {
    const SeqStep& s = st[i];
    if (s.kind == SEQ_GEMM) {
      if (++n_gemm > kSeqMaxGemm) return false;
      if (s.N % (2 * BM) || s.K % BK || gemm_cg(s.N, s.K) != 2) return false;
      if (s.epi.mode != EPI_PARTIAL && s.epi.mode != EPI_SWIGLU_ACT && s.epi.mode != EPI_QKV_ROPE) return false;
      const int n_tiles = s.N / (2 * BM), kb = s.K / BK;
      const int G = sk_groups(2, n_tiles, kb);
      const int drain = s.epi.drain >= 0 ? s.epi.drain : sk_drain(s.epi.mode);
      if (!sk_fits(G, n_tiles, kb, drain)) return false;
      if (s.epi.mode == EPI_PARTIAL && n_tiles > G) return false;
      prev_mode = s.epi.mode;
      prevN = s.N;
    } else {
      if (i == 0 || prev_mode != EPI_PARTIAL) return false;  // a consumer of the preceding EPI_PARTIAL GEMM
      {
        const int n_tiles = prevN / (2 * BM), G = sk_groups(2, n_tiles, st[i - 1].K / BK);
        if ((G + n_tiles - 1) / n_tiles + 1 > kRnMaxSeg || 2 * n_tiles > kRnMaxTiles) return false;
      }
      if (s.kind == SEQ_RESID_NORM && (s.d != prevN || !rn_ng(s.d) || rn_ng(s.d) > 2)) return false;
      if (s.kind == SEQ_ROPE && prevN != (s.epi.rope.Hq + 2 * s.epi.rope.Hkv) * BM) return false;
      if (s.kind != SEQ_RESID_NORM && s.kind != SEQ_ROPE) return false;
      prev_mode = -1;
    }
  }
  return true;
}

cudaError_t gemm_seq_launch(int T, const SeqStep* st, int n, const GemmScratch& scratch, int* sync, cudaStream_t stream) {
  if (!gemm_seq_supported(T, st, n) || !ensure_encode() || !sync) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_seq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  SeqParams p{};
  SeqMaps maps;
  memset(&maps, 0, sizeof(maps));
  int n_sub = 1;
  tc_shape(T, &p.NT, &n_sub);
  if (n_sub != 1) return cudaErrorInvalidValue;
  p.T = T;
  p.Tp = (T + 31) / 32 * 32;
  p.nbuf = (2 * p.NT <= 512) ? 2 : 1;
  p.tmem_cols = 32;
  while ((int)p.tmem_cols < p.nbuf * p.NT) p.tmem_cols <<= 1;
  const int stage_bytes = BM * BK * 2 + (p.NT / 2) * BK * 2;
  p.stages = std::max(2, std::min(16, (205 * 1024) / stage_bytes));
  p.cgrp = 1;
  for (int cg = 8; cg >= 2; cg >>= 1)
    if (cg * 3 <= p.stages || (cg * 2 <= p.stages && cg == 2)) {
      p.cgrp = cg;
      break;
    }
  p.stages = (p.stages / p.cgrp) * p.cgrp;
  static const int env_npre = getenv("SF_GEMM_NPRE") ? atoi(getenv("SF_GEMM_NPRE")) : 4;
  p.npre = std::max(1, std::min(env_npre, p.stages));
  p.partial = scratch.partial;
  p.flags = scratch.counters;
  p.sync = sync;
  p.n_phases = n;
  const int Gmax = max_groups(2);
  if (!scratch.partial || scratch.partial_elems < (int64_t)2 * Gmax * 2 * p.Tp * BM || scratch.n_counters < Gmax * 2)
    return cudaErrorInvalidValue;
  int nm = 0;
  for (int i = 0; i < n; ++i) {
    const SeqStep& s = st[i];
    SeqPhase& P = p.ph[i];
    P.kind = s.kind;
    P.epi = s.epi;
    if (s.kind == SEQ_GEMM) {
      P.mode = s.epi.mode;
      P.kb = s.K / BK;
      P.n_tiles = s.N / (2 * BM);
      P.G = sk_groups(2, P.n_tiles, P.kb);
      P.drain = s.epi.drain >= 0 ? s.epi.drain : sk_drain(s.epi.mode);
      P.map = nm;
      if (!make_map_tiled(&maps.w[nm], s.W, (long long)s.N * P.kb) || !make_map(&maps.a[nm], s.A, T, s.K, s.lda, p.NT / 2))
        return cudaErrorInvalidValue;
      ++nm;
    } else {
      const SeqPhase& G = p.ph[i - 1];
      P.pG = G.G;
      P.pkb = G.kb;
      P.pdrain = G.drain;
      P.pntiles = G.n_tiles;
      P.Tslot = T;
      P.resid = s.resid;
      P.out = s.out;
      P.tap = s.tap;
      P.gamma = s.gamma;
      P.xn = s.xn;
      P.d = s.d;
      P.eps = s.eps;
    }
  }
  const size_t smem = (size_t)p.stages * stage_bytes + 1024 + (2 * p.stages + 4) * 8 + 16 + 36 * 4 +
                      (size_t)kRnMaxTiles * (1 + kRnMaxSeg) * 4;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * Gmax);
  cfg.blockDim = dim3(384);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 2;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, gemm_seq_kernel, maps, p);
}
