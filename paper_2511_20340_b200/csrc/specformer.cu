// specformer.cu -- runtime behind the C ABI (include/specformer.h): config validation, packed
// weight table, workspace carving, the per-step launch sequences (draft / verify / accept), the
// chunked prefill, CUDA-graph capture of the decode step and the test hooks.
//
// Step structure (PAPER P20-23):
//   draft_step  : [context layer L+1 over the previous verify's k+1 rows (Eq.8) -> gather row
//                  r_b] -> positional FFN (Eq.9) -> draft bidirectional layer (Eq.10) -> final
//                  norm + LM head (shared, C8) -> argmax -> k draft tokens
//   verify_step : base forward over [last, d_1..d_k] (taps HS[0, L/2, L-1, L] kept) -> LM head
//                  -> argmax -> greedy[k+1]
//   accept      : m = longest matching prefix, commit seq_len += m + 1 (rollback moves no data)
#include <condition_variable>
#include <mutex>
#ifdef SF_WITH_NCCL
#include <nccl.h>
#endif
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/specformer.h"
#include "gemm.cuh"
#include "kernels.cuh"

using namespace sf;

namespace {

constexpr int64_t kAlign = 256;
inline int64_t align_up(int64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct TensorSpec {
  std::string name;
  std::vector<int64_t> shape;
  bool matrix;  // stored in config dtype (else fp32)
};

bool valid_config(const sf_config* c, std::string* why) {
  auto fail = [&](const char* m) {
    if (why) *why = m;
    return false;
  };
  if (!c) return fail("null config");
  if (c->n_layers < 1 || c->d_model < 1 || c->n_heads < 1 || c->n_kv_heads < 1 || c->head_dim < 2 ||
      c->d_ff < 1 || c->vocab < 2)
    return fail("nonpositive dimension");
  if (c->n_heads % c->n_kv_heads) return fail("n_heads % n_kv_heads != 0");
  if (c->head_dim != 16 && c->head_dim != 64 && c->head_dim != 128) return fail("head_dim must be 16, 64 or 128");
  if (c->draft_len < 0 || c->draft_len > 16) return fail("draft_len must be in [0, 16]");
  if (c->draft_blocks < 0 || c->draft_blocks > 4) return fail("draft_blocks must be in [0, 4]");
  if (c->max_batch < 1 || c->max_batch > 1024) return fail("max_batch must be in [1, 1024]");
  if (c->kv_block != 16) return fail("kv_block must be 16");
  if (c->max_seq < 16 || c->max_seq % 16) return fail("max_seq must be a positive multiple of 16");
  // (bf16 flash-decoding attention: a row folds at most 64 key segments of kAttnSeg keys)
  if (c->dtype == SF_BF16 && c->head_dim == 128 && c->max_seq > 64 * kAttnSeg) return fail("max_seq must be <= 131072");
  if (!(c->rms_eps > 0.f)) return fail("rms_eps must be > 0");
  if (!(c->rope_theta > 0.f)) return fail("rope_theta must be > 0");
  if (c->dtype != SF_FP32 && c->dtype != SF_BF16) return fail("dtype must be SF_FP32 or SF_BF16");
  if (c->tp_size < 1 || c->tp_rank < 0 || c->tp_rank >= c->tp_size) return fail("need 0 <= tp_rank < tp_size");
  if (c->tp_size > 1) {  // Megatron TP: heads / FFN / vocab / W_D input split over the ranks
    const int tp = c->tp_size;
    if (c->dtype != SF_BF16) return fail("tensor parallelism needs the bf16 path");
    if (c->n_heads % tp || c->n_kv_heads % tp) return fail("n_heads and n_kv_heads must divide by tp_size");
    if (c->d_ff % (64 * tp)) return fail("d_ff must be a multiple of 64 tp_size");
    if ((4 * c->d_model) % (64 * tp)) return fail("4 d_model must be a multiple of 64 tp_size");
    if (c->vocab % 128 || c->vocab / 128 < tp) return fail("vocab must be a multiple of 128 with >= tp_size tiles");
  }
  if (c->d_ff % 64) return fail("d_ff must be a multiple of 64 (interleaved gate/up groups)");
  if (c->pool_pages < 0) return fail("pool_pages must be >= 0");
  if (c->tp_size > 1 && (c->flags & (SF_FLAG_NO_POS_FFN | SF_FLAG_DRAFT_PREFIX)))
    return fail("the -Pos / BIDIR_PREFIX draft variants are single-GPU");
  if (c->dtype == SF_BF16) {
    const int qkv = (c->n_heads + 2 * c->n_kv_heads) * c->head_dim;
    if (c->d_model % 128 || qkv % 128 || (2 * c->d_ff) % 128 || c->vocab % 128 ||
        (c->n_heads * c->head_dim) % 64 || c->d_ff % 64)
      return fail("bf16 path needs d, qkv width, 2F, V multiples of 128 and K multiples of 64");
  }
  return true;
}

// Tensor-parallel rank r of tp: q / kv heads [r H/tp, (r+1) H/tp), FFN rows [r F/tp, ..), the LM head's
// vocabulary rows [v0, v1) (whole 128-row tiles, as even as possible), W_D's input columns
// [r 4d/tp, ..). tp = 1: everything.
static int tp_of(const sf_config* c) { return c->tp_size > 1 ? c->tp_size : 1; }
static void vocab_shard(const sf_config* c, int* v0, int* v1) {
  const int tp = tp_of(c), r = tp > 1 ? c->tp_rank : 0, tiles = c->vocab / 128;
  if (tp == 1) {
    *v0 = 0;
    *v1 = c->vocab;
    return;
  }
  *v0 = (int)((int64_t)tiles * r / tp) * 128;
  *v1 = (int)((int64_t)tiles * (r + 1) / tp) * 128;
}

// draft bidirectional blocks (Eq.10 has one; NEXT-2 "+Larger" stacks more): 0 reads as 1
static int draft_blocks(const sf_config* c) { return c->draft_blocks > 1 ? c->draft_blocks : 1; }

std::vector<TensorSpec> tensor_specs(const sf_config* c) {
  const int tp = tp_of(c);
  int v0, v1;
  vocab_shard(c, &v0, &v1);
  const int64_t d = c->d_model, F = c->d_ff / tp, V = c->vocab, Vl = v1 - v0, k = c->draft_len;
  const int64_t qkv = (int64_t)(c->n_heads + 2 * c->n_kv_heads) / tp * c->head_dim,
                ao = (int64_t)c->n_heads / tp * c->head_dim;
  std::vector<TensorSpec> t;
  t.push_back({"embed", {V, d}, true});
  for (int l = 0; l < c->n_layers; ++l) {
    const std::string p = "layers." + std::to_string(l) + ".";
    t.push_back({p + "attn_norm", {d}, false});
    t.push_back({p + "wqkv", {qkv, d}, true});
    t.push_back({p + "wo", {d, ao}, true});
    t.push_back({p + "ffn_norm", {d}, false});
    t.push_back({p + "w_gu", {2 * F, d}, true});
    t.push_back({p + "w_down", {d, F}, true});
  }
  t.push_back({"final_norm", {d}, false});
  t.push_back({"lm_head", {Vl, d}, true});
  if (k > 0) {
    t.push_back({"sf.group_scale", {4, d}, false});
    t.push_back({"sf.w_d", {d, 4 * d / tp}, true});
    t.push_back({"sf.ctx_norm", {d}, false});
    t.push_back({"sf.ctx_wqkv", {qkv, d}, true});
    t.push_back({"sf.ctx_wo", {d, ao}, true});
    t.push_back({"sf.pos_norm", {d}, false});
    if (!(c->flags & SF_FLAG_NO_POS_FFN)) t.push_back({"sf.w_p", {k * d, d}, true});
    t.push_back({"sf.b_p", {k * d}, false});
    for (int i = 0; i < draft_blocks(c); ++i) {  // block 0: "sf.blk_*", block i > 0: "sf.blk<i>_*"
      const std::string b = i == 0 ? "sf.blk_" : "sf.blk" + std::to_string(i) + "_";
      t.push_back({b + "attn_norm", {d}, false});
      t.push_back({b + "wqkv", {qkv, d}, true});
      t.push_back({b + "wo", {d, ao}, true});
      t.push_back({b + "ffn_norm", {d}, false});
      t.push_back({b + "w_gu", {2 * F, d}, true});
      t.push_back({b + "w_down", {d, F}, true});
    }
  }
  return t;
}

int64_t tensor_bytes(const sf_config* c, const TensorSpec& s) {
  int64_t n = 1;
  for (auto v : s.shape) n *= v;
  return n * ((s.matrix && c->dtype == SF_BF16) ? 2 : 4);
}

// ----------------------------------------------------------------- workspace plan
struct Plan {
  int B, k, d, Hq, Hkv, hd, F, V, L, qkvw, ao;  // Hq, Hkv, F, V: this rank's share (tensor parallelism)
  int tp, tp_rank, V_full, v0, wd_k;            // ranks, full vocabulary, vocab shard offset, W_D input width
  int pps, n_pages, nchunk, rows_v, rows_d, C_pf, rows_pf, R;
  bool pool;  // SF_FLAG_PAGE_POOL: pages from a device-side free-page stack
  int64_t act, kv_layer_bytes;
  // offsets
  int64_t o_k, o_v, o_bt, o_rope, o_resid, o_xn, o_qkv, o_qrot, o_attn, o_ffn, o_taps, o_ctx, o_idrow, o_D,
      o_hlast, o_logits, o_dlogits, o_apo, o_apml, o_gpart, o_gcnt, o_amv, o_ami, o_ints, o_prompt, o_acnt,
      o_tpbuf, o_tpbf, o_tpkey, o_seqsync, o_pool;
  int64_t n_acnt;
  int64_t gpart_elems, n_amrows;
  int64_t total;
};

Plan make_plan(const sf_config* c) {
  Plan p{};
  p.B = c->max_batch;
  p.k = c->draft_len;
  p.d = c->d_model;
  p.tp = tp_of(c);
  p.tp_rank = p.tp > 1 ? c->tp_rank : 0;
  p.Hq = c->n_heads / p.tp;
  p.Hkv = c->n_kv_heads / p.tp;
  p.hd = c->head_dim;
  p.F = c->d_ff / p.tp;
  int v1 = 0;
  vocab_shard(c, &p.v0, &v1);
  p.V = v1 - p.v0;
  p.V_full = c->vocab;
  p.wd_k = 4 * c->d_model / p.tp;
  p.L = c->n_layers;
  p.qkvw = (p.Hq + 2 * p.Hkv) * p.hd;
  p.ao = p.Hq * p.hd;
  p.act = c->dtype == SF_BF16 ? 2 : 4;
  p.pps = c->max_seq / 16;
  p.pool = (c->flags & SF_FLAG_PAGE_POOL) != 0;
  p.n_pages = (p.pool && c->pool_pages > 0) ? c->pool_pages : p.B * p.pps;
  p.nchunk = (c->max_seq + kAttnChunk - 1) / kAttnChunk;
  p.rows_v = p.B * (p.k + 1);
  p.rows_d = std::max(1, p.B * p.k);
  // prefill chunk: rows per sequence such that a chunk is one 512-row GEMM pass (the weights are
  // streamed once per chunk; 512 = the TMEM accumulator width)
  static const int pf_cap = getenv("SF_PF_CAP") ? atoi(getenv("SF_PF_CAP")) : 512;
  p.C_pf = std::max(p.k + 1, std::min(pf_cap, std::max(1, 512 / p.B)));
  p.rows_pf = p.B * p.C_pf;
  p.R = std::max(p.rows_v, p.rows_pf);
  p.kv_layer_bytes = (int64_t)p.n_pages * p.Hkv * 16 * p.hd * p.act;
  // split-K partial scratch: worst case over every GEMM shape at R rows
  const bool bf = c->dtype == SF_BF16;
  const int shapes[][2] = {{p.qkvw, p.d}, {p.d, p.ao}, {2 * p.F, p.d}, {p.d, p.F}, {p.V, p.d},
                           {p.d, p.wd_k}, {std::max(1, p.k) * p.d, p.d}};
  p.gpart_elems = 0;
  for (auto& s : shapes) p.gpart_elems = std::max<int64_t>(p.gpart_elems, gemm_partial_elems(bf, std::min(p.R, 512), s[0], s[1]));
  if (bf) p.gpart_elems = std::max<int64_t>(p.gpart_elems, gemm_chain_partial_elems(std::min(p.R, 512)));
  p.n_amrows = std::max(p.rows_v, std::max(p.rows_d, p.B));
  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    const int64_t r = o;
    o += align_up(std::max<int64_t>(bytes, 1));
    return r;
  };
  p.o_k = take(p.kv_layer_bytes * (p.L + 1));
  p.o_v = take(p.kv_layer_bytes * (p.L + 1));
  p.o_bt = take((int64_t)p.B * p.pps * 4);
  p.o_pool = take((int64_t)(p.n_pages + p.B + 8) * 4);  // free-page stack, per-sequence page counts, stack top
  p.o_rope = take((int64_t)c->max_seq * (p.hd / 2) * 8);
  p.o_resid = take((int64_t)p.R * p.d * 4);
  p.o_xn = take((int64_t)p.R * 4 * p.d * p.act);
  p.o_qkv = take((int64_t)p.R * p.qkvw * p.act);
  p.o_qrot = take((int64_t)p.R * p.ao * 4);
  p.o_attn = take((int64_t)p.R * p.ao * p.act);
  p.o_ffn = take((int64_t)p.R * p.F * p.act);
  p.o_taps = take((int64_t)4 * p.R * p.d * 4);
  p.o_ctx = take((int64_t)p.R * p.d * 4);
  p.o_idrow = take((int64_t)p.B * p.d * 4);
  p.o_D = take((int64_t)p.rows_d * p.d * 4);
  p.o_hlast = take((int64_t)p.B * p.d * 4);
  p.o_logits = take((int64_t)p.rows_v * p.V * 4);
  p.o_dlogits = take((int64_t)p.rows_d * p.V * 4);
  p.o_apo = take((int64_t)p.R * p.Hq * p.nchunk * kAttnWarps * p.hd * 4);
  p.o_apml = take((int64_t)p.R * p.Hq * p.nchunk * kAttnWarps * 2 * 4);
  // split-KV arrival counters: one per (sequence, kv head, query tile) at the longest block
  constexpr int TR = kAttnTileRows;
  p.n_acnt = std::max<int64_t>((int64_t)p.B * p.Hkv * ((std::max(p.k + 1, p.C_pf) * (p.Hq / p.Hkv) + TR - 1) / TR),
                               (int64_t)p.Hkv * ((p.R * (p.Hq / p.Hkv) + TR - 1) / TR + 1));  // (one long sequence)
  p.o_acnt = take(p.n_acnt * 4);
  p.o_gpart = take(p.gpart_elems * 4);
  p.o_gcnt = take(4096 * 4);
  p.o_amv = take(p.n_amrows * argmax_splits(p.V) * 4);
  p.o_ami = take(p.n_amrows * argmax_splits(p.V) * 4);
  p.o_ints = take((int64_t)(16 * p.B + 2 * p.R + 8 + p.rows_v * 2 + p.rows_d) * 4);
  p.o_prompt = take((int64_t)p.B * c->max_seq * 4);
  p.o_tpbuf = p.tp > 1 ? take((int64_t)p.R * p.d * 4) : 0;   // row-parallel GEMM output, all-reduced
  p.o_tpbf = p.tp > 1 ? take((int64_t)p.R * p.d * 2) : 0;     // its bf16 form (the default all-reduce)
  p.o_tpkey = bf ? take(p.n_amrows * 8) : 0;  // packed (logit, id) argmax keys (fused LM-head argmax; TP max-reduces them)
  p.o_seqsync = bf ? take((int64_t)p.L * kSeqSyncInts * 4) : 0;  // layer-sequence launches' sync blocks (zeroed)
  p.total = o;
  return p;
}

enum State { ST_INIT = 0, ST_READY = 1, ST_DRAFTED = 2, ST_VERIFIED = 3 };

}  // namespace

struct sf_handle {
  sf_config c{};
  Plan p{};
  bool bf = false;
  cudaStream_t st = nullptr;
  char* W = nullptr;
  char* ws = nullptr;
  // weights
  struct Lw {
    const float *attn_norm, *ffn_norm;
    const void *wqkv, *wo, *wgu, *wdown;
  };
  std::vector<Lw> lw;
  const void *embed = nullptr, *lm_head = nullptr;
  const float* final_norm = nullptr;
  const float *group_scale = nullptr, *ctx_norm = nullptr, *pos_norm = nullptr, *b_p = nullptr,
              *blk_attn_norm = nullptr, *blk_ffn_norm = nullptr;
  const void *w_d = nullptr, *ctx_wqkv = nullptr, *ctx_wo = nullptr, *w_p = nullptr, *blk_wqkv = nullptr,
             *blk_wo = nullptr, *blk_wgu = nullptr, *blk_wdown = nullptr;
  struct Blk {
    const float *attn_norm, *ffn_norm;
    const void *wqkv, *wo, *wgu, *wdown;
  };
  std::vector<Blk> blks;  // the draft blocks in order (blks[0] = the blk_* pointers above)
  // workspace views
  char *kpool = nullptr, *vpool = nullptr;
  int* bt = nullptr;
  float2* rope = nullptr;
  float *resid, *qrot, *taps, *ctx, *idrow, *D, *hlast, *logits, *dlogits, *apo, *apml, *gpart, *amv;
  void *xn, *qkv, *attn, *ffn;
  int *gcnt, *ami, *acnt;
  int* seqsync = nullptr;  // [L][kSeqSyncInts] (layer_seq)
  PagePool pp;                 // NEXT-4 page pool (null pointers: static per-sequence page ranges)
  std::vector<char> released;  // slots released and not yet re-filled (page pool)
  // tensor parallelism: row-parallel GEMM output / argmax keys, and the collective that reduces them
  float* tpbuf = nullptr;
  __nv_bfloat16* tpbf = nullptr;  // the bf16 copy that is all-reduced (unless SF_FLAG_TP_F32_REDUCE)
  unsigned long long* tpkey = nullptr;
  struct Coll {
    cudaError_t (*sum_f32)(void* ctx, float* buf, int64_t n, cudaStream_t s) = nullptr;
    cudaError_t (*sum_bf16)(void* ctx, __nv_bfloat16* buf, int64_t n, cudaStream_t s) = nullptr;
    cudaError_t (*max_u64)(void* ctx, unsigned long long* buf, int64_t n, cudaStream_t s) = nullptr;
    void* ctx = nullptr;
    bool graph_safe = false;  // only device work is enqueued (NCCL): decode_steps may capture it
  } coll;
  void* nccl_comm = nullptr;
  // NEXT-3 fused TP all-reduce over peer memory: this rank's exchange region ([0, 128) the epochs the
  // peers published into it, [128] this rank's epoch counter, [256 ..) two bf16 [R, d] slots), the
  // peers' regions (mapped through CUDA IPC, or direct pointers in a local group), mode 0 off / 1 IPC /
  // 2 local group (eager: a host barrier after every signal, so no kernel waits on another rank's)
  char* xch = nullptr;
  size_t xch_bytes = 0;
  char* xpeer[kTpMax] = {};
  bool xopened[kTpMax] = {};
  int xmode = 0;
  void* xgroup = nullptr;  // (mode 2) the sf_local_group
  int *tok_rows, *pos0_pf, *seq_len, *n_prev, *last_token, *r_b, *prompt_len, *draft, *greedy, *accept_len,
      *emitted, *err, *step_counter, *g_pf, *prompt, *d_logcap;
  // state
  int B = 0;
  int state = ST_INIT;
  bool ctx_pending = false;
  bool final_xn_ready = false;
  int fwd_rows = 0, ctx_rows = 0;  // rows of the last base forward / context-layer pass (debug capture)
  int64_t launches = 0;
  int64_t host_len_hi = 0;  // host upper bound of max(seq_len)
  std::string err_msg;
  // graph
  cudaGraphExec_t gexec = nullptr;
  int g_B = 0;  // batch size the cached step graph was captured at (its grids, T = B(k+1), accept B)
  int64_t graph_launches = 0;
  int *g_acc_log = nullptr, *g_em_log = nullptr;
  // per-kernel-class profiling (eager launches only; bench roofline)
  struct Prof {
    int cls;
    cudaEvent_t a, b;
    double bytes;
  };
  bool prof_on = false;
  bool prof_capture = false;  // records become external event-record nodes of the profiling graph
  std::vector<Prof> prof;
  double prof_ms[4] = {0, 0, 0, 0}, prof_bytes[4] = {0, 0, 0, 0};  // graph replays, accumulated
  int64_t prof_n[4] = {0, 0, 0, 0};
  std::vector<cudaEvent_t> ev_free;
  cudaEvent_t ev_get() {
    if (ev_free.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = ev_free.back();
    ev_free.pop_back();
    return e;
  }
  // GEMM weights in launch order (draft, verify): the successor of each launch is prefetched to L2
  std::vector<std::pair<const void*, size_t>> wchain;
  size_t wchain_pos = 0;
  // forced drafts (bench)
  const int *f_cont = nullptr, *f_corrupt = nullptr;
  int f_cont_len = 0, f_corrupt_steps = 0;
  bool forced = false;

  void* kp(int layer) { return kpool + (size_t)layer * p.kv_layer_bytes; }
  void* vp(int layer) { return vpool + (size_t)layer * p.kv_layer_bytes; }
};

// ----------------------------------------------------------------- helpers
#define SF_TRY(expr)                                              \
  do {                                                            \
    cudaError_t e__ = (expr);                                     \
    if (e__ != cudaSuccess) {                                     \
      h->err_msg = std::string(#expr) + ": " + cudaGetErrorString(e__); \
      return SF_ERR_CUDA;                                         \
    }                                                             \
  } while (0)

static sf_status set_err(sf_handle* h, sf_status s, const std::string& m) {
  if (h) h->err_msg = m;
  return s;
}

// Kernel classes for sf_profile_read: 0 GEMM (tcgen05 / SIMT), 1 paged attention (RoPE+append,
// partial, combine), 2 norms / embedding / gathers, 3 argmax + accept + draft attention + misc.
struct ProfScope {
  sf_handle* h;
  size_t idx = (size_t)-1;
  ProfScope(sf_handle* hh, int cls, double bytes) : h(hh) {
    if (!h->prof_on) return;
    sf_handle::Prof r{cls, h->ev_get(), h->ev_get(), bytes};
    ev_record(r.a);
    h->prof.push_back(r);
    idx = h->prof.size() - 1;
  }
  ~ProfScope() {
    if (idx != (size_t)-1) ev_record(h->prof[idx].b);
  }
  void ev_record(cudaEvent_t e) {
    if (h->prof_capture)
      cudaEventRecordWithFlags(e, h->st, cudaEventRecordExternal);
    else
      cudaEventRecord(e, h->st);
  }
};

// SF_DEBUG_SYNC=1 (debugging only): synchronise after every launch group and name the first failure
static bool dbg_on() {
  static const bool on = getenv("SF_DEBUG_SYNC") && atoi(getenv("SF_DEBUG_SYNC")) > 0;
  return on;
}
static cudaError_t dbg_sync(sf_handle* h, const char* what, cudaError_t e) {
  if (!dbg_on() || e != cudaSuccess) return e;
  cudaError_t r = cudaStreamSynchronize(h->st);
  if (r != cudaSuccess) fprintf(stderr, "SF_DEBUG_SYNC: %s failed: %s\n", what, cudaGetErrorString(r));
  return r;
}

static cudaError_t gemm(sf_handle* h, const void* A, int lda, const void* W, int T, int N, int K, GemmEpi epi) {
  const double wb = h->bf ? 2.0 : 4.0;
  const double ob = (epi.mode == EPI_STORE_ACT || epi.mode == EPI_SWIGLU_ACT) ? wb : 4.0;
  const double outc = epi.amax && !epi.out ? 2 : epi.mode == EPI_SWIGLU_ACT ? N / 2 : N;  // (fused argmax: a key)
  // algorithmic bytes: weight once + activation once + output once (+ residual read for ADD)
  ProfScope ps(h, 0, (double)N * K * wb + (double)T * K * wb + (double)T * outc * ob * (epi.mode == EPI_ADD_F32 ? 2 : 1));
  static const size_t cap = (size_t)(getenv("SF_GEMM_PF_MB") ? atof(getenv("SF_GEMM_PF_MB")) : 0.0) * (1 << 20);
  if (h->bf && !h->wchain.empty() && cap > 0) {
    // (measured: prefetching the successor's weights into L2 during the tail loses at every batch --
    // it competes with the tail's own loads -- so it is off unless SF_GEMM_PF_MB asks for it)
    const size_t n = h->wchain.size();
    for (size_t i = 0; i < n; ++i) {  // forward search from the last position: launch order is fixed
      const size_t j = (h->wchain_pos + i) % n;
      if (h->wchain[j].first == W) {
        const auto& nx = h->wchain[(j + 1) % n];
        epi.pf = nx.first;
        epi.pf_bytes = std::min(nx.second, cap);
        h->wchain_pos = j + 1;
        break;
      }
    }
  }
  GemmScratch sc;
  sc.partial = h->gpart;
  sc.partial_elems = h->p.gpart_elems;
  sc.counters = h->gcnt;
  sc.n_counters = 4096;
  h->launches += (T + 511) / 512;
  const cudaError_t e = gemm_launch(h->bf, A, lda, W, h->bf, T, N, K, epi, sc, h->st);
  if (!dbg_on()) return e;
  char nm[96];
  snprintf(nm, sizeof nm, "gemm T=%d N=%d K=%d mode=%d", T, N, K, epi.mode);
  return dbg_sync(h, nm, e);
}
static GemmEpi epi_act(void* out, int ldo) {
  GemmEpi e;
  e.mode = EPI_STORE_ACT;
  e.out = out;
  e.ldo = ldo;
  return e;
}
static GemmEpi epi_f32(void* out, int ldo) {
  GemmEpi e;
  e.mode = EPI_STORE_F32;
  e.out = out;
  e.ldo = ldo;
  return e;
}
static GemmEpi epi_add(float* out, int ldo, float* tap) {
  GemmEpi e;
  e.mode = EPI_ADD_F32;
  e.out = out;
  e.ldo = ldo;
  e.tap = tap;
  return e;
}

static cudaError_t rmsnorm(sf_handle* h, const float* in, int in_ld, const float* g, int T, void* out, int out_ld) {
  ProfScope ps(h, 2, (double)T * h->p.d * (4.0 + (h->bf ? 2.0 : 4.0)));
  h->launches++;
  return launch_rmsnorm(h->bf, in, in_ld, g, h->c.rms_eps, T, h->p.d, out, out_ld, h->st);
}

// Fused "GEMM -> residual (+bias) -> [tap] -> RMSNorm" (bf16 path): the GEMM writes its k-segment
// partials (EPI_PARTIAL) and resid_norm_kernel sums them in k order while applying the residual and
// the next norm. Returns false (nothing launched) when the shape does not allow it; callers then use
// the unfused ADD / STORE epilogue + rmsnorm. rep > 1 views each GEMM row as rep rows of d columns.
// Tensor parallelism: every rank holds the full residual stream and a K-slice of the row-parallel
// weights (O, down, W_D: row_parallel = true); its GEMM output is a partial sum over the ranks, so
// the rank writes it dense (fp32), the collective sums it over the ranks (rank order / NCCL's), and
// the consumer adds it to the residual before the norm.
static cudaError_t tp_sum(sf_handle* h, float* buf, int64_t n) {
  if (!h->coll.sum_f32) {
    h->err_msg = "tensor parallelism: no collective attached (sf_nccl_attach / sf_local_group_attach)";
    return cudaErrorNotReady;
  }
  h->launches++;
  if (!(h->c.flags & SF_FLAG_TP_F32_REDUCE)) {
    // the row-parallel partial sums travel as bf16 (half the bytes of fp32)
    cudaError_t e = launch_cvt_f32_bf16(buf, h->tpbf, n, true, h->st);
    if (e == cudaSuccess) e = h->coll.sum_bf16(h->coll.ctx, h->tpbf, n, h->st);
    if (e == cudaSuccess) e = launch_cvt_f32_bf16(buf, h->tpbf, n, false, h->st);
    h->launches += 2;
    return e;
  }
  return h->coll.sum_f32(h->coll.ctx, buf, n, h->st);
}
static cudaError_t tp_max(sf_handle* h, unsigned long long* buf, int64_t n) {
  if (!h->coll.max_u64) {
    h->err_msg = "tensor parallelism: no collective attached (sf_nccl_attach / sf_local_group_attach)";
    return cudaErrorNotReady;
  }
  h->launches++;
  return h->coll.max_u64(h->coll.ctx, buf, n, h->st);
}

static constexpr size_t kXchHead = 256;  // flags [0, 128), epoch counter at 128
static void local_xch_barrier(sf_handle* h);

static bool gemm_resid_norm(sf_handle* h, cudaError_t* err, const void* A, int lda, const void* W, int T, int N,
                            int K, int rep, const float* resid, const float* bias, float* out, float* tap,
                            const float* gamma, bool row_parallel = false) {
  if (row_parallel && h->p.tp > 1 && h->xmode && rep == 1 && N == h->p.d) {
    // NEXT-3: the GEMM stores its bf16 output straight into this rank's exchange slot of the coming
    // epoch, tp_signal publishes the epoch to every peer, and the residual + norm consumer sums the
    // ranks' slots in rank order over peer memory (the all-reduce fused into the consumer; no NCCL
    // launch, no fp32 round trip). Every rank adds the same values in the same order: same bits.
    const Plan& p = h->p;
    int* ctr = (int*)(h->xch + 128);
    GemmEpi ep = epi_act(h->xch + kXchHead, N);
    ep.out_sel = ctr;
    ep.out_sel_stride = (long long)p.R * p.d;
    if ((*err = gemm(h, A, lda, W, T, N, K, ep)) != cudaSuccess) return true;
    int* pf[kTpMax];
    for (int q = 0; q < p.tp; ++q) pf[q] = (int*)h->xpeer[q];
    h->launches += 2;
    if ((*err = launch_tp_signal(ctr, pf, p.tp, p.tp_rank, h->st)) != cudaSuccess) return true;
    if (h->xmode == 2) local_xch_barrier(h);
    TpSrc ts;
    for (int q = 0; q < p.tp; ++q) ts.slot[q] = (const __nv_bfloat16*)(h->xpeer[q] + kXchHead);
    ts.ctr = ctr;
    ts.flags = (const int*)h->xch;
    ts.err = h->err;
    ts.slot_elems = (long long)p.R * p.d;
    ts.n = p.tp;
    ts.own = p.tp_rank;
    ProfScope ps(h, 2, (double)T * N * (2.0 * p.tp + 4.0 * 2));
    *err = dbg_sync(h, "resid_norm(tp fused)", launch_resid_norm(nullptr, nullptr, T, rep, p.d, resid, nullptr, bias, out,
                                                                 tap, gamma, h->c.rms_eps,
                                                                 gamma ? (__nv_bfloat16*)h->xn : nullptr, h->st, &ts));
    return true;
  }
  if (row_parallel && h->p.tp > 1) {
    if ((*err = gemm(h, A, lda, W, T, N, K, epi_f32(h->tpbuf, N))) != cudaSuccess) return true;
    if ((*err = tp_sum(h, h->tpbuf, (int64_t)T * N)) != cudaSuccess) return true;
    ProfScope ps(h, 2, (double)T * N * 4.0 * 3);
    h->launches++;
    *err = dbg_sync(h, "resid_norm(tp)", launch_resid_norm(nullptr, nullptr, T, rep, h->p.d, resid, h->tpbuf, bias, out,
                                                          tap, gamma, h->c.rms_eps,
                                                          gamma ? (__nv_bfloat16*)h->xn : nullptr, h->st));
    return true;
  }
  if (!h->bf) return false;
  // blocks of more than 512 rows (13B k = 8 at B = 64; prefill chunks) run as balanced row chunks of
  // <= 512 (the TMEM accumulator width), each GEMM publishing its partials for its own consumer: every
  // row gets the same additions in the same order at every T (batch invariance, reading C23)
  const int n_chunks = (T + 511) / 512;
  const int chunk = n_chunks == 1 ? T : std::min(512, ((T + n_chunks - 1) / n_chunks + 15) / 16 * 16);
  if (!resid_norm_supported(h->p.d, chunk, N, K)) return false;
  PartialGeom g;
  if (!gemm_partial_geom(chunk, N, K, &g)) return false;
  const int64_t rd = (int64_t)rep * h->p.d;  // elements of one GEMM row in the [T rep, d] views
  for (int t0 = 0; t0 < T; t0 += chunk) {
    const int Tc = std::min(chunk, T - t0);
    if (!gemm_partial_geom(Tc, N, K, &g)) {
      *err = cudaErrorInvalidValue;
      return true;
    }
    GemmEpi e;
    e.mode = EPI_PARTIAL;
    if ((*err = gemm(h, (const char*)A + (size_t)t0 * lda * h->p.act, lda, W, Tc, N, K, e)) != cudaSuccess) return true;
    ProfScope ps(h, 2, (double)Tc * N * 4.0 * 3);
    h->launches++;
    *err = dbg_sync(h, "resid_norm",
                    launch_resid_norm(h->gpart, &g, Tc, rep, h->p.d, resid ? resid + t0 * rd : nullptr, nullptr, bias,
                                      out + t0 * rd, tap ? tap + t0 * rd : nullptr, gamma, h->c.rms_eps,
                                      gamma ? (__nv_bfloat16*)h->xn + t0 * rd : nullptr, h->st));
    if (*err != cudaSuccess) return true;
  }
  return true;
}

// Gate/up -> down + residual (+ tap) + next norm with the two GEMMs chained in one launch
// (gemm_chain_launch; bit-identical to the unchained pair). Opt-in, SF_GEMM_CHAIN=1 (read per call):
// measured no faster than the two launches -- every gate/up tile is finished by its
// head group near the end of the gate/up pass, so the down pass still waits for it. Returns false
// (nothing launched) when off or when the shapes do not allow it.
static bool chain_ffn(sf_handle* h, cudaError_t* err, const void* wgu, const void* wdown, int T, float* resid,
                      float* tap, const float* gamma) {
  const char* env = getenv("SF_GEMM_CHAIN");
  if (!env || atoi(env) == 0) return false;
  const Plan& p = h->p;
  if (!h->bf || p.tp > 1 || T > 512 || !gemm_chain_supported(T, 2 * p.F, p.d, p.d) ||
      !resid_norm_supported(p.d, T, p.d, p.F))
    return false;
  PartialGeom g;
  if (!gemm_partial_geom(T, p.d, p.F, &g)) return false;
  GemmScratch sc;
  sc.partial = h->gpart;
  sc.partial_elems = p.gpart_elems;
  sc.counters = h->gcnt;
  sc.n_counters = 4096;
  {
    ProfScope ps(h, 0, (double)2 * p.F * p.d * 2 + (double)p.d * p.F * 2);
    h->launches++;
    if ((*err = dbg_sync(h, "gemm chain", gemm_chain_launch(h->xn, p.d, wgu, 2 * p.F, p.d, h->ffn, wdown, p.d, T, sc,
                                                            h->st))) != cudaSuccess)
      return true;
  }
  ProfScope ps(h, 2, (double)T * p.d * 4.0 * 3);
  h->launches++;
  *err = dbg_sync(h, "resid_norm", launch_resid_norm(h->gpart + gemm_chain_partial_offset(T), &g, T, 1, p.d, resid,
                                                     nullptr, nullptr, resid, tap, gamma, h->c.rms_eps,
                                                     gamma ? (__nv_bfloat16*)h->xn : nullptr, h->st));
  return true;
}

static const int* taps_layers(int L, int* out4) {
  out4[0] = 0;
  out4[1] = L / 2;
  out4[2] = L - 1;
  out4[3] = L;
  return out4;
}

// One attention sub-layer's "RoPE + append + attention" for rows (T, q_len, pos0) of layer `layer`.
// bf16, head_dim 128: RoPE and the paged K/V append can run in the QKV GEMM's epilogue (EPI_QKV_ROPE;
// one launch fewer per attention) for blocks of < SF_ROPE_FUSE_T rows (read per call; tests). Both
// paths rotate the same bf16-rounded projections with the same operations, so the choice per T keeps
// every row's bits (batch invariance). Off by default: the partials + rope consumer form is faster at
// every batch since the GEMM main loop got faster -- the fused form's head-tile fixup is a tail after
// the last MMA (7B ms per step, consumer vs fused: B = 1 3.61 vs 3.72, B = 4 3.78 vs 3.94, B = 8 4.11
// vs 4.35; B >= 13 already used the consumer).
static bool fused_rope(const sf_handle* h, int T) {
  const char* e = getenv("SF_ROPE_FUSE_T");
  const int thr = e ? atoi(e) : 0;
  return h->bf && h->p.hd == 128 && T < thr;
}

// The QKV projection's stream-K k segmentation is the same in every mode it runs in (fused RoPE,
// partials + rope_partial, plain): a row's bits do not depend on the block size.
constexpr int kQkvDrain = 0;
// bf16, head_dim 128, blocks too long for the fused epilogue: the GEMM publishes its k-segment
// partials and launch_rope_partial reduces them while rotating / appending (no fixup tail in the
// GEMM). SF_QKV_PARTIAL=0 (read per call; tests) selects the plain GEMM + rope_append instead.
static bool qkv_partial(const sf_handle* h, int T) {
  const char* e = getenv("SF_QKV_PARTIAL");
  if (e && atoi(e) == 0) return false;
  const Plan& p = h->p;
  return h->bf && p.hd == 128 && !fused_rope(h, T) && T <= 512 &&
         rope_partial_supported(T, p.qkvw, p.d, p.Hq, p.Hkv, kQkvDrain);
}

// QKV projection of layer `layer` (its KV pool): fused RoPE / append, partials for rope_partial, or
// the plain GEMM (rope later)
static cudaError_t qkv_gemm(sf_handle* h, const void* W, int layer, int T, int q_len, const int* pos0) {
  const Plan& p = h->p;
  if (qkv_partial(h, T)) {
    GemmEpi e;
    e.mode = EPI_PARTIAL;
    e.drain = kQkvDrain;
    return gemm(h, h->xn, p.d, W, T, p.qkvw, p.d, e);
  }
  if (!fused_rope(h, T)) {
    GemmEpi e = epi_act(h->qkv, p.qkvw);
    e.drain = kQkvDrain;
    return gemm(h, h->xn, p.d, W, T, p.qkvw, p.d, e);
  }
  GemmEpi e;
  e.drain = kQkvDrain;
  e.mode = EPI_QKV_ROPE;
  e.ldo = 128;
  e.rope.pos0 = pos0;
  e.rope.q_len = q_len;
  e.rope.table = h->rope;
  e.rope.Hq = p.Hq;
  e.rope.Hkv = p.Hkv;
  e.rope.bt = h->bt;
  e.rope.pps = p.pps;
  e.rope.Kp = h->kp(layer);
  e.rope.Vp = h->vp(layer);
  e.rope.q_out = h->qrot;
  return gemm(h, h->xn, p.d, W, T, p.qkvw, p.d, e);
}

static cudaError_t attn_layer(sf_handle* h, int layer, int T, int q_len, const int* pos0, int max_key,
                              bool rope_done = false) {
  const Plan& p = h->p;
  ProfScope ps(h, 1, 0.0);  // KV bytes depend on device-resident lengths: the bench computes them
  cudaError_t e = cudaSuccess;
  if (rope_done) {
    // q rotated and K / V appended already (the layer-sequence kernel's QKV phase)
  } else if (qkv_partial(h, T)) {
    PartialGeom g;
    e = gemm_partial_geom(T, p.qkvw, p.d, &g, kQkvDrain)
            ? launch_rope_partial(h->gpart, &g, T, q_len, pos0, (const float2*)h->rope, p.Hq, p.Hkv, h->bt, p.pps,
                                  h->kp(layer), h->vp(layer), h->qrot, h->st)
            : cudaErrorInvalidValue;
  } else if (!fused_rope(h, T)) {
    e = launch_rope_append(h->bf, h->qkv, T, q_len, pos0, h->rope, p.Hq, p.Hkv, p.hd, h->bt, p.pps, h->kp(layer),
                           h->vp(layer), h->qrot, h->bf && p.hd == 128, h->st);
  }
  if (e != cudaSuccess) return e;
  AttnParams ap{};
  ap.q = h->qrot;
  ap.Kp = h->kp(layer);
  ap.Vp = h->vp(layer);
  ap.block_table = h->bt;
  ap.pages_per_seq = p.pps;
  ap.pos0 = pos0;
  ap.q_len = q_len;
  ap.B = T / q_len;
  ap.Hq = p.Hq;
  ap.Hkv = p.Hkv;
  ap.hd = p.hd;
  ap.nchunk_max = p.nchunk;
  ap.part_o = h->apo;
  ap.part_ml = h->apml;
  ap.seg_cnt = h->acnt;
  ap.out = h->attn;
  ap.max_key = std::min(max_key, h->c.max_seq);
  ap.n_pages = p.n_pages;
  h->launches += 3;
  if ((e = dbg_sync(h, "rope_append", e)) != cudaSuccess) return e;
  return dbg_sync(h, "attention", launch_attention(h->bf, ap, h->st));
}

// Small verify blocks (T <= SF_SEQ_T; off by default, see seq_T): the part of base layer l
// between two attentions -- O-proj + residual + RMS_ffn, gate/up SwiGLU, down + residual (+ tap) +
// the next norm, and layer l+1's QKV with RoPE / KV append -- as ONE persistent launch
// (gemm_seq_launch, csrc/gemm_seq.cuh) with the standalone launches' partition and arithmetic
// (bit-identical; SF_SEQ_T=0 turns it off). Returns false (nothing launched) when the shapes or
// switches call for the standalone path.
static int seq_T() {
  const char* e = getenv("SF_SEQ_T");  // (read per call: tests compare both paths)
  // Off by default (opt-in, SF_SEQ_T=80): it won 3-5% at B = 1..4 against the standalone launches
  // while their MMA issue loop was the main-loop bound; with that loop fixed the standalone path is
  // faster at every batch (7B, ms per step: B = 1 3.72 vs 4.15, B = 2 3.79 vs 4.23, B = 4 3.95 vs
  // 4.47, B = 8 4.35 vs 5.23) -- the per-phase grid-wide dependencies now cost more than the launch
  // boundaries they remove.
  return e ? atoi(e) : 0;
}
static bool layer_seq(sf_handle* h, cudaError_t* err, int l, int T, int q_len, const int* pos0, float* tap,
                      const float* next_g) {
  const Plan& p = h->p;
  const char* chain = getenv("SF_GEMM_CHAIN");
  if (!h->bf || p.hd != 128 || p.tp > 1 || T > seq_T() || T > 128 || (chain && atoi(chain) != 0)) return false;
  if (!resid_norm_supported(p.d, T, p.d, p.ao) || !resid_norm_supported(p.d, T, p.d, p.F)) return false;
  const auto& w = h->lw[l];
  SeqStep st[kSeqMaxPhases];
  int n = 0;
  SeqStep& o = st[n++];  // O-proj -> k-segment partials
  o.A = h->attn, o.lda = p.ao, o.W = w.wo, o.N = p.d, o.K = p.ao;
  o.epi.mode = EPI_PARTIAL;
  SeqStep& r1 = st[n++];  // residual + RMS_ffn
  r1.kind = SEQ_RESID_NORM;
  r1.resid = h->resid, r1.out = h->resid, r1.gamma = w.ffn_norm, r1.xn = (__nv_bfloat16*)h->xn, r1.d = p.d;
  r1.eps = h->c.rms_eps;
  SeqStep& gu = st[n++];  // gate/up SwiGLU
  gu.A = h->xn, gu.lda = p.d, gu.W = w.wgu, gu.N = 2 * p.F, gu.K = p.d;
  gu.epi.mode = EPI_SWIGLU_ACT, gu.epi.out = h->ffn, gu.epi.ldo = p.F;
  SeqStep& dn = st[n++];  // down -> partials
  dn.A = h->ffn, dn.lda = p.F, dn.W = w.wdown, dn.N = p.d, dn.K = p.F;
  dn.epi.mode = EPI_PARTIAL;
  SeqStep& r2 = st[n++];  // residual (+ tap) + the next norm
  r2.kind = SEQ_RESID_NORM;
  r2.resid = h->resid, r2.out = h->resid, r2.tap = tap, r2.gamma = next_g;
  r2.xn = next_g ? (__nv_bfloat16*)h->xn : nullptr, r2.d = p.d, r2.eps = h->c.rms_eps;
  if (l + 1 < p.L) {  // layer l+1's QKV projection, as qkv_gemm would run it at this T
    RopeEpi R;
    R.pos0 = pos0, R.q_len = q_len, R.table = h->rope, R.Hq = p.Hq, R.Hkv = p.Hkv, R.bt = h->bt, R.pps = p.pps;
    R.Kp = h->kp(l + 1), R.Vp = h->vp(l + 1), R.q_out = h->qrot;
    SeqStep& q = st[n++];
    q.A = h->xn, q.lda = p.d, q.W = h->lw[l + 1].wqkv, q.N = p.qkvw, q.K = p.d;
    q.epi.drain = kQkvDrain;
    if (fused_rope(h, T)) {
      q.epi.mode = EPI_QKV_ROPE, q.epi.ldo = 128, q.epi.rope = R;
    } else if (qkv_partial(h, T)) {
      q.epi.mode = EPI_PARTIAL;
      SeqStep& rp = st[n++];
      rp.kind = SEQ_ROPE;
      rp.epi.rope = R;
    } else {
      return false;
    }
  }
  if (!gemm_seq_supported(T, st, n)) return false;
  double wbytes = 2.0 * ((double)p.d * p.ao + 3.0 * p.d * p.F + (l + 1 < p.L ? (double)p.qkvw * p.d : 0.0));
  ProfScope ps(h, 0, wbytes);
  GemmScratch sc;
  sc.partial = h->gpart;
  sc.partial_elems = p.gpart_elems;
  sc.counters = h->gcnt;
  sc.n_counters = 4096;
  h->launches++;
  *err = dbg_sync(h, "layer_seq", gemm_seq_launch(T, st, n, sc, h->seqsync + (size_t)l * kSeqSyncInts, h->st));
  return true;
}

// Base decoder forward over T rows (q_len per sequence, positions pos0[b] + i); writes resid and
// the 4 hook taps (P175) into h->taps.
static cudaError_t base_forward(sf_handle* h, int T, int q_len, const int* pos0, int max_key,
                                bool final_norm = true) {
  const Plan& p = h->p;
  const int64_t tstride = (int64_t)p.R * p.d;
  int tl[4];
  taps_layers(p.L, tl);
  cudaError_t e = launch_embed(h->bf, h->tok_rows, h->embed, T, p.d, p.V_full, h->resid, h->taps, h->st);
  h->launches++;
  h->fwd_rows = T;
  if (e != cudaSuccess) return e;
  for (int g = 1; g < 4; ++g)
    if (tl[g] == 0) cudaMemcpyAsync(h->taps + g * tstride, h->taps, (size_t)T * p.d * 4, cudaMemcpyDeviceToDevice, h->st);
  bool xn_ready = false;  // xn already holds RMS_attn(resid) of this layer (fused into the last consumer)
  bool qkv_done = false;  // layer l's QKV projection, RoPE and KV append ran in the previous layer_seq launch
  for (int l = 0; l < p.L; ++l) {
    const auto& w = h->lw[l];
    if (qkv_done) {
      if ((e = attn_layer(h, l, T, q_len, pos0, max_key, true))) return e;
    } else {
      if (!xn_ready && (e = rmsnorm(h, h->resid, p.d, w.attn_norm, T, h->xn, p.d))) return e;
      if ((e = qkv_gemm(h, w.wqkv, l, T, q_len, pos0))) return e;
      if ((e = attn_layer(h, l, T, q_len, pos0, max_key))) return e;
    }
    qkv_done = false;
    {
      int first = -1;
      for (int g = 0; g < 4; ++g)
        if (tl[g] == l + 1 && first < 0) first = g;
      float* tap = first >= 0 ? h->taps + first * tstride : nullptr;
      const float* next_g = (l + 1 < p.L) ? h->lw[l + 1].attn_norm : (final_norm ? h->final_norm : nullptr);
      if (layer_seq(h, &e, l, T, q_len, pos0, tap, next_g)) {
        if (e) return e;
        for (int g = first + 1; first >= 0 && g < 4; ++g)
          if (tl[g] == l + 1)
            cudaMemcpyAsync(h->taps + g * tstride, tap, (size_t)T * p.d * 4, cudaMemcpyDeviceToDevice, h->st);
        xn_ready = next_g != nullptr;
        qkv_done = l + 1 < p.L;
        continue;
      }
    }
    // o-proj + residual + RMS_ffn
    if (!gemm_resid_norm(h, &e, h->attn, p.ao, w.wo, T, p.d, p.ao, 1, h->resid, nullptr, h->resid, nullptr,
                         w.ffn_norm, true)) {
      if ((e = gemm(h, h->attn, p.ao, w.wo, T, p.d, p.ao, epi_add(h->resid, p.d, nullptr)))) return e;
      e = rmsnorm(h, h->resid, p.d, w.ffn_norm, T, h->xn, p.d);
    }
    if (e) return e;
    // down-proj + residual (+ hook tap HS[l+1]) + the next RMSNorm
    int first = -1;
    for (int g = 0; g < 4; ++g)
      if (tl[g] == l + 1 && first < 0) first = g;
    float* tap = first >= 0 ? h->taps + first * tstride : nullptr;
    const float* next_g = (l + 1 < p.L) ? h->lw[l + 1].attn_norm : (final_norm ? h->final_norm : nullptr);
    if (chain_ffn(h, &e, w.wgu, w.wdown, T, h->resid, tap, next_g)) {
      xn_ready = next_g != nullptr;
    } else {
      GemmEpi sw;
      sw.mode = EPI_SWIGLU_ACT;
      sw.out = h->ffn;
      sw.ldo = p.F;
      if ((e = gemm(h, h->xn, p.d, w.wgu, T, 2 * p.F, p.d, sw))) return e;
      if (gemm_resid_norm(h, &e, h->ffn, p.F, w.wdown, T, p.d, p.F, 1, h->resid, nullptr, h->resid, tap, next_g,
                          true)) {
        xn_ready = next_g != nullptr;
      } else {
        if ((e = gemm(h, h->ffn, p.F, w.wdown, T, p.d, p.F, epi_add(h->resid, p.d, tap)))) return e;
        xn_ready = false;
      }
    }
    if (e) return e;
    for (int g = first + 1; first >= 0 && g < 4; ++g)
      if (tl[g] == l + 1)
        cudaMemcpyAsync(h->taps + g * tstride, tap, (size_t)T * p.d * 4, cudaMemcpyDeviceToDevice, h->st);
  }
  h->final_xn_ready = xn_ready;  // xn = RMS_f(HS[L]) when the last consumer applied the final norm
  return cudaSuccess;
}

// SpecFormer context layer L+1 (Eq.8) over T rows of taps -> h->ctx (= I_D rows).
static cudaError_t ctx_forward(sf_handle* h, int T, int q_len, const int* pos0, int max_key) {
  const Plan& p = h->p;
  cudaError_t e;
  h->ctx_rows = T;
  if ((e = launch_group_rms(h->bf, h->taps, (int64_t)p.R * p.d, h->group_scale, h->c.rms_eps, T, p.d, h->xn, h->st)))
    return e;
  h->launches++;
  // X = W_D I_Cat -> ctx, xn = RMS_c(X)
  // (tensor parallelism: this rank's W_D input columns [r 4d/tp, ..) of I_Cat)
  const void* icat = (const char*)h->xn + (size_t)p.tp_rank * p.wd_k * p.act;
  if (!gemm_resid_norm(h, &e, icat, 4 * p.d, h->w_d, T, p.d, p.wd_k, 1, nullptr, nullptr, h->ctx, nullptr,
                       h->ctx_norm, true)) {
    if ((e = gemm(h, h->xn, 4 * p.d, h->w_d, T, p.d, 4 * p.d, epi_f32(h->ctx, p.d)))) return e;
    e = rmsnorm(h, h->ctx, p.d, h->ctx_norm, T, h->xn, p.d);
  }
  if (e) return e;
  if ((e = qkv_gemm(h, h->ctx_wqkv, p.L, T, q_len, pos0))) return e;
  if ((e = attn_layer(h, p.L, T, q_len, pos0, max_key))) return e;
  // I_D = X + MSA(...)
  if (!gemm_resid_norm(h, &e, h->attn, p.ao, h->ctx_wo, T, p.d, p.ao, 1, h->ctx, nullptr, h->ctx, nullptr, nullptr,
                       true))
    e = gemm(h, h->attn, p.ao, h->ctx_wo, T, p.d, p.ao, epi_add(h->ctx, p.d, nullptr));
  return e;
}

// final norm + LM head + argmax over T rows of `src` (f32 [T, d])
static cudaError_t head_argmax(sf_handle* h, const float* src, int T, float* logits, int* out, bool xn_ready = false) {
  const Plan& p = h->p;
  cudaError_t e;
  if (!xn_ready && (e = rmsnorm(h, src, p.d, h->final_norm, T, h->xn, p.d))) return e;
  if (h->bf) {
    // LM head with the argmax fused into its epilogue (packed (logit, id) keys, NEXT-4); a
    // vocabulary-sharded head max-reduces the shards' keys (TP), then the winner's id is unpacked
    GemmEpi ea = epi_f32((h->c.flags & SF_FLAG_NO_LOGITS) ? nullptr : logits, p.V);
    ea.amax = h->tpkey;
    ea.amax_v0 = (unsigned)p.v0;
    ea.amax_err = h->err;
    if ((e = gemm(h, h->xn, p.d, h->lm_head, T, p.V, p.d, ea))) return e;
    h->launches++;
    ProfScope ps(h, 3, (double)T * 8.0);
    if (p.tp > 1 && (e = tp_max(h, h->tpkey, T))) return e;
    return launch_argmax_unkey(h->tpkey, T, out, h->st, true);
  }
  if ((e = gemm(h, h->xn, p.d, h->lm_head, T, p.V, p.d, epi_f32(logits, p.V)))) return e;
  h->launches += 2;
  ProfScope ps(h, 3, (double)T * p.V * 4.0);
  return launch_argmax(logits, T, p.V, h->amv, h->ami, out, h->err, h->st);
}

static cudaError_t do_draft(sf_handle* h) {
  const Plan& p = h->p;
  const int B = h->B, k = p.k;
  cudaError_t e;
  if (h->ctx_pending) {
    if ((e = ctx_forward(h, B * (k + 1), k + 1, h->n_prev, h->c.max_seq))) return e;
    if ((e = launch_gather_rows(h->ctx, k + 1, h->r_b, 0, B, p.d, h->idrow, h->st))) return e;
    h->launches++;
    h->ctx_pending = false;
  }
  // positional FFN (Eq.9): D = W_P RMS(I_D) + b_P  -> [B, k*d] == [B*k, d]
  const int Tk = B * k;
  if (h->c.flags & SF_FLAG_NO_POS_FFN) {
    // "-Pos" (NEXT-2): D_j = RMS_p(I_D) + b_P[j]; xn = RMS_1(D)
    h->launches += 2;
    if ((e = launch_pos_broadcast(h->idrow, h->pos_norm, h->b_p, B, k, p.d, h->c.rms_eps, h->D, h->st))) return e;
    if ((e = rmsnorm(h, h->D, p.d, h->blk_attn_norm, Tk, h->xn, p.d))) return e;
  } else if ((e = rmsnorm(h, h->idrow, p.d, h->pos_norm, B, h->xn, p.d))) {
    return e;
  }
  // D = W_P RMS_p(I_D) + b_P viewed as [B*k, d]; xn = RMS_1(D)
  if ((h->c.flags & SF_FLAG_NO_POS_FFN)) {
  } else if (!gemm_resid_norm(h, &e, h->xn, p.d, h->w_p, B, k * p.d, p.d, k, nullptr, h->b_p, h->D, nullptr,
                              h->blk_attn_norm)) {
    GemmEpi eb;
    eb.mode = EPI_BIAS_F32;
    eb.out = h->D;
    eb.ldo = k * p.d;
    eb.bias = h->b_p;
    if ((e = gemm(h, h->xn, p.d, h->w_p, B, k * p.d, p.d, eb))) return e;
    e = rmsnorm(h, h->D, p.d, h->blk_attn_norm, Tk, h->xn, p.d);
  }
  if (e) return e;
  // draft bidirectional layer(s) (Eq.10; more than one: NEXT-2 "+Larger")
  bool xn_ready = false;
  for (size_t bi = 0; bi < h->blks.size(); ++bi) {
    const auto& bw = h->blks[bi];
    if ((e = gemm(h, h->xn, p.d, bw.wqkv, Tk, p.qkvw, p.d, epi_act(h->qkv, p.qkvw)))) return e;
    if (h->c.flags & SF_FLAG_DRAFT_PREFIX) {
      // BIDIR_PREFIX (NEXT-2): slots at positions seq_len..seq_len+k-1 of the context layer's pages (beyond
      // the committed length: the next context pass overwrites them), every slot sees the committed keys
      // and all k slots. The draft block's q|k|v rows are in natural order (no RoPE pairing).
      if ((e = launch_rope_append(h->bf, h->qkv, Tk, k, h->seq_len, h->rope, p.Hq, p.Hkv, p.hd, h->bt, p.pps,
                                  h->kp(p.L), h->vp(p.L), h->qrot, h->bf && p.hd == 128, h->st, false)))
        return e;
      AttnParams ap{};
      ap.q = h->qrot;
      ap.Kp = h->kp(p.L);
      ap.Vp = h->vp(p.L);
      ap.block_table = h->bt;
      ap.pages_per_seq = p.pps;
      ap.pos0 = h->seq_len;
      ap.q_len = k;
      ap.B = B;
      ap.Hq = p.Hq;
      ap.Hkv = p.Hkv;
      ap.hd = p.hd;
      ap.nchunk_max = p.nchunk;
      ap.part_o = h->apo;
      ap.part_ml = h->apml;
      ap.seg_cnt = h->acnt;
      ap.out = h->attn;
      ap.max_key = h->c.max_seq;
      ap.n_pages = p.n_pages;
      ap.bidir_tail = 1;
      h->launches += 2;
      if ((e = launch_attention(h->bf, ap, h->st))) return e;
    } else {
      if ((e = launch_bidir_attention(h->bf, h->qkv, B, k, p.Hq, p.Hkv, p.hd, (h->c.flags & SF_FLAG_DRAFT_CAUSAL) != 0,
                                      h->attn, h->st)))
        return e;
      h->launches++;
    }
    if (!gemm_resid_norm(h, &e, h->attn, p.ao, bw.wo, Tk, p.d, p.ao, 1, h->D, nullptr, h->D, nullptr, bw.ffn_norm,
                         true)) {
      if ((e = gemm(h, h->attn, p.ao, bw.wo, Tk, p.d, p.ao, epi_add(h->D, p.d, nullptr)))) return e;
      e = rmsnorm(h, h->D, p.d, bw.ffn_norm, Tk, h->xn, p.d);
    }
    if (e) return e;
    GemmEpi sw;
    sw.mode = EPI_SWIGLU_ACT;
    sw.out = h->ffn;
    sw.ldo = p.F;
    if ((e = gemm(h, h->xn, p.d, bw.wgu, Tk, 2 * p.F, p.d, sw))) return e;
    // E = Y + SwiGLU(...); xn = the next block's RMS_1(E), after the last RMS_f(E) (shared frozen
    // final norm, C8)
    const bool last = bi + 1 == h->blks.size();
    const float* next_g = last ? h->final_norm : h->blks[bi + 1].attn_norm;
    xn_ready = gemm_resid_norm(h, &e, h->ffn, p.F, bw.wdown, Tk, p.d, p.F, 1, h->D, nullptr, h->D, nullptr, next_g,
                               true);
    if (!xn_ready) {
      if ((e = gemm(h, h->ffn, p.F, bw.wdown, Tk, p.d, p.F, epi_add(h->D, p.d, nullptr)))) return e;
      if (!last && (e = rmsnorm(h, h->D, p.d, next_g, Tk, h->xn, p.d))) return e;
    }
    if (e) return e;
  }
  // shared frozen LM head -> k draft tokens
  return head_argmax(h, h->D, Tk, h->dlogits, h->draft, xn_ready);
}

static cudaError_t do_verify(sf_handle* h) {
  const Plan& p = h->p;
  const int B = h->B, k = p.k;
  const int T = B * (k + 1);
  cudaError_t e;
  if ((e = launch_build_verify_rows(B, k, h->last_token, h->draft, h->tok_rows, h->st))) return e;
  h->launches++;
  if ((e = base_forward(h, T, k + 1, h->seq_len, h->c.max_seq))) return e;
  return head_argmax(h, h->resid, T, h->logits, h->greedy, h->final_xn_ready);
}

static cudaError_t do_accept(sf_handle* h, int* acc_log, int* em_log) {
  const Plan& p = h->p;
  h->launches++;
  cudaError_t e = launch_accept(h->B, p.k, h->draft, h->greedy, h->seq_len, h->n_prev, h->last_token, h->r_b,
                                h->accept_len, h->emitted, h->step_counter, acc_log, em_log, h->d_logcap, h->pp, h->st);
  if (p.k > 0) h->ctx_pending = true;
  return e;
}

static bool any_released(const sf_handle* h) {
  for (char r : h->released)
    if (r) return true;
  return false;
}

static cudaError_t copy_out(sf_handle* h, void* dst, const void* src, size_t bytes) {
  if (!dst) return cudaSuccess;
  return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, h->st);
}

// ================================================================= collectives (tensor parallelism)
#ifdef SF_WITH_NCCL
static cudaError_t nccl_sum_f32(void* ctx, float* buf, int64_t n, cudaStream_t s) {
  return ncclAllReduce(buf, buf, (size_t)n, ncclFloat32, ncclSum, (ncclComm_t)ctx, s) == ncclSuccess
             ? cudaSuccess
             : cudaErrorUnknown;
}
static cudaError_t nccl_sum_bf16(void* ctx, __nv_bfloat16* buf, int64_t n, cudaStream_t s) {
  return ncclAllReduce(buf, buf, (size_t)n, ncclBfloat16, ncclSum, (ncclComm_t)ctx, s) == ncclSuccess
             ? cudaSuccess
             : cudaErrorUnknown;
}
static cudaError_t nccl_max_u64(void* ctx, unsigned long long* buf, int64_t n, cudaStream_t s) {
  return ncclAllReduce(buf, buf, (size_t)n, ncclUint64, ncclMax, (ncclComm_t)ctx, s) == ncclSuccess
             ? cudaSuccess
             : cudaErrorUnknown;
}
#endif

// Several handles of one process on one device, one host thread each (tests: tensor parallelism
// without a second GPU). Every reduction: each rank records its input, a host barrier, each rank
// sums / maxes all inputs in rank order into its own scratch, a barrier, each copies the result
// back, a barrier (events and inputs are reused by the next reduction). Host barriers cannot be
// captured, so handles on a local group run their steps eagerly.
struct sf_local_group {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t gen = 0;
  std::vector<const void*> bufs;
  std::vector<cudaEvent_t> ev_in, ev_mid;
  std::vector<void*> tmp;
  std::vector<size_t> tmp_bytes;
  std::vector<char*> xch;          // NEXT-3: the ranks' exchange regions
  std::vector<cudaEvent_t> ev_x;   // and their signal events
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const int64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct LocalCtx {
  sf_local_group* g;
  int rank;
};
static cudaError_t local_reduce(void* ctx, void* buf, int64_t n, int mode, cudaStream_t s) {
  LocalCtx* c = (LocalCtx*)ctx;
  sf_local_group* g = c->g;
  const int r = c->rank;
  const size_t bytes = (size_t)n * (mode == 1 ? 8 : mode == 2 ? 2 : 4);
  if (g->tmp_bytes[r] < bytes) {  // (test scratch, owned by the group)
    cudaStreamSynchronize(s);
    if (g->tmp[r]) cudaFree(g->tmp[r]);
    if (cudaMalloc(&g->tmp[r], bytes) != cudaSuccess) return cudaErrorMemoryAllocation;
    g->tmp_bytes[r] = bytes;
  }
  g->bufs[r] = buf;
  cudaEventRecord(g->ev_in[r], s);
  g->barrier();
  for (int q = 0; q < g->n; ++q) cudaStreamWaitEvent(s, g->ev_in[q], 0);
  cudaError_t e = launch_reduce_bufs(g->bufs.data(), g->n, n, mode, g->tmp[r], s);
  cudaEventRecord(g->ev_mid[r], s);
  g->barrier();
  for (int q = 0; q < g->n; ++q) cudaStreamWaitEvent(s, g->ev_mid[q], 0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(buf, g->tmp[r], bytes, cudaMemcpyDeviceToDevice, s);
  g->barrier();
  return e;
}
// (local group, fused TP all-reduce) every rank's epoch signal has executed before any rank's
// consumer starts: its flag waits are then already satisfied, no kernel waits on another rank's
static void local_xch_barrier(sf_handle* h) {
  sf_local_group* g = (sf_local_group*)h->xgroup;
  const int r = h->p.tp_rank;
  cudaEventRecord(g->ev_x[r], h->st);
  g->barrier();
  for (int q = 0; q < g->n; ++q) cudaStreamWaitEvent(h->st, g->ev_x[q], 0);
  g->barrier();  // (every wait enqueued before any rank re-records its event)
}
static cudaError_t local_sum_f32(void* ctx, float* buf, int64_t n, cudaStream_t s) {
  return local_reduce(ctx, buf, n, 0, s);
}
static cudaError_t local_sum_bf16(void* ctx, __nv_bfloat16* buf, int64_t n, cudaStream_t s) {
  return local_reduce(ctx, buf, n, 2, s);
}
static cudaError_t local_max_u64(void* ctx, unsigned long long* buf, int64_t n, cudaStream_t s) {
  return local_reduce(ctx, buf, n, 1, s);
}

// ================================================================= C ABI
// ---- kernel timeline (SF_KTRACE=1; tools/ktrace.py)
static void* g_kt_rec = nullptr;
static unsigned* g_kt_cnt = nullptr;
static constexpr unsigned kKtCap = 1u << 21;
static bool g_kt_on = false;
static bool kt_set(bool on) {
  if (on && !g_kt_rec) {
    if (cudaMalloc(&g_kt_rec, (size_t)kKtCap * kKtRecBytes) != cudaSuccess) return false;
    if (cudaMalloc((void**)&g_kt_cnt, 4) != cudaSuccess) return false;
  }
  if (!g_kt_rec) return !on;
  cudaDeviceSynchronize();
  cudaMemset(g_kt_cnt, 0, 4);
  void* rec = on ? g_kt_rec : nullptr;  // a null record pointer turns every probe off
  kt_setup_kernels(rec, g_kt_cnt, kKtCap);
  kt_setup_gemm(rec, g_kt_cnt, kKtCap);
  kt_setup_attn_fd(rec, g_kt_cnt, kKtCap);
  cudaDeviceSynchronize();
  g_kt_on = on;
  return true;
}
static bool kt_enable() {  // SF_KTRACE=1: on from the first handle on
  static const bool env = getenv("SF_KTRACE") && atoi(getenv("SF_KTRACE")) > 0;
  if (env && !g_kt_on) kt_set(true);
  return g_kt_on;
}

extern "C" {

int sf_weight_table(const sf_config* cfg, sf_tensor_desc* out, int cap) {
  if (!valid_config(cfg, nullptr)) return -1;
  auto specs = tensor_specs(cfg);
  int64_t off = 0;
  for (size_t i = 0; i < specs.size(); ++i) {
    if (out && (int)i < cap) {
      sf_tensor_desc& d = out[i];
      memset(&d, 0, sizeof(d));
      strncpy(d.name, specs[i].name.c_str(), sizeof(d.name) - 1);
      d.ndim = (int32_t)specs[i].shape.size();
      for (int j = 0; j < d.ndim; ++j) d.shape[j] = specs[i].shape[j];
      d.offset_bytes = off;
      d.dtype = (specs[i].matrix && cfg->dtype == SF_BF16) ? SF_BF16 : SF_FP32;
      d.layout = (specs[i].matrix && cfg->dtype == SF_BF16 && specs[i].name != "embed") ? 1 : 0;
    }
    off += align_up(tensor_bytes(cfg, specs[i]));
  }
  return (int)specs.size();
}

int64_t sf_weights_bytes(const sf_config* cfg) {
  if (!valid_config(cfg, nullptr)) return -1;
  int64_t off = 0;
  for (auto& s : tensor_specs(cfg)) off += align_up(tensor_bytes(cfg, s));
  return off;
}

int64_t sf_workspace_bytes(const sf_config* cfg) {
  if (!valid_config(cfg, nullptr)) return -1;
  return make_plan(cfg).total;
}

const char* specformer_build_info(void) {
  return "specformer sm_100a (tcgen05/TMA bf16 GEMM, SIMT fp32 mode), built " __DATE__ " " __TIME__;
}

sf_status specformer_init(const sf_config* cfg, void* weights_dev, void* workspace_dev, void* stream,
                          sf_handle** out) {
  if (!out) return SF_ERR_ARG;
  *out = nullptr;
  std::string why;
  if (!valid_config(cfg, &why)) return SF_ERR_ARG;
  if (!weights_dev || !workspace_dev) return SF_ERR_ARG;
  if (((uintptr_t)weights_dev | (uintptr_t)workspace_dev) % kAlign) return SF_ERR_ARG;
  kt_enable();  // no-op unless SF_KTRACE=1
  auto* h = new sf_handle();
  h->c = *cfg;
  h->p = make_plan(cfg);
  h->bf = cfg->dtype == SF_BF16;
  h->st = (cudaStream_t)stream;
  h->W = (char*)weights_dev;
  h->ws = (char*)workspace_dev;
  // bind weights
  auto specs = tensor_specs(cfg);
  int64_t off = 0;
  std::vector<std::pair<std::string, char*>> ptrs;
  for (auto& s : specs) {
    ptrs.push_back({s.name, h->W + off});
    off += align_up(tensor_bytes(cfg, s));
  }
  auto get = [&](const std::string& n) -> char* {
    for (auto& pr : ptrs)
      if (pr.first == n) return pr.second;
    return nullptr;
  };
  h->lw.resize(cfg->n_layers);
  for (int l = 0; l < cfg->n_layers; ++l) {
    const std::string p = "layers." + std::to_string(l) + ".";
    h->lw[l].attn_norm = (const float*)get(p + "attn_norm");
    h->lw[l].ffn_norm = (const float*)get(p + "ffn_norm");
    h->lw[l].wqkv = get(p + "wqkv");
    h->lw[l].wo = get(p + "wo");
    h->lw[l].wgu = get(p + "w_gu");
    h->lw[l].wdown = get(p + "w_down");
  }
  h->embed = get("embed");
  h->final_norm = (const float*)get("final_norm");
  h->lm_head = get("lm_head");
  if (cfg->draft_len > 0) {
    h->group_scale = (const float*)get("sf.group_scale");
    h->w_d = get("sf.w_d");
    h->ctx_norm = (const float*)get("sf.ctx_norm");
    h->ctx_wqkv = get("sf.ctx_wqkv");
    h->ctx_wo = get("sf.ctx_wo");
    h->pos_norm = (const float*)get("sf.pos_norm");
    h->w_p = get("sf.w_p");
    h->b_p = (const float*)get("sf.b_p");
    h->blk_attn_norm = (const float*)get("sf.blk_attn_norm");
    h->blk_wqkv = get("sf.blk_wqkv");
    h->blk_wo = get("sf.blk_wo");
    h->blk_ffn_norm = (const float*)get("sf.blk_ffn_norm");
    h->blk_wgu = get("sf.blk_w_gu");
    h->blk_wdown = get("sf.blk_w_down");
    for (int i = 0; i < draft_blocks(cfg); ++i) {
      const std::string b = i == 0 ? "sf.blk_" : "sf.blk" + std::to_string(i) + "_";
      h->blks.push_back({(const float*)get(b + "attn_norm"), (const float*)get(b + "ffn_norm"), get(b + "wqkv"),
                         get(b + "wo"), get(b + "w_gu"), get(b + "w_down")});
    }
  }  {
    // GEMM weight chain in launch order: draft (W_D, ctx QKV/O, W_P, block QKV/O/gate-up/down, LM
    // head), then verify (per layer QKV, O, gate-up, down; LM head), then the next step's draft
    const int64_t d = cfg->d_model, F = h->p.F, V = h->p.V, k = cfg->draft_len;
    const int64_t qkv = h->p.qkvw, ao = h->p.ao;
    auto add = [&](const void* w, int64_t n, int64_t kk) { h->wchain.push_back({w, (size_t)(n * kk * 2)}); };
    if (k > 0) {
      add(h->w_d, d, h->p.wd_k);
      add(h->ctx_wqkv, qkv, d);
      add(h->ctx_wo, d, ao);
      add(h->w_p, k * d, d);
      for (const auto& b : h->blks) {
        add(b.wqkv, qkv, d);
        add(b.wo, d, ao);
        add(b.wgu, 2 * F, d);
        add(b.wdown, d, F);
      }
      add(h->lm_head, V, d);
    }
    for (int l = 0; l < cfg->n_layers; ++l) {
      add(h->lw[l].wqkv, qkv, d);
      add(h->lw[l].wo, d, ao);
      add(h->lw[l].wgu, 2 * F, d);
      add(h->lw[l].wdown, d, F);
    }
    add(h->lm_head, V, d);
  }

  // carve workspace
  const Plan& p = h->p;
  char* w = h->ws;
  h->kpool = w + p.o_k;
  h->vpool = w + p.o_v;
  h->bt = (int*)(w + p.o_bt);
  h->rope = (float2*)(w + p.o_rope);
  h->resid = (float*)(w + p.o_resid);
  h->xn = w + p.o_xn;
  h->qkv = w + p.o_qkv;
  h->qrot = (float*)(w + p.o_qrot);
  h->attn = w + p.o_attn;
  h->ffn = w + p.o_ffn;
  h->taps = (float*)(w + p.o_taps);
  h->ctx = (float*)(w + p.o_ctx);
  h->idrow = (float*)(w + p.o_idrow);
  h->D = (float*)(w + p.o_D);
  h->hlast = (float*)(w + p.o_hlast);
  h->logits = (float*)(w + p.o_logits);
  h->dlogits = (float*)(w + p.o_dlogits);
  h->apo = (float*)(w + p.o_apo);
  h->apml = (float*)(w + p.o_apml);
  h->acnt = (int*)(w + p.o_acnt);
  h->gpart = (float*)(w + p.o_gpart);
  h->gcnt = (int*)(w + p.o_gcnt);
  h->amv = (float*)(w + p.o_amv);
  h->ami = (int*)(w + p.o_ami);
  h->tpbuf = p.tp > 1 ? (float*)(w + p.o_tpbuf) : nullptr;
  h->tpbf = p.tp > 1 ? (__nv_bfloat16*)(w + p.o_tpbf) : nullptr;
  h->tpkey = h->bf ? (unsigned long long*)(w + p.o_tpkey) : nullptr;
  h->seqsync = h->bf ? (int*)(w + p.o_seqsync) : nullptr;
  int* ip = (int*)(w + p.o_ints);
  auto ints = [&](int n) {
    int* r = ip;
    ip += n;
    return r;
  };
  h->tok_rows = ints(p.R);
  h->pos0_pf = ints(p.B);
  h->seq_len = ints(p.B);
  h->n_prev = ints(p.B);
  h->last_token = ints(p.B);
  h->r_b = ints(p.B);
  h->prompt_len = ints(p.B);
  h->draft = ints(p.rows_d);
  h->greedy = ints(p.rows_v);
  h->accept_len = ints(p.B);
  h->emitted = ints(p.rows_v);
  h->err = ints(1);
  h->step_counter = ints(1);
  h->d_logcap = ints(1);
  h->g_pf = ints(p.B);
  h->prompt = (int*)(w + p.o_prompt);
  cudaError_t e = cudaSuccess;
  // page table: identity (sequence b owns pages [b*pps, (b+1)*pps)); tests may permute it. With the page
  // pool, entries are filled as pages are taken.
  std::vector<int> bt((size_t)p.B * p.pps);
  for (size_t i = 0; i < bt.size(); ++i) bt[i] = p.pool ? 0 : (int)i;
  e = cudaMemcpyAsync(h->bt, bt.data(), bt.size() * 4, cudaMemcpyHostToDevice, h->st);
  if (p.pool) {
    int* pw = (int*)(w + p.o_pool);
    h->pp.pool = pw;
    h->pp.alloc_cnt = pw + p.n_pages;
    h->pp.top = pw + p.n_pages + p.B;
    h->pp.bt = h->bt;
    h->pp.err = h->err;
    h->pp.pps = p.pps;
    h->released.assign(p.B, 0);
    if (e == cudaSuccess) e = launch_page_reset(p.n_pages, p.B, h->pp, h->st);
  }
  if (e == cudaSuccess) e = cudaMemsetAsync(h->gcnt, 0, 4096 * 4, h->st);
  if (e == cudaSuccess) e = cudaMemsetAsync(h->acnt, 0, (size_t)p.n_acnt * 4, h->st);
  if (e == cudaSuccess && h->seqsync) e = cudaMemsetAsync(h->seqsync, 0, (size_t)p.L * kSeqSyncInts * 4, h->st);
  // whole 16-key pages are staged by TMA: never-written slots must hold finite values (masked keys
  // get probability exactly 0, and 0 * finite = 0)
  if (e == cudaSuccess) e = cudaMemsetAsync(h->kpool, 0, (size_t)p.kv_layer_bytes * (p.L + 1), h->st);
  if (e == cudaSuccess) e = cudaMemsetAsync(h->vpool, 0, (size_t)p.kv_layer_bytes * (p.L + 1), h->st);
  if (e == cudaSuccess) e = cudaMemsetAsync(h->ws + p.o_ints, 0, (16 * p.B + 2 * p.R + 8 + p.rows_v * 2 + p.rows_d) * 4, h->st);
  if (e == cudaSuccess) e = launch_rope_table(h->rope, cfg->max_seq, p.hd, cfg->rope_theta, h->st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->st);  // host vector bt must outlive the copy
  if (e != cudaSuccess) {
    delete h;
    return SF_ERR_CUDA;
  }
  *out = h;
  return SF_OK;
}

sf_status sf_debug_set_block_table(sf_handle* h, const int32_t* table_host, int32_t B, int32_t n_pages_per_seq) {
  if (!h || !table_host) return SF_ERR_ARG;
  if (h->state != ST_INIT) return set_err(h, SF_ERR_STATE, "block table can only be set before prefill");
  if (h->p.pool) return set_err(h, SF_ERR_UNSUPPORTED, "the page pool owns the block table");
  if (B != h->p.B || n_pages_per_seq != h->p.pps) return set_err(h, SF_ERR_SHAPE, "block table shape");
  std::vector<char> seen(h->p.n_pages, 0);
  for (int i = 0; i < B * n_pages_per_seq; ++i) {
    const int v = table_host[i];
    if (v < 0 || v >= h->p.n_pages || seen[v]) return set_err(h, SF_ERR_ARG, "block table not a permutation");
    seen[v] = 1;
  }
  SF_TRY(cudaMemcpyAsync(h->bt, table_host, (size_t)B * n_pages_per_seq * 4, cudaMemcpyHostToDevice, h->st));
  SF_TRY(cudaStreamSynchronize(h->st));
  return SF_OK;
}

sf_status specformer_prefill(sf_handle* h, const int32_t* tokens, int32_t B, int32_t P, int32_t* first_token) {
  if (!h || !tokens) return SF_ERR_ARG;
  if (B < 1 || B > h->p.B) return set_err(h, SF_ERR_SHAPE, "batch out of range");
  if (P < 1) return set_err(h, SF_ERR_SHAPE, "empty prompt");
  if (P + h->p.k + 1 > h->c.max_seq) return set_err(h, SF_ERR_CAPACITY, "prompt exceeds max_seq");
  h->launches = 0;
  if (h->gexec && h->g_B != B) {  // the cached step graph was captured for another batch size
    SF_TRY(cudaStreamSynchronize(h->st));
    cudaGraphExecDestroy(h->gexec);
    h->gexec = nullptr;
  }
  h->B = B;
  const Plan& p = h->p;
  SF_TRY(cudaMemcpyAsync(h->prompt, tokens, (size_t)B * P * 4, cudaMemcpyDefault, h->st));
  SF_TRY(cudaMemsetAsync(h->err, 0, 4, h->st));
  if (p.pool) {  // a new batch: every page back to the pool, then the prompts' pages (+ the first verify block)
    SF_TRY(launch_page_reset(p.n_pages, p.B, h->pp, h->st));
    SF_TRY(launch_page_take(0, B, nullptr, P + p.k + 1, h->pp, h->st));
    std::fill(h->released.begin(), h->released.end(), 0);
  }
  if (h->tpkey) SF_TRY(cudaMemsetAsync(h->tpkey, 0, (size_t)p.n_amrows * 8, h->st));
  // chunk rows per sequence for THIS batch (one 512-row GEMM pass per chunk; a handle sized for a large
  // batch prefills a small one in few chunks), within the plan's row capacity
  static const int pf_cap = getenv("SF_PF_CAP") ? atoi(getenv("SF_PF_CAP")) : 512;
  // Sequence groups: Bg sequences per pass with as many rows each as a 512-row pass holds (P = 512: one
  // sequence per pass), so each pass's attention reads one group's KV prefix (L2-resident) instead of
  // every sequence's. The same rows, positions and weight passes as chunking all B sequences together
  // (every row's arithmetic is independent of the block it runs in, C23): the same bits.
  const char* env_g = getenv("SF_PF_GROUP");  // (read per call: tests compare both)
  const bool grouped = !env_g || atoi(env_g) != 0;
  const int Bg = grouped ? std::max(1, std::min(B, std::max(1, std::min(pf_cap, p.R) / std::max(1, P)))) : B;
  const int C = std::max(p.k + 1, std::min(std::min(pf_cap, std::max(1, 512 / Bg)), p.R / Bg));
  int* bt_all = h->bt;
  for (int b0 = 0; b0 < B; b0 += Bg) {
    const int nb = std::min(Bg, B - b0);
    h->bt = bt_all + (size_t)b0 * p.pps;  // the group's page-table rows as rows 0 .. nb - 1
    int Cc = 0;
    cudaError_t e = cudaSuccess;
    for (int c0 = 0; c0 < P && e == cudaSuccess; c0 += C) {
      Cc = std::min(C, P - c0);
      e = launch_build_prefill_rows(nb, P, c0, Cc, h->prompt + (size_t)b0 * P, h->tok_rows, h->pos0_pf, h->st);
      if (e == cudaSuccess) e = base_forward(h, nb * Cc, Cc, h->pos0_pf, c0 + Cc, /*final_norm=*/false);
      if (e == cudaSuccess && p.k > 0) e = ctx_forward(h, nb * Cc, Cc, h->pos0_pf, c0 + Cc);
    }
    h->bt = bt_all;
    SF_TRY(e);
    // last prompt row per sequence: I_D row (draft input) and the final hidden state (LM head -> g0)
    if (p.k > 0) SF_TRY(launch_gather_rows(h->ctx, Cc, nullptr, Cc - 1, nb, p.d, h->idrow + (size_t)b0 * p.d, h->st));
    SF_TRY(launch_gather_rows(h->resid, Cc, nullptr, Cc - 1, nb, p.d, h->hlast + (size_t)b0 * p.d, h->st));
  }
  SF_TRY(head_argmax(h, h->hlast, B, h->logits, h->g_pf));
  SF_TRY(launch_prefill_finish(B, P, h->g_pf, h->seq_len, h->n_prev, h->last_token, h->r_b, h->prompt_len, nullptr,
                               h->st));
  SF_TRY(copy_out(h, first_token, h->g_pf, (size_t)B * 4));
  h->ctx_pending = false;
  h->host_len_hi = P;
  h->state = ST_READY;
  return SF_OK;
}

sf_status specformer_draft_step(sf_handle* h, int32_t* draft, float* draft_logits) {
  if (!h) return SF_ERR_ARG;
  if (h->p.k == 0) return set_err(h, SF_ERR_UNSUPPORTED, "draft_len == 0 (AR mode) has no draft head");
  if (h->state != ST_READY) return set_err(h, SF_ERR_STATE, "draft_step needs prefill or accept_commit first");
  if (any_released(h)) return set_err(h, SF_ERR_STATE, "a released slot must be re-filled (specformer_prefill_slot)");
  if (draft_logits && (h->c.flags & SF_FLAG_NO_LOGITS))
    return set_err(h, SF_ERR_STATE, "logits not kept (SF_FLAG_NO_LOGITS)");
  if ((h->c.flags & SF_FLAG_DRAFT_PREFIX) && h->host_len_hi + h->p.k > h->c.max_seq) {
    // the BIDIR_PREFIX slots occupy positions seq_len .. seq_len + k - 1 of the context layer's pages
    std::vector<int> sl(h->B);
    SF_TRY(cudaMemcpyAsync(sl.data(), h->seq_len, (size_t)h->B * 4, cudaMemcpyDeviceToHost, h->st));
    SF_TRY(cudaStreamSynchronize(h->st));
    h->host_len_hi = *std::max_element(sl.begin(), sl.end());
    if (h->host_len_hi + h->p.k > h->c.max_seq) return set_err(h, SF_ERR_CAPACITY, "seq_len + k > max_seq");
  }
  h->launches = 0;
  SF_TRY(do_draft(h));
  SF_TRY(copy_out(h, draft, h->draft, (size_t)h->B * h->p.k * 4));
  SF_TRY(copy_out(h, draft_logits, h->dlogits, (size_t)h->B * h->p.k * h->p.V * 4));
  h->state = ST_DRAFTED;
  return SF_OK;
}

sf_status specformer_verify_step(sf_handle* h, const int32_t* draft_in, int32_t* greedy, float* logits) {
  if (!h) return SF_ERR_ARG;
  const int k = h->p.k;
  if (logits && (h->c.flags & SF_FLAG_NO_LOGITS)) return set_err(h, SF_ERR_STATE, "logits not kept (SF_FLAG_NO_LOGITS)");
  const bool ok_state = h->state == ST_DRAFTED || (h->state == ST_READY && (k == 0 || draft_in));
  if (!ok_state) return set_err(h, SF_ERR_STATE, "verify_step needs a draft (draft_step or draft_in)");
  if (any_released(h)) return set_err(h, SF_ERR_STATE, "a released slot must be re-filled (specformer_prefill_slot)");
  if (h->host_len_hi + k + 1 > h->c.max_seq) {
    // refresh the host bound from the device lengths before failing
    std::vector<int> sl(h->B);
    SF_TRY(cudaMemcpyAsync(sl.data(), h->seq_len, (size_t)h->B * 4, cudaMemcpyDeviceToHost, h->st));
    SF_TRY(cudaStreamSynchronize(h->st));
    h->host_len_hi = *std::max_element(sl.begin(), sl.end());
    if (h->host_len_hi + k + 1 > h->c.max_seq) return set_err(h, SF_ERR_CAPACITY, "seq_len + k + 1 > max_seq");
  }
  if (h->state == ST_READY && k > 0 && h->ctx_pending) {
    // forced draft without a draft step: the context layer still has to see the previous rows
    h->launches = 0;
    SF_TRY(ctx_forward(h, h->B * (k + 1), k + 1, h->n_prev, h->c.max_seq));
    SF_TRY(launch_gather_rows(h->ctx, k + 1, h->r_b, 0, h->B, h->p.d, h->idrow, h->st));
    h->ctx_pending = false;
  } else if (h->state != ST_READY) {
    h->launches = 0;
  } else {
    h->launches = 0;
  }
  if (draft_in && k > 0) SF_TRY(cudaMemcpyAsync(h->draft, draft_in, (size_t)h->B * k * 4, cudaMemcpyDefault, h->st));
  SF_TRY(do_verify(h));
  SF_TRY(copy_out(h, greedy, h->greedy, (size_t)h->B * (k + 1) * 4));
  SF_TRY(copy_out(h, logits, h->logits, (size_t)h->B * (k + 1) * h->p.V * 4));
  h->state = ST_VERIFIED;
  return SF_OK;
}

sf_status specformer_accept_commit(sf_handle* h, int32_t* accept_len, int32_t* emitted, int32_t* seq_len) {
  if (!h) return SF_ERR_ARG;
  if (h->state != ST_VERIFIED) return set_err(h, SF_ERR_STATE, "accept_commit needs verify_step first");
  SF_TRY(do_accept(h, nullptr, nullptr));
  const int k = h->p.k;
  SF_TRY(copy_out(h, accept_len, h->accept_len, (size_t)h->B * 4));
  SF_TRY(copy_out(h, emitted, h->emitted, (size_t)h->B * (k + 1) * 4));
  SF_TRY(copy_out(h, seq_len, h->seq_len, (size_t)h->B * 4));
  h->host_len_hi += k + 1;
  h->state = ST_READY;
  return SF_OK;
}

sf_status specformer_release(sf_handle* h, int32_t slot) {
  if (!h) return SF_ERR_ARG;
  if (!h->p.pool) return set_err(h, SF_ERR_UNSUPPORTED, "specformer_release needs SF_FLAG_PAGE_POOL");
  if (h->state != ST_READY) return set_err(h, SF_ERR_STATE, "release needs prefill or accept_commit first");
  if (slot < 0 || slot >= h->B) return set_err(h, SF_ERR_SHAPE, "slot out of range");
  if (h->released[slot]) return SF_OK;
  SF_TRY(launch_page_release(slot, 1, h->pp, h->st));
  h->released[slot] = 1;
  return SF_OK;
}

sf_status specformer_prefill_slot(sf_handle* h, int32_t slot, const int32_t* tokens, int32_t P, int32_t* first_token) {
  if (!h || !tokens) return SF_ERR_ARG;
  const Plan& p = h->p;
  if (!p.pool) return set_err(h, SF_ERR_UNSUPPORTED, "specformer_prefill_slot needs SF_FLAG_PAGE_POOL");
  if (h->state != ST_READY || h->B == 0) return set_err(h, SF_ERR_STATE, "prefill_slot needs a batch prefill first");
  if (slot < 0 || slot >= h->B) return set_err(h, SF_ERR_SHAPE, "slot out of range");
  if (P < 1) return set_err(h, SF_ERR_SHAPE, "empty prompt");
  if (P + p.k + 1 > h->c.max_seq) return set_err(h, SF_ERR_CAPACITY, "prompt exceeds max_seq");
  h->launches = 0;
  if (!h->released[slot]) SF_TRY(launch_page_release(slot, 1, h->pp, h->st));
  if (p.k > 0 && h->ctx_pending) {
    // the other sequences' pending context pass (over the last verify's rows) runs first: the slot's
    // prefill reuses the activation buffers
    SF_TRY(ctx_forward(h, h->B * (p.k + 1), p.k + 1, h->n_prev, h->c.max_seq));
    SF_TRY(launch_gather_rows(h->ctx, p.k + 1, h->r_b, 0, h->B, p.d, h->idrow, h->st));
    h->ctx_pending = false;
  }
  SF_TRY(cudaMemcpyAsync(h->prompt, tokens, (size_t)P * 4, cudaMemcpyDefault, h->st));
  SF_TRY(launch_page_take(slot, 1, nullptr, P + p.k + 1, h->pp, h->st));
  // the one-sequence prefill sees the slot's page-table row as row 0 (chunks of up to R rows)
  int* bt_all = h->bt;
  h->bt = bt_all + (size_t)slot * p.pps;
  const int C = std::min(p.R, std::max(p.C_pf, 1) * std::max(1, p.B));
  int Cc = 0;
  cudaError_t e = cudaSuccess;
  for (int c0 = 0; c0 < P && e == cudaSuccess; c0 += C) {
    Cc = std::min(C, P - c0);
    e = launch_build_prefill_rows(1, P, c0, Cc, h->prompt, h->tok_rows, h->pos0_pf, h->st);
    if (e == cudaSuccess) e = base_forward(h, Cc, Cc, h->pos0_pf, c0 + Cc, /*final_norm=*/false);
    if (e == cudaSuccess && p.k > 0) e = ctx_forward(h, Cc, Cc, h->pos0_pf, c0 + Cc);
  }
  h->bt = bt_all;
  SF_TRY(e);
  if (p.k > 0) SF_TRY(launch_gather_rows(h->ctx, Cc, nullptr, Cc - 1, 1, p.d, h->idrow + (size_t)slot * p.d, h->st));
  SF_TRY(launch_gather_rows(h->resid, Cc, nullptr, Cc - 1, 1, p.d, h->hlast, h->st));
  SF_TRY(head_argmax(h, h->hlast, 1, h->logits, h->g_pf + slot));
  SF_TRY(launch_prefill_finish(1, P, h->g_pf + slot, h->seq_len + slot, h->n_prev + slot, h->last_token + slot,
                               h->r_b + slot, h->prompt_len + slot, nullptr, h->st));
  SF_TRY(copy_out(h, first_token, h->g_pf + slot, 4));
  h->released[slot] = 0;
  h->host_len_hi = std::max<int64_t>(h->host_len_hi, P);
  return SF_OK;
}

static cudaError_t one_step(sf_handle* h, int* acc_log, int* em_log) {
  cudaError_t e;
  if (h->p.k > 0) {
    if ((e = do_draft(h))) return e;
    if (h->forced) {
      h->launches++;
      if ((e = launch_force_drafts(h->B, h->p.k, h->p.V_full, h->f_cont, h->f_cont_len, h->f_corrupt,
                                   h->f_corrupt_steps, h->seq_len, h->prompt_len, h->step_counter, h->draft, h->st)))
        return e;
    }
  }
  if ((e = do_verify(h))) return e;
  return do_accept(h, acc_log, em_log);
}

sf_status specformer_decode_steps(sf_handle* h, int32_t n_steps, int32_t* emitted_log, int32_t* accept_log) {
  if (!h) return SF_ERR_ARG;
  if (n_steps < 0) return SF_ERR_ARG;
  if (h->state != ST_READY) return set_err(h, SF_ERR_STATE, "decode_steps needs prefill or accept_commit first");
  if (any_released(h)) return set_err(h, SF_ERR_STATE, "a released slot must be re-filled (specformer_prefill_slot)");
  const int k = h->p.k;
  if (h->host_len_hi + (int64_t)n_steps * (k + 1) > h->c.max_seq) {
    std::vector<int> sl(h->B);
    SF_TRY(cudaMemcpyAsync(sl.data(), h->seq_len, (size_t)h->B * 4, cudaMemcpyDeviceToHost, h->st));
    SF_TRY(cudaStreamSynchronize(h->st));
    h->host_len_hi = *std::max_element(sl.begin(), sl.end());
    if (h->host_len_hi + (int64_t)n_steps * (k + 1) > h->c.max_seq)
      return set_err(h, SF_ERR_CAPACITY, "decode_steps could exceed max_seq");
  }
  h->launches = 0;
  SF_TRY(cudaMemsetAsync(h->step_counter, 0, 4, h->st));
  if (accept_log || emitted_log) SF_TRY(launch_fill(h->d_logcap, 1, n_steps, h->st));  // logs hold n_steps rows
  int done = 0;
  if (k > 0 && !h->ctx_pending && n_steps > 0) {  // first step after prefill: no context pass
    SF_TRY(one_step(h, accept_log, emitted_log));
    done = 1;
  }
  const bool use_graph = (h->c.flags & SF_FLAG_CUDA_GRAPH) != 0 && (h->p.tp == 1 || h->coll.graph_safe);
  if (use_graph && h->prof_on && done < n_steps) {
    // profiling: the step graph re-captured with an event-record node around every launch (this
    // serialises the launches -- no PDL overlap across a record node), replayed one step at a time
    // with each replay's per-launch times accumulated per kernel class
    cudaGraph_t g;
    cudaGraphExec_t ge = nullptr;
    const size_t r0 = h->prof.size();
    const int64_t before = h->launches;
    h->prof_capture = true;
    SF_TRY(cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal));
    cudaError_t e = one_step(h, accept_log, emitted_log);
    cudaError_t e2 = cudaStreamEndCapture(h->st, &g);
    h->prof_capture = false;
    if (e != cudaSuccess || e2 != cudaSuccess) {
      h->err_msg = std::string("profiling graph capture failed: ") + cudaGetErrorString(e != cudaSuccess ? e : e2);
      return SF_ERR_CUDA;
    }
    SF_TRY(cudaGraphInstantiate(&ge, g, 0));
    cudaGraphDestroy(g);
    const int64_t per_step = h->launches - before;
    h->launches = before;
    std::vector<sf_handle::Prof> recs(h->prof.begin() + r0, h->prof.end());
    h->prof.resize(r0);
    for (int s = done; s < n_steps; ++s) {
      SF_TRY(cudaGraphLaunch(ge, h->st));
      SF_TRY(cudaStreamSynchronize(h->st));
      h->launches += per_step;
      for (auto& r : recs) {
        float t = 0;
        SF_TRY(cudaEventElapsedTime(&t, r.a, r.b));
        h->prof_ms[r.cls] += t;
        h->prof_bytes[r.cls] += r.bytes;
        h->prof_n[r.cls] += 1;
      }
    }
    cudaGraphExecDestroy(ge);
    for (auto& r : recs) {
      h->ev_free.push_back(r.a);
      h->ev_free.push_back(r.b);
    }
    h->ctx_pending = k > 0;
  } else if (use_graph && done < n_steps) {
    // the graph depends on the log pointers only (the log capacity is read on the device)
    if (h->gexec && (h->g_acc_log != accept_log || h->g_em_log != emitted_log || h->g_B != h->B)) {
      cudaGraphExecDestroy(h->gexec);
      h->gexec = nullptr;
    }
    if (!h->gexec) {
      cudaGraph_t g;
      const int64_t before = h->launches;
      SF_TRY(cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal));
      cudaError_t e = one_step(h, accept_log, emitted_log);
      cudaError_t e2 = cudaStreamEndCapture(h->st, &g);
      if (e != cudaSuccess || e2 != cudaSuccess) {
        h->err_msg = std::string("graph capture failed: ") + cudaGetErrorString(e != cudaSuccess ? e : e2);
        return SF_ERR_CUDA;
      }
      SF_TRY(cudaGraphInstantiate(&h->gexec, g, 0));
      cudaGraphDestroy(g);
      h->graph_launches = h->launches - before;
      h->launches = before;
      h->g_acc_log = accept_log;
      h->g_em_log = emitted_log;
      h->g_B = h->B;
    }
    for (int s = done; s < n_steps; ++s) {
      SF_TRY(cudaGraphLaunch(h->gexec, h->st));
      h->launches += h->graph_launches;
    }
    h->ctx_pending = k > 0;
  } else {
    for (int s = done; s < n_steps; ++s) SF_TRY(one_step(h, accept_log, emitted_log));
  }
  h->host_len_hi += (int64_t)n_steps * (k + 1);
  h->state = ST_READY;
  return SF_OK;
}

sf_status specformer_sync(sf_handle* h) {
  if (!h) return SF_ERR_ARG;
  SF_TRY(cudaStreamSynchronize(h->st));
  int err = 0;
  SF_TRY(cudaMemcpy(&err, h->err, 4, cudaMemcpyDeviceToHost));
  if (err & 1) return set_err(h, SF_ERR_NONFINITE, "non-finite logits");
  if (err & 2) return set_err(h, SF_ERR_CAPACITY, "KV page pool exhausted");
  if (err & 4) return set_err(h, SF_ERR_NCCL, "tensor-parallel exchange: a peer's epoch flag did not arrive within 5 s");
#ifdef SF_WITH_NCCL
  if (h->nccl_comm) {  // asynchronous communicator errors (a peer failed, a network / NVLink error)
    ncclResult_t ar = ncclSuccess;
    const ncclResult_t r = ncclCommGetAsyncError((ncclComm_t)h->nccl_comm, &ar);
    if (r != ncclSuccess || ar != ncclSuccess)
      return set_err(h, SF_ERR_NCCL, std::string("NCCL async error: ") + ncclGetErrorString(r != ncclSuccess ? r : ar));
  }
#endif
  return SF_OK;
}

const char* specformer_last_error(const sf_handle* h) { return h ? h->err_msg.c_str() : "null handle"; }

void specformer_destroy(sf_handle* h) {
  if (!h) return;
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  for (auto& r : h->prof) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : h->ev_free) cudaEventDestroy(e);
#ifdef SF_WITH_NCCL
  if (h->nccl_comm) ncclCommDestroy((ncclComm_t)h->nccl_comm);
#endif
  if (h->coll.sum_f32 == local_sum_f32) delete (LocalCtx*)h->coll.ctx;
  for (int q = 0; q < kTpMax; ++q)
    if (h->xopened[q]) cudaIpcCloseMemHandle(h->xpeer[q]);
  if (h->xch) cudaFree(h->xch);
  delete h;
}

int32_t sf_nccl_unique_id(uint8_t* out) {
#ifdef SF_WITH_NCCL
  if (!out) return -1;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return -1;
  static_assert(sizeof(id.internal) == 128, "ncclUniqueId is 128 bytes");
  memcpy(out, id.internal, 128);
  return 0;
#else
  (void)out;
  return -1;
#endif
}

sf_status sf_nccl_attach(sf_handle* h, const uint8_t* id, int32_t nranks, int32_t rank) {
  if (!h || !id) return SF_ERR_ARG;
  if (nranks != h->p.tp || rank != h->p.tp_rank) return set_err(h, SF_ERR_ARG, "nranks / rank differ from tp_size / tp_rank");
  if (h->coll.sum_f32) return set_err(h, SF_ERR_STATE, "a collective is already attached");
#ifdef SF_WITH_NCCL
  ncclUniqueId uid;
  memcpy(uid.internal, id, 128);
  ncclComm_t comm = nullptr;
  const ncclResult_t r = ncclCommInitRank(&comm, nranks, uid, rank);
  if (r != ncclSuccess) return set_err(h, SF_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  h->nccl_comm = comm;
  h->coll.sum_f32 = nccl_sum_f32;
  h->coll.sum_bf16 = nccl_sum_bf16;
  h->coll.max_u64 = nccl_max_u64;
  h->coll.ctx = comm;
  h->coll.graph_safe = true;
  return SF_OK;
#else
  return set_err(h, SF_ERR_UNSUPPORTED, "built without NCCL");
#endif
}

sf_local_group* sf_local_group_create(int32_t n) {
  if (n < 1 || n > 8) return nullptr;
  sf_local_group* g = new sf_local_group();
  g->n = n;
  g->bufs.assign(n, nullptr);
  g->tmp.assign(n, nullptr);
  g->tmp_bytes.assign(n, 0);
  g->ev_in.resize(n);
  g->ev_mid.resize(n);
  g->ev_x.resize(n);
  g->xch.assign(n, nullptr);
  for (int i = 0; i < n; ++i) {
    cudaEventCreateWithFlags(&g->ev_in[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&g->ev_mid[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&g->ev_x[i], cudaEventDisableTiming);
  }
  return g;
}

void sf_local_group_destroy(sf_local_group* g) {
  if (!g) return;
  cudaDeviceSynchronize();
  for (int i = 0; i < g->n; ++i) {
    cudaEventDestroy(g->ev_in[i]);
    cudaEventDestroy(g->ev_mid[i]);
    cudaEventDestroy(g->ev_x[i]);
    if (g->tmp[i]) cudaFree(g->tmp[i]);
  }
  delete g;
}

sf_status sf_local_group_attach(sf_handle* h, sf_local_group* g, int32_t rank) {
  if (!h || !g) return SF_ERR_ARG;
  if (g->n != h->p.tp || rank != h->p.tp_rank) return set_err(h, SF_ERR_ARG, "group size / rank differ from tp_size / tp_rank");
  if (h->coll.sum_f32) return set_err(h, SF_ERR_STATE, "a collective is already attached");
  h->coll.sum_f32 = local_sum_f32;
  h->coll.sum_bf16 = local_sum_bf16;
  h->coll.max_u64 = local_max_u64;
  h->coll.ctx = new LocalCtx{g, rank};
  h->coll.graph_safe = false;
  return SF_OK;
}

// ---- NEXT-3: the fused TP all-reduce's exchange regions
static sf_status xch_alloc(sf_handle* h) {
  if (h->p.tp < 2 || h->p.tp > kTpMax) return set_err(h, SF_ERR_STATE, "exchange regions need 2 <= tp_size <= 8");
  if (!h->bf) return set_err(h, SF_ERR_UNSUPPORTED, "the fused TP all-reduce is bf16 only");
  if (h->state != ST_INIT) return set_err(h, SF_ERR_STATE, "attach the exchange before the first prefill");
  if (h->xch) return SF_OK;
  const size_t bytes = kXchHead + (size_t)2 * h->p.R * h->p.d * 2;
  void* x = nullptr;
  SF_TRY(cudaMalloc(&x, bytes));
  SF_TRY(cudaMemset(x, 0, bytes));
  SF_TRY(cudaDeviceSynchronize());
  h->xch = (char*)x;
  h->xch_bytes = bytes;
  return SF_OK;
}

sf_status sf_tp_xch_handle(sf_handle* h, uint8_t* out_64) {
  if (!h || !out_64) return SF_ERR_ARG;
  const sf_status s = xch_alloc(h);
  if (s != SF_OK) return s;
  cudaIpcMemHandle_t ih;
  static_assert(sizeof(ih) == 64, "cudaIpcMemHandle_t is 64 bytes");
  SF_TRY(cudaIpcGetMemHandle(&ih, h->xch));
  memcpy(out_64, &ih, 64);
  return SF_OK;
}

sf_status sf_tp_xch_attach(sf_handle* h, const uint8_t* handles) {
  if (!h || !handles) return SF_ERR_ARG;
  if (h->xmode) return set_err(h, SF_ERR_STATE, "an exchange is already attached");
  const sf_status s = xch_alloc(h);
  if (s != SF_OK) return s;
  const int tp = h->p.tp, r = h->p.tp_rank;
  for (int q = 0; q < tp; ++q) {
    if (q == r) {
      h->xpeer[q] = h->xch;
      continue;
    }
    cudaIpcMemHandle_t ih;
    memcpy(&ih, handles + 64 * q, 64);
    void* ptr = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&ptr, ih, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      for (int j = 0; j < q; ++j)
        if (h->xopened[j]) cudaIpcCloseMemHandle(h->xpeer[j]), h->xopened[j] = false, h->xpeer[j] = nullptr;
      return set_err(h, SF_ERR_CUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
    }
    h->xpeer[q] = (char*)ptr;
    h->xopened[q] = true;
  }
  h->xmode = 1;
  return SF_OK;
}

sf_status sf_local_group_xch_attach(sf_handle* h, sf_local_group* g) {
  if (!h || !g) return SF_ERR_ARG;
  if (h->coll.sum_f32 != local_sum_f32 || ((LocalCtx*)h->coll.ctx)->g != g)
    return set_err(h, SF_ERR_STATE, "attach the local group (sf_local_group_attach) first");
  if (h->xmode) return set_err(h, SF_ERR_STATE, "an exchange is already attached");
  const sf_status s = xch_alloc(h);
  if (s != SF_OK) return s;
  g->xch[h->p.tp_rank] = h->xch;
  g->barrier();  // every rank's region registered
  for (int q = 0; q < g->n; ++q) h->xpeer[q] = g->xch[q];
  g->barrier();
  h->xgroup = g;
  h->xmode = 2;
  return SF_OK;
}

int64_t specformer_kernel_launches(const sf_handle* h) { return h ? h->launches : -1; }

sf_status sf_debug_capture(sf_handle* h, int32_t what, void* dst, int64_t* nbytes) {
  if (!h || !dst) return SF_ERR_ARG;
  const Plan& p = h->p;
  const int B = h->B, k = p.k;
  const void* src = nullptr;
  size_t bytes = 0;
  switch (what) {
    case 0: {  // taps [4, B(k+1), d]
      for (int g = 0; g < 4; ++g)
        SF_TRY(cudaMemcpyAsync((char*)dst + (size_t)g * B * (k + 1) * p.d * 4, h->taps + (size_t)g * p.R * p.d,
                               (size_t)B * (k + 1) * p.d * 4, cudaMemcpyDefault, h->st));
      bytes = (size_t)4 * B * (k + 1) * p.d * 4;
      break;
    }
    case 1: src = h->idrow; bytes = (size_t)B * p.d * 4; break;
    case 2: src = h->D; bytes = (size_t)B * k * p.d * 4; break;
    case 3: src = h->seq_len; bytes = (size_t)B * 4; break;
    case 4: src = h->last_token; bytes = (size_t)B * 4; break;
    case 5: src = h->n_prev; bytes = (size_t)B * 4; break;
    case 6: {  // taps of every row of the last base forward [4, fwd_rows, d]
      const int R = h->fwd_rows;
      for (int g = 0; g < 4; ++g)
        SF_TRY(cudaMemcpyAsync((char*)dst + (size_t)g * R * p.d * 4, h->taps + (size_t)g * p.R * p.d,
                               (size_t)R * p.d * 4, cudaMemcpyDefault, h->st));
      bytes = (size_t)4 * R * p.d * 4;
      break;
    }
    case 7: src = h->ctx; bytes = (size_t)h->ctx_rows * p.d * 4; break;
    case 8: src = h->prompt_len; bytes = (size_t)B * 4; break;
    case 9: src = h->seqsync; bytes = h->seqsync ? (size_t)p.L * kSeqSyncInts * 4 : 0; break;  // layer_seq sync blocks
    default: return set_err(h, SF_ERR_ARG, "unknown capture id");
  }
  if (src) SF_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, h->st));
  SF_TRY(cudaStreamSynchronize(h->st));
  if (nbytes) *nbytes = (int64_t)bytes;
  return SF_OK;
}

sf_status sf_debug_force_drafts(sf_handle* h, const int32_t* cont_dev, int32_t cont_len, const int32_t* corrupt_dev) {
  if (!h || !cont_dev || cont_len < 1) return SF_ERR_ARG;
  if (h->state != ST_DRAFTED && h->state != ST_READY) return set_err(h, SF_ERR_STATE, "force_drafts before verify");
  SF_TRY(launch_force_drafts(h->B, h->p.k, h->p.V_full, cont_dev, cont_len, corrupt_dev, 1, h->seq_len, h->prompt_len,
                             nullptr, h->draft, h->st));
  h->state = ST_DRAFTED;
  return SF_OK;
}

sf_status sf_set_forced_drafts(sf_handle* h, const int32_t* cont_dev, int32_t cont_len, const int32_t* corrupt_dev,
                               int32_t corrupt_steps) {
  if (!h) return SF_ERR_ARG;
  if (h->gexec) {
    cudaGraphExecDestroy(h->gexec);
    h->gexec = nullptr;
  }
  h->forced = cont_dev != nullptr;
  h->f_cont = cont_dev;
  h->f_cont_len = cont_len;
  h->f_corrupt = corrupt_dev;
  h->f_corrupt_steps = std::max(1, corrupt_steps);
  return SF_OK;
}

sf_status sf_profile(sf_handle* h, int32_t enable) {
  if (!h) return SF_ERR_ARG;
  SF_TRY(cudaStreamSynchronize(h->st));
  for (auto& r : h->prof) {
    h->ev_free.push_back(r.a);
    h->ev_free.push_back(r.b);
  }
  h->prof.clear();
  for (int c = 0; c < 4; ++c) h->prof_ms[c] = h->prof_bytes[c] = 0, h->prof_n[c] = 0;
  h->prof_on = enable != 0;
  return SF_OK;
}

sf_status sf_profile_read(sf_handle* h, int32_t cls, double* total_ms, int64_t* count, double* bytes) {
  if (!h || !total_ms || !count || !bytes) return SF_ERR_ARG;
  SF_TRY(cudaStreamSynchronize(h->st));
  if (cls < 0 || cls > 3) return SF_ERR_ARG;
  double ms = h->prof_ms[cls], by = h->prof_bytes[cls];
  int64_t n = h->prof_n[cls];
  for (auto& r : h->prof) {
    if (r.cls != cls) continue;
    float t = 0;
    SF_TRY(cudaEventElapsedTime(&t, r.a, r.b));
    ms += t;
    by += r.bytes;
    ++n;
  }
  *total_ms = ms;
  *count = n;
  *bytes = by;
  return SF_OK;
}

int32_t sf_debug_ktrace_enable(int32_t on) { return kt_set(on != 0) ? 0 : -1; }

int32_t sf_debug_ktrace(void* dst_host, int32_t cap) {
  if (!kt_enable() || !dst_host || cap <= 0) return 0;
  cudaDeviceSynchronize();
  unsigned n = 0;
  cudaMemcpy(&n, g_kt_cnt, 4, cudaMemcpyDeviceToHost);
  n = std::min<unsigned>(std::min<unsigned>(n, kKtCap), (unsigned)cap);
  cudaMemcpy(dst_host, g_kt_rec, (size_t)n * kKtRecBytes, cudaMemcpyDeviceToHost);
  cudaMemset(g_kt_cnt, 0, 4);
  return (int32_t)n;
}

int32_t sf_debug_gemm_trace(uint64_t* dst_host, int32_t cap) {
  if (!dst_host || cap <= 0) return 0;
  return gemm_trace_copy(reinterpret_cast<unsigned long long*>(dst_host), cap);
}

sf_status sf_test_gemm(int32_t dtype, const void* A, const void* W, float* out, int32_t T, int32_t N, int32_t K,
                       void* stream) {
  if (!A || !W || !out || T < 1 || N < 1 || K < 1) return SF_ERR_ARG;
  const bool pretiled = dtype == 2;  // bf16 W already in layout 1 (sf_pack_matrix)
  const bool bf = dtype == SF_BF16 || pretiled;
  cudaStream_t st = (cudaStream_t)stream;
  // test-only scratch, grown on demand and kept (flags stay zeroed: kernels re-arm them)
  static float* partial = nullptr;
  static int64_t partial_cap = 0;
  static int* counters = nullptr;
  static void* wt = nullptr;
  static int64_t wt_cap = 0;
  const int64_t pe = gemm_partial_elems(bf, std::min(T, 512), N, K);
  if (pe > partial_cap) {
    if (partial) cudaFree(partial);
    if (cudaMalloc((void**)&partial, pe * 4) != cudaSuccess) return SF_ERR_CUDA;
    partial_cap = pe;
  }
  if (!counters) {
    if (cudaMalloc((void**)&counters, 4096 * 4) != cudaSuccess) return SF_ERR_CUDA;
    cudaMemset(counters, 0, 4096 * 4);
  }
  const void* Wuse = W;
  if (bf && !pretiled) {  // the hot path stores bf16 weights tile-contiguous: pack into scratch
    const int64_t wb = (int64_t)N * K * 2;
    if (wb > wt_cap) {
      if (wt) cudaFree(wt);
      if (cudaMalloc(&wt, wb) != cudaSuccess) return SF_ERR_CUDA;
      wt_cap = wb;
    }
    if (gemm_pack_weight(W, wt, N, K, st) != cudaSuccess) return SF_ERR_ARG;
    Wuse = wt;
  }
  GemmScratch sc;
  sc.partial = partial;
  sc.partial_elems = partial_cap;
  sc.counters = counters;
  sc.n_counters = 4096;
  GemmEpi e;
  e.mode = EPI_STORE_F32;
  e.out = out;
  e.ldo = N;
  return gemm_launch(bf, A, K, Wuse, bf, T, N, K, e, sc, st) == cudaSuccess ? SF_OK : SF_ERR_CUDA;
}

sf_status sf_bench_gemm(int32_t impl, int32_t T, int32_t N, int32_t K, int32_t reps, float* ms_out) {
  // tools only: the GEMM main loop in isolation -- impl 0 the standalone EPI_PARTIAL launch, 1 the
  // same GEMM as a one-phase layer-sequence launch; random bf16 weights / activations
  if (T < 1 || N < 256 || K < 64 || reps < 1 || !ms_out) return SF_ERR_ARG;
  void *A = nullptr, *W = nullptr;
  float* part = nullptr;
  int *cnt = nullptr, *sync = nullptr;
  const int64_t pe = gemm_partial_elems(true, std::min(T, 512), N, K);
  if (cudaMalloc(&A, (size_t)T * K * 2) || cudaMalloc(&W, (size_t)N * K * 2) || cudaMalloc((void**)&part, pe * 4) ||
      cudaMalloc((void**)&cnt, 4096 * 4) || cudaMalloc((void**)&sync, kSeqSyncInts * 4))
    return SF_ERR_CUDA;
  cudaMemset(sync, 0, kSeqSyncInts * 4);
  cudaMemset(A, 0, (size_t)T * K * 2);
  cudaMemset(W, 0, (size_t)N * K * 2);
  cudaMemset(cnt, 0, 4096 * 4);
  GemmScratch sc;
  sc.partial = part;
  sc.partial_elems = pe;
  sc.counters = cnt;
  sc.n_counters = 2048;
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  SeqStep step;
  step.A = A, step.lda = K, step.W = W, step.N = N, step.K = K;
  step.epi.mode = EPI_PARTIAL;
  GemmEpi e;
  e.mode = EPI_PARTIAL;
  cudaError_t err = cudaSuccess;
  for (int r = -2; r < reps; ++r) {
    if (r == 0) cudaEventRecord(e0, st);
    err = impl == 0 ? gemm_launch(true, A, K, W, true, T, N, K, e, sc, st) : gemm_seq_launch(T, &step, 1, sc, sync, st);
    if (err != cudaSuccess) break;
  }
  cudaEventRecord(e1, st);
  cudaStreamSynchronize(st);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  *ms_out = ms / reps;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(st);
  cudaFree(A);
  cudaFree(W);
  cudaFree(part);
  cudaFree(cnt);
  cudaFree(sync);
  return err == cudaSuccess ? SF_OK : SF_ERR_CUDA;
}

sf_status sf_pack_matrix(int32_t dtype, const void* src_dev, void* dst_dev, int64_t N, int64_t K, void* stream) {
  if (!src_dev || !dst_dev || N < 1 || K < 1) return SF_ERR_ARG;
  if (dtype != SF_BF16) return SF_ERR_UNSUPPORTED;
  return gemm_pack_weight(src_dev, dst_dev, (int)N, (int)K, (cudaStream_t)stream) == cudaSuccess ? SF_OK : SF_ERR_SHAPE;
}

}  // extern "C"
