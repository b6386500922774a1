// kernels.cuh -- launchers for the non-GEMM kernels of the hot path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sf {

struct AttnParams {
  const float* q;            // [T, Hq, hd] rotated queries (fp32; bf16 for the bf16 hd=128 kernel)
  const void* Kp;            // paged K pool of one layer: [n_pages, Hkv, 16, hd]
  const void* Vp;            // paged V pool
  const int* block_table;    // [B, pages_per_seq]
  int pages_per_seq;
  const int* pos0;           // [B] absolute position of each sequence's first query row
  int q_len;                 // query rows per sequence (rows b*q_len + i at pos0[b] + i)
  int B, Hq, Hkv, hd;
  int nchunk_max;            // partial-buffer capacity in 128-key chunks
  float* part_o;             // [T, Hq, nchunk_max, 4, hd] (flash-decoding: per segment and warp slot)
  float* part_ml;            // [T, Hq, nchunk_max, 4, 2]
  void* out;                 // [T, Hq*hd] act dtype
  int max_key;               // upper bound of pos0[b] + q_len (grid sizing), <= max_seq
  int n_pages;               // pages in the pool (TMA tensor-map extent)
  int* seg_cnt;              // [B * Hkv * query tiles] zeroed arrival counters (bf16 hd=128 kernel)
  // 0: CAUSAL_PREFIX (row i of sequence b sees keys <= pos0[b] + i); 1: BIDIR_PREFIX (every row of
  // sequence b sees keys <= pos0[b] + q_len - 1: the whole prefix and all of the block's rows; the
  // NEXT-2 draft mask variant)
  int bidir_tail;
};
// last key position row qi of a sequence may see, relative to pos0
__host__ __device__ inline int attn_row_last(const AttnParams& p, int qi) { return p.bidir_tail ? p.q_len - 1 : qi; }

constexpr int kAttnChunk = 128;  // fixed absolute key-chunk size (split-KV boundaries, C23)
constexpr int kAttnSeg = 2048;   // flash-decoding key segment (fixed absolute bounds; defines the arithmetic)
constexpr int kAttnTileRows = 8; // bf16 flash-decoding query tile: (query, head) rows per work item
constexpr int kAttnWarps = 8;    // its compute warps: warp w owns keys [16 w, 16 w + 16) of every 128-key chunk

// act dtype: bf16 (is_bf16) or fp32.
cudaError_t launch_rope_table(float2* table, int max_seq, int hd, float theta, cudaStream_t s);
cudaError_t launch_build_verify_rows(int B, int k, const int* last_token, const int* draft, int* tok_rows,
                                     cudaStream_t s);
cudaError_t launch_build_prefill_rows(int B, int P, int c0, int C, const int* tokens, int* tok_rows, int* pos0,
                                      cudaStream_t s);
cudaError_t launch_embed(bool is_bf16, const int* tok, const void* embed, int T, int d, int vocab, float* resid,
                         float* tap0, cudaStream_t s);
cudaError_t launch_rmsnorm(bool is_bf16, const float* in, int in_ld, const float* gamma, float eps, int T, int d,
                           void* out, int out_ld, cudaStream_t s);
cudaError_t launch_group_rms(bool is_bf16, const float* taps, int64_t tap_stride, const float* scales, float eps,
                             int T, int d, void* out, cudaStream_t s);
// q_bf16: rotated queries written as bf16 (the flash-decoding attention's operand precision)
cudaError_t launch_rope_append(bool is_bf16, const void* qkv, int T, int q_len, const int* pos0,
                               const float2* rope, int Hq, int Hkv, int hd, const int* block_table,
                               int pages_per_seq, void* Kp, void* Vp, void* q_out, bool q_bf16, cudaStream_t s, bool pair_rows = true);
cudaError_t launch_attention(bool is_bf16, const AttnParams& p, cudaStream_t s);
cudaError_t launch_attention_fd(const AttnParams& p, cudaStream_t s);   // bf16, hd 128 (flash-decoding)
cudaError_t launch_bidir_attention(bool is_bf16, const void* qkv, int B, int k, int Hq, int Hkv, int hd,
                                   bool causal, void* out, cudaStream_t s);
// "-Pos" draft variant (NEXT-2): D[b k + j] = RMS(src[b]) * gamma + bias[j d .. (j+1) d) (fp32 rows)
cudaError_t launch_pos_broadcast(const float* src, const float* gamma, const float* bias, int B, int k, int d, float eps,
                                 float* D, cudaStream_t s);
cudaError_t launch_gather_rows(const float* src, int q_len, const int* idx, int const_idx, int B, int d,
                               float* dst, cudaStream_t s);
cudaError_t launch_argmax(const float* logits, int R, int V, float* pval, int* pidx, int* out, int* err,
                          cudaStream_t s);
// tensor parallelism: per-row packed (logit, v0 + id) keys of this vocabulary shard / their unpacking
cudaError_t launch_argmax_key(const float* logits, int R, int V, int v0, float* pval, int* pidx,
                              unsigned long long* keys, int* err, cudaStream_t s);
// (reset: zero the keys after reading them, for the next fused-argmax LM head)
cudaError_t launch_argmax_unkey(unsigned long long* keys, int R, int* out, cudaStream_t s, bool reset = false);
// tensor parallelism, tests (one process, several handles): out[i] = sum / max over the n buffers in
// buffer order
// tensor-parallel test group: out = reduction of n equal buffers (mode 0: fp32 sum, 1: u64 max, 2: bf16 sum)
cudaError_t launch_cvt_f32_bf16(float* f32, __nv_bfloat16* bf, int64_t n, bool to_bf, cudaStream_t s);
cudaError_t launch_reduce_bufs(const void* const* bufs, int n, int64_t count, int mode, void* out, cudaStream_t s);
// KV page pool (NEXT-4; csrc/kernels.cu): all pointers null = static per-sequence page ranges
struct PagePool {
  int* pool = nullptr;       // [n_pages] free page ids, a stack
  int* top = nullptr;        // [1] stack height
  int* alloc_cnt = nullptr;  // [B] pages held by each sequence (bt[b pps + i], i < alloc_cnt[b])
  int* bt = nullptr;         // [B, pps] page table
  int* err = nullptr;        // sticky error flags (bit 1: pool exhausted)
  int pps = 0;
};
cudaError_t launch_page_take(int b0, int nb, const int* seq_len, int extra, const PagePool& pp, cudaStream_t s);
cudaError_t launch_page_release(int b0, int nb, const PagePool& pp, cudaStream_t s);
cudaError_t launch_page_reset(int n_pages, int B, const PagePool& pp, cudaStream_t s);
cudaError_t launch_accept(int B, int k, const int* draft, const int* greedy, int* seq_len, int* n_prev,
                          int* last_token, int* r_b, int* accept_len, int* emitted, int* step_counter,
                          int* accept_log, int* emitted_log, const int* log_cap /* device */, const PagePool& pp, cudaStream_t s);
cudaError_t launch_force_drafts(int B, int k, int V, const int* cont, int cont_len, const int* corrupt,
                                int corrupt_steps, const int* seq_len, const int* prompt_len,
                                const int* step_counter, int* draft, cudaStream_t s);
cudaError_t launch_fill(int* p, int n, int v, cudaStream_t s);
cudaError_t launch_prefill_finish(int B, int P, const int* greedy, int* seq_len, int* n_prev, int* last_token,
                                  int* r_b, int* prompt_len, int* first_out, cudaStream_t s);

int argmax_splits(int V);

// kernel timeline (SF_KTRACE=1, tools only): point every translation unit's device log at rec/cnt
cudaError_t kt_setup_kernels(void* rec, unsigned* cnt, unsigned cap);
cudaError_t kt_setup_gemm(void* rec, unsigned* cnt, unsigned cap);
cudaError_t kt_setup_attn_fd(void* rec, unsigned* cnt, unsigned cap);
constexpr int kKtRecBytes = 40;

}  // namespace sf
