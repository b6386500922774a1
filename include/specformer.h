/*
 * specformer.h -- C ABI of the B200-native SpecFormer speculative-decoding hot path.
 *
 * The three calls mirror the paper's three-step SD protocol (PAPER.md P20-23, §Intro):
 *   specformer_draft_step   "Multi-token generation: based on information from the previous
 *                            forward pass, the model samples multiple draft tokens"
 *                            = SpecFormer context causal attention (Eq.8, P179-188), positional
 *                              FFN (Eq.9, P189-193), draft bi-directional layer (Eq.10,
 *                              P195-204), shared frozen LM head + argmax (reading C8).
 *   specformer_verify_step  "Multi-token verification: ... evaluates all draft tokens
 *                            simultaneously ... while also extracting and storing information
 *                            for the next round" = one base-decoder forward over
 *                            [last_token, d_1..d_k] that keeps the hook taps HS[0], HS[L/2],
 *                            HS[L-1], HS[L] (P175) of those k+1 rows in the workspace.
 *   specformer_accept_commit "Multi-token acceptance ... accordingly updates the contextual
 *                            information" = lossless greedy accept (P25: "only draft tokens
 *                            that exactly match the outputs of the large model") + KV commit;
 *                            rollback moves no data (rejected rows lie beyond seq_len).
 *
 * Conventions (DESIGN.md §3 lists every reading of the paper):
 *  - Tokens are int32. Matrices are row-major [out, in]; y = x W^T.
 *  - Pointers named *_dev are device pointers; pointers documented "dev or host" may be device
 *    memory or pinned host memory (they are moved with cudaMemcpyAsync(..., cudaMemcpyDefault)).
 *  - Ownership: the caller allocates ALL device memory (packed weights, workspace, I/O). The
 *    library never calls cudaMalloc/cudaFree on caller memory; it owns only host state and
 *    CUDA graph objects. Weights and workspace must outlive the handle.
 *  - All calls are asynchronous on the handle's stream; outputs are valid after the stream
 *    (or specformer_sync) completes. One host thread per handle.
 *  - Errors: argument / shape / state / capacity errors return synchronously and leave the
 *    handle unchanged. Device-detected errors (non-finite logits) are sticky flags surfaced by
 *    specformer_sync as SF_ERR_NONFINITE. specformer_last_error() describes the last failure.
 *  - There is no CPU fallback: every step runs in this library's sm_100a kernels.
 */
#ifndef SPECFORMER_H_
#define SPECFORMER_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SF_OK = 0,
  SF_ERR_ARG = 1,        /* bad argument value (e.g. eps <= 0, d % heads != 0, NULL handle) */
  SF_ERR_SHAPE = 2,      /* dimension mismatch (batch > max_batch, bad prompt length ...)    */
  SF_ERR_CAPACITY = 3,   /* seq_len + k + 1 would exceed max_seq                             */
  SF_ERR_STATE = 4,      /* call order violated: init -> prefill -> (draft -> verify -> accept)* */
  SF_ERR_CUDA = 5,       /* a CUDA runtime call failed                                       */
  SF_ERR_NCCL = 6,       /* NCCL communicator setup failed (tensor-parallel path)            */
  SF_ERR_NONFINITE = 7,  /* NaN/Inf met in logits (SPEC S26: an error condition)             */
  SF_ERR_UNSUPPORTED = 8 /* configuration not supported by this build                        */
} sf_status;

typedef enum { SF_FP32 = 0, SF_BF16 = 1 } sf_dtype;

/* flags */
#define SF_FLAG_CUDA_GRAPH  (1ull << 0) /* capture draft+verify+accept as one CUDA graph for decode_steps */
#define SF_FLAG_DRAFT_CAUSAL (1ull << 1) /* NEXT-2 ablation "+Att Mask": causal draft-slot mask (not default) */
/* NEXT-4, bf16 only: the LM-head GEMMs do not store the fp32 logits (the greedy / draft tokens come
 * from the argmax fused into their epilogue either way); specformer_read_logits then
 * returns SF_ERR_STATE. */
#define SF_FLAG_NO_LOGITS   (1ull << 2)
/* NEXT-2 ablation "-Pos" (T4, PAPER P497-514; reading in DESIGN.md §3): no positional FFN matrix -- each
 * draft slot is D_j = RMS_p(I_D) + b_P[j] (the weight table has no sf.w_p). Not the default. */
#define SF_FLAG_NO_POS_FFN  (1ull << 3)
/* NEXT-2 variant BIDIR_PREFIX (the north_star's wording: "draft slots attend causally over the prefix KV
 * cache and bidirectionally among themselves"; reading in DESIGN.md §3): the draft block's slots sit at
 * positions seq_len .. seq_len + k - 1 (RoPE'd there; their K / V written to the context layer's pages
 * beyond the committed length) and every slot sees the context layer's committed keys and all k slots.
 * Not the default; bf16 / fp32, no tensor parallelism. */
#define SF_FLAG_DRAFT_PREFIX (1ull << 4)
/* NEXT-4: KV pages come from a device-side pool of sf_config.pool_pages pages (0: max_batch x
 * max_seq / 16) instead of fixed per-sequence ranges: a sequence takes pages just before it writes them
 * (prefill: P + k + 1 positions; each accept_commit: up to seq_len + k + 1, fused into the accept kernel)
 * and returns them with specformer_release; specformer_prefill_slot admits a new sequence into a released
 * slot while the others keep decoding (continuous batching, PAPER P18). An exhausted pool is a sticky
 * SF_ERR_CAPACITY at specformer_sync. */
#define SF_FLAG_PAGE_POOL   (1ull << 5)
/* Tensor parallelism: the row-parallel partial outputs are all-reduced in bf16 by default (rounded RNE
 * from the fp32 GEMM output, summed by the collective, widened back: SURVEY 8e's volume, half the bytes
 * of fp32); this flag all-reduces them in fp32 instead. Parity of both measured in DESIGN.md §8. */
#define SF_FLAG_TP_F32_REDUCE (1ull << 6)

typedef struct {
  int32_t n_layers, d_model, n_heads, n_kv_heads, head_dim, d_ff, vocab;
  int32_t draft_len;   /* k = l_d (chain draft, no tree; PAPER P6, P37). 0 = plain greedy AR
                          decoding through verify_step + accept_commit (no draft head), used by
                          the GPU SD == AR losslessness test.                               */
  int32_t max_batch;   /* B_max sequences handled by this handle                          */
  int32_t max_seq;     /* per-sequence KV capacity (positions), multiple of kv_block;
                          <= 131072 for bf16 head_dim 128 (64 attention key segments of 2048) */
  int32_t kv_block;    /* paged-KV page size in tokens; must be 16                        */
  float rope_theta;    /* 10000 (reading C5)                                               */
  float rms_eps;       /* 1e-6 (reading C3)                                                */
  int32_t dtype;       /* sf_dtype: SF_FP32 (fp32 weights/activations/KV, SIMT kernels) or
                          SF_BF16 (bf16 weights/KV, tcgen05 GEMMs, fp32 residual/accum)     */
  int32_t tp_size, tp_rank; /* tensor parallelism (see sf_nccl_attach); 1, 0 = one GPU        */
  uint64_t flags;
  int32_t draft_blocks; /* bidirectional draft blocks (Eq.10 has one; 0 reads as 1). NEXT-2 "+Larger"
                           (T4 P497-514): 2..4 stacked blocks, weights sf.blk<i>_* for i >= 1 */
  int32_t pool_pages;   /* SF_FLAG_PAGE_POOL: KV pages in the pool (0: max_batch x max_seq / 16); the
                           per-layer KV pools are sized to it */
} sf_config;

typedef struct {
  char name[64];
  int32_t ndim;
  int64_t shape[4];
  int64_t offset_bytes; /* from the start of the packed weight blob (256-byte aligned) */
  int32_t dtype;        /* sf_dtype of the stored elements                              */
  int32_t layout;       /* 0: row-major [out, in]; 1: tile-contiguous bf16 GEMM layout written
                           by sf_pack_matrix (128 x 64 tiles, 128B-swizzled, t-major then k) */
} sf_tensor_desc;

typedef struct sf_handle sf_handle;

/* Packed weight layout. Returns the number of tensors (writes at most `cap` descriptors;
 * out may be NULL to query the count), or -1 on an invalid config.
 * Names: embed[V,d]; layers.<l>.{attn_norm[d] f32, wqkv[(Hq+2Hkv)hd, d] (rows q|k|v),
 * wo[d, Hq hd], ffn_norm[d] f32, w_gu[2F,d], w_down[d,F]}; final_norm[d] f32;
 * lm_head[V,d]; sf.group_scale[4,d] f32; sf.w_d[d,4d]; sf.ctx_norm[d] f32; sf.ctx_wqkv;
 * sf.ctx_wo; sf.pos_norm[d] f32; sf.w_p[k d, d]; sf.b_p[k d] f32; sf.blk_attn_norm[d] f32;
 * sf.blk_wqkv; sf.blk_wo; sf.blk_ffn_norm[d] f32; sf.blk_w_gu[2F,d]; sf.blk_w_down[d,F].
 * w_gu interleaves the SwiGLU gate and up projections row by row: row 2i is gate row i, row
 * 2i+1 is up row i, so a GEMM tile holds matching gate/up rows in adjacent accumulator lanes
 * for the fused SwiGLU epilogue (F % 64 == 0). In bf16 mode with head_dim 128, the rows of
 * layers.<l>.wqkv and sf.ctx_wqkv are pair-interleaved within each 128-row head: row 2i of a head is
 * its dimension i, row 2i+1 its dimension i + 64 (the rotate-half RoPE partners land in adjacent
 * accumulator lanes of the fused RoPE / KV-append epilogue); sf.blk_wqkv (no RoPE) keeps the
 * natural order.
 * Matrices are stored in the config dtype, vectors in fp32. In bf16 mode every matrix except
 * `embed` uses layout 1: fill it with sf_pack_matrix from a row-major device copy. */
int sf_weight_table(const sf_config* cfg, sf_tensor_desc* out, int cap);
int64_t sf_weights_bytes(const sf_config* cfg);   /* -1 on invalid config */
int64_t sf_workspace_bytes(const sf_config* cfg); /* KV pools (L+1 layers) + activations; -1 if invalid */

/* Validates cfg, carves `workspace_dev` (sf_workspace_bytes, 256-byte aligned), binds the
 * weight pointers. `stream` is a cudaStream_t (NULL = legacy default stream). */
sf_status specformer_init(const sf_config* cfg, void* weights_dev, void* workspace_dev, void* stream,
                          sf_handle** out);

/* Setup pass (untimed): base forward over the B x P prompt tokens (dev or host, [B,P] row-major)
 * in chunks, context layer L+1 over all P rows; first_token (dev or host, [B], may be NULL)
 * receives g0 = argmax logits[P-1]. Afterwards seq_len = P, last_token = g0. */
sf_status specformer_prefill(sf_handle* h, const int32_t* tokens, int32_t B, int32_t P, int32_t* first_token);

/* SpecFormer draft forward. draft (dev or host [B,k], may be NULL), draft_logits (dev [B,k,V]
 * fp32, may be NULL). The draft is also kept internally for verify_step. */
sf_status specformer_draft_step(sf_handle* h, int32_t* draft, float* draft_logits);

/* Base verify forward over [last_token, d_1..d_k] at positions seq_len..seq_len+k.
 * draft_in: dev or host [B,k] to verify instead of the internal draft (forced/adversarial
 * drafts), or NULL. greedy (dev or host [B,k+1]) and logits (dev [B,k+1,V] fp32) may be NULL. */
sf_status specformer_verify_step(sf_handle* h, const int32_t* draft_in, int32_t* greedy, float* logits);

/* Greedy accept + commit: m_b = longest prefix with draft[b,i] == greedy[b,i];
 * emitted[b, 0..m_b] = greedy[b, 0..m_b] (rest -1); seq_len += m_b + 1; last_token = greedy[b,m_b].
 * Outputs (dev or host, may be NULL): accept_len [B], emitted [B,k+1], seq_len [B]. */
sf_status specformer_accept_commit(sf_handle* h, int32_t* accept_len, int32_t* emitted, int32_t* seq_len);

/* Run n_steps x (draft -> verify -> accept) with no host synchronisation (CUDA-graph replay
 * when SF_FLAG_CUDA_GRAPH). emitted_log (dev, [n_steps, B, k+1]) and accept_log (dev,
 * [n_steps, B]) may be NULL. Fails with SF_ERR_CAPACITY if a step could overflow max_seq. */
sf_status specformer_decode_steps(sf_handle* h, int32_t n_steps, int32_t* emitted_log, int32_t* accept_log);

/* SF_FLAG_PAGE_POOL only (NEXT-4, continuous batching). specformer_release returns sequence slot's KV
 * pages to the pool; the slot must then be re-filled with specformer_prefill_slot before the next
 * draft / verify / decode call (SF_ERR_STATE otherwise). specformer_prefill_slot runs the prefill of one
 * new sequence (tokens dev or host [P]) into slot (< the batch of the last specformer_prefill) while the
 * other slots keep their state: seq_len[slot] = P, first_token (dev or host [1], may be NULL) = g0.
 * Errors: SF_ERR_UNSUPPORTED without the flag, SF_ERR_STATE before the first batch prefill or between
 * verify and accept, SF_ERR_SHAPE for a bad slot / P, SF_ERR_CAPACITY if P + k + 1 > max_seq. */
sf_status specformer_release(sf_handle* h, int32_t slot);
sf_status specformer_prefill_slot(sf_handle* h, int32_t slot, const int32_t* tokens, int32_t P, int32_t* first_token);

/* Stream sync + sticky device error flags -> status. */
sf_status specformer_sync(sf_handle* h);
const char* specformer_last_error(const sf_handle* h);
void specformer_destroy(sf_handle* h);

/* Number of kernels launched by the last call (host-side count; graph replays count their nodes). */
int64_t specformer_kernel_launches(const sf_handle* h);
/* Name of the library build ("sm_100a ...") for provenance. */
const char* specformer_build_info(void);

/* ------------------------------------------------------------------ test / bench hooks */
/* Replace the page table (host [B, max_seq/kv_block] of distinct page ids < B*max_seq/kv_block).
 * Only valid right after init (before prefill). */
sf_status sf_debug_set_block_table(sf_handle* h, const int32_t* table_host, int32_t B, int32_t n_pages_per_seq);
/* Copy an internal buffer to dst (dev or host). what: 0 taps [4, B(k+1), d] f32 of the last
 * verify; 1 I_D rows used by the last draft [B, d] f32; 2 E (draft block output) [B, k, d] f32;
 * 3 seq_len [B] i32; 4 last_token [B] i32; 5 n_prev [B] i32 (length before the last commit);
 * 6 hook taps of EVERY row of the last base forward (prefill: its last chunk, rows b-major) [4, rows, d]
 * f32; 7 context-layer output I_D of every row of the last context pass [rows, d] f32; 8 prompt_len
 * [B] i32. Returns bytes copied via *nbytes (6 / 7: query the size with a first call into a buffer of
 * sf_workspace-sized capacity, or compute rows from the call sequence). */
sf_status sf_debug_capture(sf_handle* h, int32_t what, void* dst, int64_t* nbytes);
/* Forced-acceptance drafts: overwrite the internal draft with
 * cont[b, g + j] (j = 1..k, g = seq_len - prompt_len, cont = AR continuation with cont[b,0] = g0)
 * and replace slot corrupt[b] (1..k; > k means none) with (token + 1) % V. Device pointers. */
sf_status sf_debug_force_drafts(sf_handle* h, const int32_t* cont_dev, int32_t cont_len, const int32_t* corrupt_dev);
/* Bench hook: make decode_steps overwrite each step's draft (after the draft forward ran and was
 * paid for) with forced drafts as in sf_debug_force_drafts, slot corrupt_dev[(step % corrupt_steps) * B + b].
 * cont_dev NULL disables. Device pointers must stay valid while enabled. */
sf_status sf_set_forced_drafts(sf_handle* h, const int32_t* cont_dev, int32_t cont_len, const int32_t* corrupt_dev,
                               int32_t corrupt_steps);
/* Per-kernel-class profiling for the bench roofline: when enabled, every launch is bracketed by
 * CUDA events on the handle's stream. With SF_FLAG_CUDA_GRAPH, decode_steps captures a profiling
 * copy of the step graph whose event records are graph nodes (cudaEventRecordExternal) and replays
 * it one step at a time, so the times carry no host launch gaps (a record node between two launches
 * does remove their programmatic overlap); without the flag the launches are eager.
 * Classes: 0 GEMM, 1 paged attention (RoPE/append + partial + combine), 2 RMSNorm/embedding,
 * 3 argmax. sf_profile(h, 1) clears and enables; sf_profile_read sums the elapsed milliseconds,
 * launch count and host-known algorithmic bytes (GEMM: weights + activations + outputs; 0 for
 * attention, whose KV bytes depend on device-resident lengths) of one class. */
sf_status sf_profile(sf_handle* h, int32_t enable);
sf_status sf_profile_read(sf_handle* h, int32_t cls, double* total_ms, int64_t* count, double* bytes);
/* Write row-major bf16 src[N, K] (device) into the tile-contiguous layout 1 at dst (device, N*K*2
 * bytes): 128-row x 64-column tiles stored contiguously (tile (t, k) at ((t * K/64) + k) * 16 KB)
 * as the exact image of a 128-byte-swizzled K-major shared-memory tile, so each GEMM pipeline
 * stage is one contiguous bulk copy and a stream-K range is one contiguous stretch of HBM.
 * Requires N % 128 == 0, K % 64 == 0. Asynchronous on `stream`. */
sf_status sf_pack_matrix(int32_t dtype, const void* src_dev, void* dst_dev, int64_t N, int64_t K, void* stream);
/* Direct GEMM entry (T-kernel parity): out[T,N] = A[T,K] W[N,K]^T with fp32 accumulation;
 * dtype SF_FP32 (A, W fp32), SF_BF16 (A, W bf16 row-major; W is packed to layout 1 internally) or
 * 2 (A bf16, W already in layout 1). out dev fp32. Uses the same kernels as the hot path. */
sf_status sf_test_gemm(int32_t dtype, const void* A, const void* W, float* out, int32_t T, int32_t N, int32_t K,
                       void* stream);
/* Tools only: average device time (ms, CUDA events over `reps` back-to-back launches after 2 warm-up
 * launches) of one bf16 EPI_PARTIAL GEMM out[T, N] = A[T, K] W[N, K]^T on zeroed inputs the call
 * allocates and frees: impl 0 the standalone stream-K launch, 1 the same GEMM as a one-phase
 * layer-sequence launch. */
sf_status sf_bench_gemm(int32_t impl, int32_t T, int32_t N, int32_t K, int32_t reps, float* ms_out);
/* Tools only: when the process ran with SF_GEMM_TRACE=1, copy (and clear) the per-CTA %globaltimer
 * timeline (ns; [CTA][64] uint64, slot map in csrc/gemm.cu) of the last tcgen05 GEMM launches into
 * host memory dst_host (cap entries). Returns the number of entries copied, 0 if tracing is off. */
int32_t sf_debug_gemm_trace(uint64_t* dst_host, int32_t cap);
/* Tools only: when the process ran with SF_KTRACE=1, copy (and clear) the kernel timeline: one
 * 40-byte record per CTA of every kernel launched since the last call -- {uint32 kind<<24|param,
 * uint32 smid, uint64 start_ns, uint64 dependency_resolved_ns, uint64 end_ns, uint64 0} -- into
 * host memory dst_host (cap records). Synchronises the device. Returns the number of records
 * copied, 0 if tracing is off. */
int32_t sf_debug_ktrace(void* dst_host, int32_t cap);
/* Turn the kernel timeline on (1) or off (0) at run time (bench.py's timeline pass; SF_KTRACE=1
 * turns it on at the first handle). Takes effect for launches -- graph replays included -- made
 * after the call: the probes read a device-global record pointer, null when off. Synchronises
 * the device and clears the log. Returns 0, or -1 if the 80 MB log cannot be allocated. */
int32_t sf_debug_ktrace_enable(int32_t on);

/* ---- Tensor parallelism (Megatron-style; sf_config.tp_size > 1, bf16 only) ----
 * Rank r of tp holds: q / kv heads [r H/tp, (r+1) H/tp) of every attention (QKV rows and O columns
 * sliced alike; the KV pools hold the rank's kv heads), FFN rows [r F/tp, ..) of gate/up and the
 * matching down-proj columns, the LM head's vocabulary rows [v0, v1) (whole 128-row tiles split as
 * evenly as possible; sf_weight_table reports the rank's shapes), W_D's input columns [r 4d/tp, ..)
 * (the rank's slice of I_Cat); embedding, norms, W_P / b_P and the residual stream are replicated.
 * The row-parallel outputs (base O / down, context W_D / O, draft O / down) are summed over the
 * ranks in fp32 before the residual add; the argmax max-reduces per-row packed keys
 * (orderable float logit << 32 | ~global id: largest logit, lowest id on ties). Every rank computes
 * the same tokens. Logits copied out (verify_step / draft_step) are the rank's vocabulary shard
 * [rows, v1 - v0]. One of the two collectives below must be attached before prefill. */
/* 128-byte NCCL unique id for sf_nccl_attach (rank 0 creates it; the caller broadcasts it).
 * Returns 0, -1 if NCCL is unavailable in this build. */
int32_t sf_nccl_unique_id(uint8_t* out_128);
/* Create this handle's NCCL communicator (nranks == tp_size, rank == tp_rank; call on the handle's
 * device). Reductions run as ncclAllReduce on the handle's stream and are captured by
 * SF_FLAG_CUDA_GRAPH. Errors: SF_ERR_ARG, SF_ERR_STATE (already attached), SF_ERR_NCCL. */
sf_status sf_nccl_attach(sf_handle* h, const uint8_t* id_128, int32_t nranks, int32_t rank);
/* Tests without a second GPU: n (<= 8) handles of one process on one device, each driven by its
 * own host thread, reduce through device memory with host barriers (rank order sums). Handles on
 * a local group run eagerly (decode_steps does not capture). The group owns its device scratch;
 * destroy it after its handles. */
typedef struct sf_local_group sf_local_group;
sf_local_group* sf_local_group_create(int32_t n);
void sf_local_group_destroy(sf_local_group* g);
sf_status sf_local_group_attach(sf_handle* h, sf_local_group* g, int32_t rank);

/* ---- NEXT-3: the row-parallel all-reduce fused into the residual + RMSNorm consumer, over peer memory
 * (PAPER P91-95: at large batch the step is compute-bound, so the ~2 L + 5
 * all-reduces per step must not sit on the critical path as separate collective launches).
 * Each rank owns an exchange region (library-allocated, 256 B of flags + two bf16 [R, d] slots, R the
 * handle's largest row block). A row-parallel GEMM (base O / down, context W_D / O, draft O / down)
 * stores its bf16 output straight into this rank's slot of the coming epoch (double-buffered, chosen
 * on the device by the epoch counter), a one-warp kernel increments the epoch and publishes it with a
 * system-scope release into every peer's flags, and the consumer on every rank waits (system-scope
 * acquire, bounded at 5 s -> SF_ERR_NCCL at specformer_sync) for all peers' flags, then adds the ranks'
 * slots to the fp32 residual in rank order 0..tp-1 (every rank: the same values in the same order,
 * hence the same bits) before the norm. Replaces the NCCL all-reduce of the row-parallel outputs
 * (the argmax max still uses the attached collective). Attach after the collective and before the
 * first prefill; every rank must attach. bf16 handles with 2 <= tp_size <= 8 only
 * (SF_ERR_UNSUPPORTED / SF_ERR_STATE otherwise). */
/* This rank's exchange region as a 64-byte cudaIpcMemHandle_t (allocates the region on first use). */
sf_status sf_tp_xch_handle(sf_handle* h, uint8_t* out_64);
/* One process per GPU: handles_64xtp = every rank's sf_tp_xch_handle bytes in rank order (this rank's
 * entry is not opened). Opens the peers' regions with cudaIpcOpenMemHandle (lazy peer access);
 * captured by SF_FLAG_CUDA_GRAPH. Errors: SF_ERR_CUDA (a peer region cannot be mapped), SF_ERR_STATE. */
sf_status sf_tp_xch_attach(sf_handle* h, const uint8_t* handles_64xtp);
/* Local group (one process, one device, tests): the ranks' regions are shared directly; after every
 * epoch signal the ranks meet at a host barrier, so no rank's kernel ever waits on another rank's
 * kernel (the flag waits are satisfied before the consumer starts). Every rank calls it (it blocks
 * until all have); needs sf_local_group_attach with the same group first. */
sf_status sf_local_group_xch_attach(sf_handle* h, sf_local_group* g);

#ifdef __cplusplus
}
#endif
#endif /* SPECFORMER_H_ */
