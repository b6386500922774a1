// gemm.cuh -- GEMM launch interface shared by the runtime.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace sf {

enum EpiMode : int {
  EPI_STORE_ACT = 0,   // out_act[t, n] = acc                     (next GEMM's operand)
  EPI_STORE_F32 = 1,   // out_f32[t, n] = acc                     (logits, residual init)
  EPI_ADD_F32 = 2,     // out_f32[t, n] += acc; tap[t, n] = result (residual stream, Eq.7)
  EPI_BIAS_F32 = 3,    // out_f32[t, n] = acc + bias[n]           (positional FFN, Eq.9)
  EPI_SWIGLU_ACT = 4,  // W rows interleaved [gate_0; up_0; gate_1; up_1; ...]:
                       // out_act[t, i] = silu(gate_i) * up_i  (SwiGLU, P197)
  EPI_PARTIAL = 5,     // bf16 path, N/128 <= #SMs: every k-segment's fp32 accumulator goes to the
                       // scratch partial slots; a consumer (launch_resid_norm) adds them in k order
  EPI_QKV_ROPE = 6,    // bf16, head_dim 128 (one head per 128-row tile), W rows pair-interleaved per
                       // head (row 2i = dim i, 2i+1 = dim i+64): RoPE on q / k heads at the rows'
                       // positions, q -> rope.q_out [T, Hq, 128] bf16, k / v -> their page slots
};
struct RopeEpi {
  const int* pos0 = nullptr;   // [B] position of each sequence's first row; row t = b q_len + i
  int q_len = 1;
  const float2* table = nullptr;  // [max_seq, 64] (cos, sin)
  int Hq = 0, Hkv = 0;
  const int* bt = nullptr;     // [B, pps] page table
  int pps = 0;
  void* Kp = nullptr;          // [pages, Hkv, 16, 128] bf16
  void* Vp = nullptr;
  void* q_out = nullptr;       // [T, Hq, 128] bf16
  int t0 = 0;                  // row offset of this launch chunk (T > 512 runs in chunks)
};

struct GemmEpi {
  int mode = EPI_STORE_ACT;
  void* out = nullptr;
  int ldo = 0;             // row stride of out (elements)
  const float* bias = nullptr;
  float* tap = nullptr;    // optional extra copy (ADD_F32 only), row stride ldo
  // optional: the next GEMM's weights; once this launch has issued its own loads, each CTA
  // prefetches a slice of them into L2 so the DRAM keeps streaming through the epilogue tail
  const void* pf = nullptr;
  size_t pf_bytes = 0;
  RopeEpi rope;  // EPI_QKV_ROPE only
  // tile-entry cost of the stream-K partition (k segmentation); < 0: the mode's default. Launches
  // whose results must agree bit for bit across modes (the QKV projection: EPI_QKV_ROPE for short
  // blocks, EPI_PARTIAL + launch_rope_partial for long ones) pass the same value.
  int drain = -1;
  // EPI_STORE_F32 on the tcgen05 path (the LM head, NEXT-4): argmax fused into the epilogue. For
  // each row t the CTA reduces its tile's packed keys orderable(acc) << 32 | (0xFFFFFFFF - (amax_v0 +
  // n)) over n with warp shuffles and atomicMax-es them into amax[t] (largest logit, lowest id on
  // ties; +0 and -0 compare equal), which must hold 0 (or a smaller key) beforehand; a non-finite
  // value sets *amax_err. out == nullptr: the fp32 values are not stored at all.
  unsigned long long* amax = nullptr;
  unsigned amax_v0 = 0;
  int* amax_err = nullptr;
  // EPI_STORE_ACT into a double-buffered slot chosen on the device (NEXT-3, the fused tensor-parallel
  // all-reduce): the rows go to out + ((*out_sel + 1) & 1) * out_sel_stride elements -- the slot of the
  // all-reduce whose epoch the next tp_signal launch will publish (*out_sel + 1)
  const int* out_sel = nullptr;
  long long out_sel_stride = 0;
};

// NEXT-3: the peers' exchange slots a fused residual + norm consumer sums (tensor parallelism over
// peer memory, include/specformer.h sf_tp_xch_*). Rank q's slot for epoch e is slot[q] +
// (e & 1) * slot_elems ([T, d] bf16, the rank's row-parallel GEMM output); flags[q] holds the last
// epoch rank q published into THIS rank's region, *ctr this rank's current epoch.
constexpr int kTpMax = 8;
struct TpSrc {
  const __nv_bfloat16* slot[kTpMax];
  const int* ctr = nullptr;
  const int* flags = nullptr;
  int* err = nullptr;         // sticky: a peer's flag did not arrive within the time limit
  long long slot_elems = 0;
  int n = 0;                  // ranks (0: off)
  int own = 0;
};
struct TpPeers {
  int* p[kTpMax];
};
// rank `own` publishes its next epoch: ++*ctr, then (system-scope release) peer_flags[q][own] = epoch
cudaError_t launch_tp_signal(int* ctr, int* const* peer_flags, int n, int own, cudaStream_t s);

struct GemmScratch {
  float* partial = nullptr;   // split-K partials
  int64_t partial_elems = 0;
  int* counters = nullptr;    // per-N-tile arrival counters (zeroed; kernels re-zero them)
  int n_counters = 0;
};

// out = A[T, K] . W[N, K]^T with fp32 accumulation.
// is_bf16: A, W bf16 (tcgen05 path, requires N % 128 == 0, K % 64 == 0); W either row-major
// [N, K] (w_tiled = false) or in the tile-contiguous layout written by gemm_pack_weight.
// Otherwise fp32 (SIMT path, W row-major). act outputs are in the same dtype as A.
cudaError_t gemm_launch(bool is_bf16, const void* A, int lda, const void* W, bool w_tiled, int T, int N, int K,
                        const GemmEpi& epi, const GemmScratch& scratch, cudaStream_t s);
// Row-major bf16 W[N, K] -> tile-contiguous 128x64 pre-swizzled layout (same byte count).
cudaError_t gemm_pack_weight(const void* src, void* dst, int N, int K, cudaStream_t s);

// Copies (and clears) the per-CTA timeline of GEMM launches made with SF_GEMM_TRACE=1 set
// (tools only); returns the number of 64-bit entries copied (0 when tracing is off).
int gemm_trace_copy(unsigned long long* host, int n);

// scratch floats needed by gemm_launch for (T, N, K)
int64_t gemm_partial_elems(bool is_bf16, int T, int N, int K);

// Stream-K geometry the EPI_PARTIAL consumer needs to locate a tile's k-segments.
struct PartialGeom {
  int G;          // CTAs
  int kb;         // k-blocks per tile
  int n_tiles;    // 128-row tiles
  int T;          // rows per launch chunk (slot stride)
  int drain;      // tile-entry cost of the stream-K partition
};
// false if EPI_PARTIAL unsupported; drain as GemmEpi::drain
bool gemm_partial_geom(int T, int N, int K, PartialGeom* g, int drain = -1);

// Fused consumer of EPI_PARTIAL (and plain residual/norm): for virtual row r (T*rep rows, source
// row r / rep, columns [(r % rep) * d, +d) of the GEMM output):
//   x = (resid ? resid[r] : 0) + (add ? add[r] : 0) + (bias ? bias[col] : 0) + sum_k-segments partial
//   (tp: + sum over the ranks q = 0, 1, .. of the bf16 exchange slots, after waiting for their epoch)
//   (fixed order; partial may be null -- add carries a tensor-parallel all-reduced GEMM output)
//   out[r] = x (fp32, out may alias resid); tap[r] = x (optional);
//   xn[r] = bf16(x / sqrt(mean(x^2) + eps) * gamma) (optional, gamma != null)
bool resid_norm_supported(int d, int T, int N, int K);
cudaError_t launch_resid_norm(const float* partial, const PartialGeom* g, int T, int rep, int d, const float* resid,
                              const float* add, const float* bias, float* out, float* tap, const float* gamma,
                              float eps, __nv_bfloat16* xn, cudaStream_t s, const TpSrc* tp = nullptr);

// Gate/up (SwiGLU, rows interleaved) -> down in ONE launch: phase A computes act = SwiGLU(A . WA^T)
// [T, NA/2] and publishes each finished 128-row tile; phase B (down, NB rows, K = NA/2) streams its
// weights into the ring while phase A drains and loads an activation k-block once published. Phase B
// is written as EPI_PARTIAL slots at scratch.partial + gemm_chain_partial_offset(T) with the
// standalone down GEMM's k segmentation (bit-identical results; launch_resid_norm consumes them).
bool gemm_chain_supported(int T, int NA, int KA, int NB);
int64_t gemm_chain_partial_offset(int T);
int64_t gemm_chain_partial_elems(int T);  // scratch floats the chain needs
cudaError_t gemm_chain_launch(const void* A, int lda, const void* WA, int NA, int KA, void* act, const void* WB,
                              int NB, int T, const GemmScratch& scratch, cudaStream_t s);

// Consumer of an EPI_PARTIAL QKV projection (bf16, head_dim 128, one 128-row tile per head, rows
// pair-interleaved per head as for EPI_QKV_ROPE): for every (row t, head h) the head's k-segment
// partials are summed in k order (the first segment, then the others: the same additions as the
// GEMM's own head-tile fixup), rounded to bf16, and -- exactly as launch_rope_append's 128-wide
// kernel does with the bf16 projection -- q / k heads rotated at position pos0[t / q_len] + t % q_len
// (q -> q_out [T, Hq, 128], k -> its page slot) and v heads copied to their page slot.
bool rope_partial_supported(int T, int N, int K, int Hq, int Hkv, int drain);
cudaError_t launch_rope_partial(const float* partial, const PartialGeom* g, int T, int q_len, const int* pos0,
                                const float2* rope, int Hq, int Hkv, const int* bt, int pps, void* Kp, void* Vp,
                                void* q_out, cudaStream_t s);

// Layer-sequence kernel (csrc/gemm_seq.cuh): several GEMM phases (bf16, CTA pairs, modes EPI_PARTIAL /
// EPI_SWIGLU_ACT / EPI_QKV_ROPE) and consumers of the preceding EPI_PARTIAL phase (residual + RMSNorm,
// RoPE / KV append) in ONE persistent launch, each with the standalone launches' partition and
// arithmetic (bit-identical results); the weight stream runs ahead across phase boundaries.
enum SeqKind : int { SEQ_GEMM = 0, SEQ_RESID_NORM = 1, SEQ_ROPE = 2 };
constexpr int kSeqMaxPhases = 8;
constexpr int kSeqMaxGemm = 4;
struct SeqStep {
  int kind = SEQ_GEMM;
  // SEQ_GEMM: out = A[T, K] . W[N, K]^T (W tile-contiguous), epilogue epi (PARTIAL / SWIGLU / QKV_ROPE)
  const void* A = nullptr;
  int lda = 0;
  const void* W = nullptr;
  int N = 0, K = 0;
  GemmEpi epi;  // (SEQ_ROPE: epi.rope)
  // SEQ_RESID_NORM (as launch_resid_norm with rep = 1, add = bias = null, d = the GEMM's N)
  const float* resid = nullptr;
  float* out = nullptr;
  float* tap = nullptr;
  const float* gamma = nullptr;
  __nv_bfloat16* xn = nullptr;
  int d = 0;
  float eps = 0.f;
};
bool gemm_seq_supported(int T, const SeqStep* steps, int n);
// sync: kSeqSyncInts device ints, zeroed once, private to one call site (the kernel keeps them
// consistent across launches with a launch epoch); scratch as gemm_launch's
constexpr int kSeqSyncInts = 64 + 8 * 128 * 36;
cudaError_t gemm_seq_launch(int T, const SeqStep* steps, int n, const GemmScratch& scratch, int* sync, cudaStream_t s);

}  // namespace sf
