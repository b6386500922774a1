"""Thin Python binding over the C ABI: device memory via torch, marshalling only.

Every step of the decode path (draft, verify, accept) runs inside libspecformer.so's sm_100a
kernels; this module allocates the packed weight blob / workspace with torch, packs the caller's
weight dict into the layout `sf_weight_table` reports (concatenating q|k|v rows and interleaving
gate/up rows in 64-row groups) and forwards calls.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _native as N


@dataclass
class EngineConfig:
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    d_ff: int
    vocab: int
    draft_len: int
    max_batch: int
    max_seq: int
    dtype: str = "bf16"          # "bf16" | "fp32"
    rope_theta: float = 10000.0
    rms_eps: float = 1e-6
    kv_block: int = 16
    flags: int = 0
    tp_size: int = 1             # tensor parallelism (include/specformer.h): ranks, this rank
    tp_rank: int = 0
    draft_blocks: int = 1        # NEXT-2 "+Larger": stacked draft blocks
    pool_pages: int = 0          # NEXT-4 (SF_FLAG_PAGE_POOL): KV pages in the pool (0: max_batch x max_seq / 16)

    @classmethod
    def from_model(cls, m, max_batch=None, max_seq=None, draft_len=None, flags=0, tp_size=1, tp_rank=0):
        """Build from any object with the model-shape attributes (e.g. synth.ModelConfig)."""
        # the NEXT-2 draft variants of the model config map to their flags
        flags |= (N.SF_FLAG_NO_POS_FFN if getattr(m, "no_pos_ffn", False) else 0) | \
            (N.SF_FLAG_DRAFT_PREFIX if getattr(m, "draft_prefix", False) else 0)
        return cls(m.n_layers, m.d_model, m.n_heads, m.n_kv_heads, m.head_dim, m.d_ff, m.vocab,
                   m.draft_len if draft_len is None else draft_len, max_batch or m.batch,
                   max_seq or m.max_seq, m.dtype, m.rope_theta, m.rms_eps, m.kv_block, flags, tp_size, tp_rank,
                   getattr(m, "draft_blocks", 1))

    def to_c(self) -> N.sf_config:
        return N.sf_config(self.n_layers, self.d_model, self.n_heads, self.n_kv_heads, self.head_dim, self.d_ff,
                           self.vocab, self.draft_len, self.max_batch, self.max_seq, self.kv_block,
                           self.rope_theta, self.rms_eps, N.SF_BF16 if self.dtype == "bf16" else N.SF_FP32,
                           self.tp_size, self.tp_rank, self.flags, self.draft_blocks, self.pool_pages)

    def vocab_shard(self):
        """[v0, v1): this rank's LM-head rows (whole 128-row tiles; the library's split)."""
        if self.tp_size <= 1:
            return 0, self.vocab
        tiles = self.vocab // 128
        return tiles * self.tp_rank // self.tp_size * 128, tiles * (self.tp_rank + 1) // self.tp_size * 128


def weight_table(cfg: EngineConfig):
    lib = N.lib()
    c = cfg.to_c()
    n = lib.sf_weight_table(C.byref(c), None, 0)
    if n < 0:
        raise N.SpecFormerError(N.SF_ERR_ARG, "invalid config")
    arr = (N.sf_tensor_desc * n)()
    lib.sf_weight_table(C.byref(c), arr, n)
    return [(d.name.decode(), tuple(d.shape[: d.ndim]), d.offset_bytes, d.dtype, d.layout) for d in arr]


def _interleave_gu(gate: torch.Tensor, up: torch.Tensor) -> torch.Tensor:
    F, d = gate.shape
    return torch.stack([gate, up], dim=1).reshape(2 * F, d)  # rows 2i = gate_i, 2i+1 = up_i


def _pair_interleave_heads(W: torch.Tensor, hd: int) -> torch.Tensor:
    """Rows of each hd-row head reordered [0, hd/2, 1, hd/2 + 1, ...] (include/specformer.h)."""
    n = W.shape[0] // hd
    half = hd // 2
    idx = torch.arange(hd, device=W.device).view(2, half).t().reshape(-1)  # 0, 64, 1, 65, ...
    return W.view(n, hd, -1)[:, idx, :].reshape(W.shape)


def _rows(t: torch.Tensor, i: int, n: int) -> torch.Tensor:
    """Block i of n equal row blocks."""
    r = t.shape[0] // n
    return t[i * r:(i + 1) * r]


def _cols(t: torch.Tensor, i: int, n: int) -> torch.Tensor:
    c = t.shape[1] // n
    return t[:, i * c:(i + 1) * c]


def _source_tensor(name: str, w: dict, rope_pairs: int = 0, cfg: EngineConfig | None = None) -> torch.Tensor:
    """Map a packed-table name to the caller's canonical tensors (see synth/weights.py).
    rope_pairs = head_dim when the RoPE'd QKV projections are pair-interleaved (bf16, hd 128).
    cfg.tp_size > 1: this rank's slice (include/specformer.h, tensor parallelism): heads of the q / k /
    v rows and O columns, FFN rows of gate / up and down columns, the vocabulary shard of the LM head,
    the input-column block of W_D; everything else whole."""
    tp, r = (cfg.tp_size, cfg.tp_rank) if cfg is not None and cfg.tp_size > 1 else (1, 0)
    pre, _, leaf = name.rpartition(".")
    pre = pre + "." if pre else ""
    if leaf.endswith("wqkv"):
        p = pre + leaf[:-4]
        W = torch.cat([_rows(w[p + "wq"], r, tp), _rows(w[p + "wk"], r, tp), _rows(w[p + "wv"], r, tp)], dim=0)
        if rope_pairs and not leaf.startswith("blk"):  # (draft blocks: no RoPE, natural rows)
            W = _pair_interleave_heads(W, rope_pairs)
        return W
    if leaf.endswith("w_gu"):
        p = pre + leaf[:-4]
        return _interleave_gu(_rows(w[p + "w_gate"], r, tp), _rows(w[p + "w_up"], r, tp))
    if tp > 1:
        if leaf.endswith("wo") or leaf.endswith("w_down") or leaf == "w_d":  # row-parallel
            return _cols(w[name], r, tp)
        if name == "lm_head":
            v0, v1 = cfg.vocab_shard()
            return w[name][v0:v1]
    return w[name]


def pack_weights(cfg: EngineConfig, weights: dict, device="cuda") -> torch.Tensor:
    """Copy the caller's tensors into the packed blob; layout-1 matrices go through the library's
    sf_pack_matrix kernel (tile-contiguous GEMM layout)."""
    lib = N.lib()
    c = cfg.to_c()
    nbytes = lib.sf_weights_bytes(C.byref(c))
    blob = torch.empty(nbytes, dtype=torch.uint8, device=device)
    stream = torch.cuda.current_stream(device)
    rope_pairs = cfg.head_dim if (cfg.dtype == "bf16" and cfg.head_dim == 128) else 0
    for name, shape, off, dt, layout in weight_table(cfg):
        t = _source_tensor(name, weights, rope_pairs, cfg)
        tdtype = torch.bfloat16 if dt == N.SF_BF16 else torch.float32
        if tuple(t.shape) != shape:
            raise ValueError(f"{name}: expected {shape}, got {tuple(t.shape)}")
        n = t.numel() * (2 if dt == N.SF_BF16 else 4)
        src = t.to(device=device, dtype=tdtype).contiguous()
        if layout == 1:
            st = lib.sf_pack_matrix(dt, C.c_void_p(src.data_ptr()), C.c_void_p(blob.data_ptr() + off), shape[0],
                                    shape[1], C.c_void_p(stream.cuda_stream))
            if st != N.SF_OK:
                raise N.SpecFormerError(st, f"sf_pack_matrix({name})")
            torch.cuda.current_stream(device).synchronize()  # src may be freed after this iteration
        else:
            blob[off: off + n].view(tdtype).view(shape).copy_(src)
    return blob


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


class Engine:
    """One handle over B_max sequences on the current CUDA device."""

    def __init__(self, cfg: EngineConfig, weights: dict, device="cuda", stream: torch.cuda.Stream | None = None):
        self.cfg = cfg
        self.lib = N.lib()
        self.device = torch.device(device)
        self.stream = stream or torch.cuda.Stream(device=self.device)
        self._c = cfg.to_c()
        self.weights = pack_weights(cfg, weights, self.device)
        ws = self.lib.sf_workspace_bytes(C.byref(self._c))
        if ws < 0:
            raise N.SpecFormerError(N.SF_ERR_ARG, "invalid config")
        self.workspace = torch.empty(ws, dtype=torch.uint8, device=self.device)
        torch.cuda.synchronize(self.device)
        h = C.c_void_p()
        st = self.lib.specformer_init(C.byref(self._c), _ptr(self.weights), _ptr(self.workspace),
                                      C.c_void_p(self.stream.cuda_stream), C.byref(h))
        if st != N.SF_OK:
            raise N.SpecFormerError(st, "specformer_init")
        self.h = h
        self.B = 0
        v0, v1 = cfg.vocab_shard()
        self.v0, self.v_local = v0, v1 - v0  # logits copied out are this rank's vocabulary shard

    # ---------------------------------------------------------------- helpers
    def _enter(self):
        # inputs produced on torch's current stream must be visible to the engine stream
        self.stream.wait_stream(torch.cuda.current_stream(self.device))

    def _exit(self):
        # outputs written on the engine stream become visible to torch's current stream
        torch.cuda.current_stream(self.device).wait_stream(self.stream)

    def _check(self, st, what):
        self._exit()
        if st != N.SF_OK:
            msg = self.lib.specformer_last_error(self.h)
            raise N.SpecFormerError(st, f"{what}: {msg.decode() if msg else ''}")

    def _i32(self, *shape):
        return torch.empty(*shape, dtype=torch.int32, device=self.device)

    @property
    def k(self):
        return self.cfg.draft_len

    # ---------------------------------------------------------------- API
    def prefill(self, tokens: torch.Tensor):
        """tokens: int32 [B, P] (device or pinned host). Returns g0 [B] (device int32)."""
        tokens = tokens.to(torch.int32).contiguous()
        B, P = tokens.shape
        first = self._i32(B)
        self._enter()
        self._check(self.lib.specformer_prefill(self.h, _ptr(tokens), B, P, _ptr(first)), "prefill")
        self.B = B
        return first

    def draft_step(self, want_logits=False):
        d = self._i32(self.B, self.k)
        lg = torch.empty(self.B, self.k, self.v_local, device=self.device) if want_logits else None
        self._enter()
        self._check(self.lib.specformer_draft_step(self.h, _ptr(d), _ptr(lg)), "draft_step")
        return (d, lg) if want_logits else d

    def verify_step(self, draft: torch.Tensor | None = None, want_logits=False):
        g = self._i32(self.B, self.k + 1)
        lg = torch.empty(self.B, self.k + 1, self.v_local, device=self.device) if want_logits else None
        if draft is not None:
            draft = draft.to(torch.int32).contiguous()
        self._enter()
        self._check(self.lib.specformer_verify_step(self.h, _ptr(draft), _ptr(g), _ptr(lg)), "verify_step")
        return (g, lg) if want_logits else g

    def accept_commit(self):
        m, em, sl = self._i32(self.B), self._i32(self.B, self.k + 1), self._i32(self.B)
        self._enter()
        self._check(self.lib.specformer_accept_commit(self.h, _ptr(m), _ptr(em), _ptr(sl)), "accept_commit")
        return m, em, sl

    def decode_steps(self, n: int, emitted_log: torch.Tensor | None = None, accept_log: torch.Tensor | None = None):
        self._enter()
        self._check(self.lib.specformer_decode_steps(self.h, n, _ptr(emitted_log), _ptr(accept_log)),
                    "decode_steps")

    def sync(self):
        self._check(self.lib.specformer_sync(self.h), "sync")

    def release(self, slot: int):
        """SF_FLAG_PAGE_POOL: return sequence `slot`'s KV pages to the pool (re-fill it with prefill_slot)."""
        self._check(self.lib.specformer_release(self.h, slot), "release")

    def prefill_slot(self, slot: int, tokens: torch.Tensor):
        """SF_FLAG_PAGE_POOL: prefill one new sequence (int32 [P]) into `slot`; returns g0 [1] (device)."""
        tokens = tokens.to(torch.int32).contiguous()
        first = self._i32(1)
        self._enter()
        self._check(self.lib.specformer_prefill_slot(self.h, slot, _ptr(tokens), tokens.numel(), _ptr(first)),
                    "prefill_slot")
        return first

    def set_block_table(self, table: torch.Tensor):
        t = table.to(torch.int32).contiguous().cpu()
        self._check(self.lib.sf_debug_set_block_table(self.h, C.c_void_p(t.data_ptr()), t.shape[0], t.shape[1]),
                    "set_block_table")

    def capture(self, what: int, shape, dtype=torch.float32):
        out = torch.empty(*shape, dtype=dtype, device=self.device)
        nb = C.c_int64()
        self._check(self.lib.sf_debug_capture(self.h, what, _ptr(out), C.byref(nb)), "capture")
        return out

    def set_forced_drafts(self, cont: torch.Tensor | None, corrupt: torch.Tensor | None = None):
        self._forced = (cont, corrupt)  # keep alive
        if cont is None:
            self._check(self.lib.sf_set_forced_drafts(self.h, None, 0, None, 1), "set_forced_drafts")
            return
        cs = corrupt.shape[0] if corrupt is not None else 1
        self._enter()
        self._check(self.lib.sf_set_forced_drafts(self.h, _ptr(cont), cont.shape[1], _ptr(corrupt), cs),
                    "set_forced_drafts")

    def profile(self, enable: bool):
        self._check(self.lib.sf_profile(self.h, 1 if enable else 0), "profile")

    def profile_read(self, cls: int):
        ms, n, by = C.c_double(), C.c_int64(), C.c_double()
        self._check(self.lib.sf_profile_read(self.h, cls, C.byref(ms), C.byref(n), C.byref(by)), "profile_read")
        return ms.value, n.value, by.value

    # ---------------------------------------------------------------- tensor parallelism
    def attach_nccl(self, unique_id: bytes, nranks: int, rank: int):
        """NCCL communicator over the tp ranks (unique_id from nccl_unique_id() on rank 0)."""
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        self._check(self.lib.sf_nccl_attach(self.h, buf, nranks, rank), "sf_nccl_attach")

    def attach_local_group(self, group, rank: int):
        """Tests: reduce with the other handles of `group` (LocalGroup) in this process."""
        self._group = group  # keep alive
        self._check(self.lib.sf_local_group_attach(self.h, group.g, rank), "sf_local_group_attach")

    def xch_handle(self) -> bytes:
        """NEXT-3: this rank's exchange region as 64 IPC-handle bytes (tp.share_xch_handles gathers them)."""
        buf = (C.c_uint8 * 64)()
        self._check(self.lib.sf_tp_xch_handle(self.h, buf), "sf_tp_xch_handle")
        return bytes(buf)

    def attach_xch(self, handles: list[bytes]):
        """NEXT-3 (one process per GPU): map the peers' exchange regions; the row-parallel all-reduce then
        runs fused into the residual + norm consumer over peer memory."""
        if len(handles) != self.cfg.tp_size or any(len(x) != 64 for x in handles):
            raise ValueError("one 64-byte handle per rank, in rank order")
        buf = (C.c_uint8 * (64 * len(handles))).from_buffer_copy(b"".join(handles))
        self._check(self.lib.sf_tp_xch_attach(self.h, buf), "sf_tp_xch_attach")

    def attach_local_xch(self):
        """NEXT-3 on a local group (tests): every rank's thread calls it after attach_local_group."""
        self._check(self.lib.sf_local_group_xch_attach(self.h, self._group.g), "sf_local_group_xch_attach")

    def kernel_launches(self) -> int:
        return int(self.lib.specformer_kernel_launches(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.lib.specformer_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pack_matrix(W: torch.Tensor) -> torch.Tensor:
    """Row-major bf16 W[N, K] (device) -> layout-1 copy (same shape/bytes, tile-contiguous)."""
    out = torch.empty_like(W)
    st = N.lib().sf_pack_matrix(N.SF_BF16, _ptr(W.contiguous()), _ptr(out), W.shape[0], W.shape[1],
                                C.c_void_p(torch.cuda.current_stream(W.device).cuda_stream))
    if st != N.SF_OK:
        raise N.SpecFormerError(st, "sf_pack_matrix")
    return out


def run_gemm(A: torch.Tensor, W: torch.Tensor, stream=None, w_tiled: bool = False) -> torch.Tensor:
    """out[T,N] = A[T,K] W[N,K]^T through the hot path's GEMM kernels (T-kernel parity hook).
    w_tiled: W was produced by pack_matrix."""
    lib = N.lib()
    T, K = A.shape
    Nn = W.shape[0]
    out = torch.empty(T, Nn, dtype=torch.float32, device=A.device)
    dt = (2 if w_tiled else N.SF_BF16) if A.dtype == torch.bfloat16 else N.SF_FP32
    s = stream or torch.cuda.current_stream(A.device)
    st = lib.sf_test_gemm(dt, _ptr(A.contiguous()), _ptr(W.contiguous()), _ptr(out), T, Nn, K,
                          C.c_void_p(s.cuda_stream))
    if st != N.SF_OK:
        raise N.SpecFormerError(st, "sf_test_gemm")
    return out


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    if N.lib().sf_nccl_unique_id(buf) != 0:
        raise N.SpecFormerError(N.SF_ERR_UNSUPPORTED, "NCCL unavailable")
    return bytes(buf)


class LocalGroup:
    """n handles of one process on one device reducing through device memory (tests only)."""

    def __init__(self, n: int):
        self.g = N.lib().sf_local_group_create(n)
        if not self.g:
            raise N.SpecFormerError(N.SF_ERR_ARG, "sf_local_group_create")

    def close(self):
        if self.g:
            N.lib().sf_local_group_destroy(self.g)
            self.g = None
