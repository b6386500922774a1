"""Algorithmic bytes / FLOPs of one decode step.

Counted once per pass: every weight byte of the base model (verify) and of the SpecFormer head +
shared LM head (draft), every KV byte once per (sequence, layer) -- the k+1 query rows share one
KV stream -- and the fp32 logits once written and once read (with SF_FLAG_NO_LOGITS: the fused
argmax's 8-byte keys per row instead). Not counted: re-reads, padded MMA rows, split-K / split-KV
partials, L2 hits.
"""
from __future__ import annotations


def _attn_params(c):
    d, hq, hkv, hd = c.d_model, c.n_heads, c.n_kv_heads, c.head_dim
    return d * (hq + 2 * hkv) * hd + hq * hd * d


def base_linear_params(c):
    return c.n_layers * (_attn_params(c) + 3 * c.d_model * c.d_ff)


def head_params(c, k):
    d = c.d_model
    return 4 * d * d + _attn_params(c) + k * d * d + _attn_params(c) + 3 * d * c.d_ff


def kv_bytes_per_token_layer(c, elt=2):
    return 2 * c.n_kv_heads * c.head_dim * elt


def attention_kv_bytes(c, lens_verify, lens_ctx, k, elt=2):
    """KV bytes read by the paged-attention launches of one step: base layers at positions
    0..n_b+k (verify), context layer L+1 at 0..n_prev_b+k (draft)."""
    per = kv_bytes_per_token_layer(c, elt)
    return per * (c.n_layers * sum(n + k + 1 for n in lens_verify) + sum(n + k + 1 for n in lens_ctx))


def step_bytes(c, B, k, lens_verify, lens_ctx, elt=2, logits=True):
    V, d = c.vocab, c.d_model
    w = (base_linear_params(c) + V * d) * elt          # verify: base + LM head
    w += (head_params(c, k) + V * d) * elt             # draft: head + LM head again
    kv = attention_kv_bytes(c, lens_verify, lens_ctx, k, elt)
    rows = B * (k + 1) + B * k
    out = rows * V * 4 * 2 if logits else rows * 8 * 2
    return w + kv + out


def step_flops(c, B, k, lens_verify):
    T = B * (k + 1)
    V, d = c.vocab, c.d_model
    f = 2 * T * (base_linear_params(c) + V * d)
    f += 2 * T * (4 * d * d + _attn_params(c))                 # W_D + context QKV/O
    f += 2 * B * k * d * d                                      # W_P
    f += 2 * B * k * (_attn_params(c) + 3 * d * c.d_ff + V * d)  # draft block + LM head
    ctx = sum(lens_verify) / max(1, len(lens_verify)) + k + 1
    f += 4 * T * ctx * c.n_heads * c.head_dim * (c.n_layers + 1)
    return f


def prefill_flops(c, B, P, k):
    """FLOPs of the prefill: base layers + the context layer L+1 (W_D, its QKV / O) over
    all B P prompt rows, causal attention over the prompt in every layer (P (P+1) / 2 query-key pairs per
    head, score + value products: 4 hd each) and the LM head on the last row of each sequence."""
    d = c.d_model
    rows = B * P
    f = 2 * rows * (base_linear_params(c) + 4 * d * d + _attn_params(c))
    f += 4 * B * (P * (P + 1) // 2) * c.n_heads * c.head_dim * (c.n_layers + 1)
    f += 2 * B * c.vocab * d
    return f


def prefill_bytes(c, B, P, k, chunks, elt=2):
    """Algorithmic bytes of the chunked prefill: every weight once per chunk pass, the KV of all L+1
    layers written once and re-read by the later chunks' attention (lower bound: written once)."""
    w = (base_linear_params(c) + 4 * c.d_model * c.d_model + _attn_params(c)) * elt * chunks
    kv = B * P * (c.n_layers + 1) * kv_bytes_per_token_layer(c, elt)
    return w + kv + c.vocab * c.d_model * elt
