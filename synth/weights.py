"""Seeded N(0, 0.02) weights (BASELINE.json configs: "weights N(0,0.02) from seed 0").

Canonical layout: every matrix is [out, in] (y = x @ W.T). Norm scales are 1
(or 1 + N(0, 0.1) when `norm_jitter` is set, to exercise the scale paths); the
positional-FFN bias b_P is N(0, 0.02) so the bias path is exercised.
Per-tensor generator seeds are derived from (seed, tensor index); draws are made
with torch.Generator on `device` (values therefore depend on the device used;
every test feeds ONE generated set to both sides).

Names (l = base layer index):
  embed [V,d]; layers.l.{attn_norm[d], wq[Hq*hd,d], wk[Hkv*hd,d], wv[Hkv*hd,d],
  wo[d,Hq*hd], ffn_norm[d], w_gate[F,d], w_up[F,d], w_down[d,F]}; final_norm[d];
  lm_head[V,d]; sf.group_scale[4,d]; sf.w_d[d,4d]; sf.ctx_norm[d]; sf.ctx_wq/wk/wv/wo;
  sf.pos_norm[d]; sf.w_p[k*d,d]; sf.b_p[k*d]; sf.blk_attn_norm[d]; sf.blk_wq/wk/wv/wo;
  sf.blk_ffn_norm[d]; sf.blk_w_gate[F,d]; sf.blk_w_up[F,d]; sf.blk_w_down[d,F].
"""
from __future__ import annotations

from collections import OrderedDict

import torch

from .configs import ModelConfig

_NORMS = ("attn_norm", "ffn_norm", "final_norm", "group_scale", "ctx_norm",
          "pos_norm", "blk_attn_norm", "blk_ffn_norm")


def _attn_shapes(prefix: str, c: ModelConfig):
    d, hq, hkv, hd = c.d_model, c.n_heads, c.n_kv_heads, c.head_dim
    return [(f"{prefix}wq", (hq * hd, d)), (f"{prefix}wk", (hkv * hd, d)),
            (f"{prefix}wv", (hkv * hd, d)), (f"{prefix}wo", (d, hq * hd))]


def weight_shapes(c: ModelConfig, n_layers: int | None = None):
    """Ordered (name, shape) list. `n_layers` may restrict to a prefix of layers."""
    L = c.n_layers if n_layers is None else n_layers
    d, F, V, k = c.d_model, c.d_ff, c.vocab, c.draft_len
    out = [("embed", (V, d))]
    for l in range(L):
        p = f"layers.{l}."
        out.append((p + "attn_norm", (d,)))
        out += _attn_shapes(p, c)
        out += [(p + "ffn_norm", (d,)), (p + "w_gate", (F, d)), (p + "w_up", (F, d)),
                (p + "w_down", (d, F))]
    out += [("final_norm", (d,)), ("lm_head", (V, d))]
    out += [("sf.group_scale", (4, d)), ("sf.w_d", (d, 4 * d)), ("sf.ctx_norm", (d,))]
    out += _attn_shapes("sf.ctx_", c)
    out += [("sf.pos_norm", (d,)), ("sf.w_p", (k * d, d)), ("sf.b_p", (k * d,)),
            ("sf.blk_attn_norm", (d,))]
    out += _attn_shapes("sf.blk_", c)
    out += [("sf.blk_ffn_norm", (d,)), ("sf.blk_w_gate", (F, d)), ("sf.blk_w_up", (F, d)),
            ("sf.blk_w_down", (d, F))]
    for i in range(1, getattr(c, "draft_blocks", 1)):  # NEXT-2 "+Larger": appended, earlier seeds unchanged
        b = f"sf.blk{i}_"
        out.append((b + "attn_norm", (d,)))
        out += _attn_shapes(b, c)
        out += [(b + "ffn_norm", (d,)), (b + "w_gate", (F, d)), (b + "w_up", (F, d)), (b + "w_down", (d, F))]
    return out


def _is_norm(name: str) -> bool:
    leaf = name.rsplit(".", 1)[-1]
    return leaf in _NORMS or (leaf.startswith("blk") and leaf.split("_", 1)[-1] in _NORMS)


def make_weights(c: ModelConfig, seed: int = 0, device="cpu", norm_jitter: float = 0.0,
                 std: float = 0.02, names=None, n_layers: int | None = None,
                 dtype: torch.dtype | None = None) -> "OrderedDict[str, torch.Tensor]":
    """Generate the weight dict. dtype defaults to fp32 for c.dtype=='fp32' and bf16
    (round-to-nearest-even cast of the fp32 draw) for 'bf16'."""
    if dtype is None:
        dtype = torch.float32 if c.dtype == "fp32" else torch.bfloat16
    out = OrderedDict()
    for idx, (name, shape) in enumerate(weight_shapes(c, n_layers)):
        if names is not None and name not in names:
            continue
        g = torch.Generator(device=device)
        g.manual_seed(seed * 1_000_003 + idx)
        if _is_norm(name):
            if norm_jitter:
                t = 1.0 + norm_jitter * torch.randn(shape, generator=g, device=device)
            else:
                t = torch.ones(shape, device=device)
        else:
            t = std * torch.randn(shape, generator=g, device=device)
        out[name] = t.to(dtype)
    return out
