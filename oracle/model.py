"""TEST INFRASTRUCTURE ONLY. fp64 NumPy oracle of the SpecFormer decode step.

Citations: P<n> = PAPER.md line n (arXiv 2511.20340 LaTeX source); S<n> = SPEC.md
line n (interface ideas only). Readings C1..C23 are SURVEY.md §8(c)'s and are
restated in DESIGN.md §3. Everything is float64; weights arrive as whatever the
caller generated (fp32, or bf16 upcast exactly -- reading C17).

Every function is a direct transcription of its definition; no blocking, fusion or
reordering. Rows of a block are pushed through one matmul (a library primitive);
attention is materialised as the full masked score matrix per head.
"""
from __future__ import annotations

import time

import numpy as np


# --------------------------------------------------------------------------- weights
class Weights:
    """Lazily upcasts a {name: tensor/ndarray} dict to float64 NumPy arrays."""

    def __init__(self, cfg, tensors):
        self.cfg = cfg
        self._src = tensors
        self._cache = {}

    def __getitem__(self, name):
        a = self._cache.get(name)
        if a is None:
            t = self._src[name]
            if hasattr(t, "detach"):  # torch tensor (bf16/fp32) -> exact fp32 -> fp64
                t = t.detach().float().cpu().numpy()
            a = np.asarray(t, dtype=np.float64)
            self._cache[name] = a
        return a


# --------------------------------------------------------------------------- primitives
def rms_norm(x, g, eps):
    """RMSNorm over the last axis: x / sqrt(mean(x^2) + eps) * g.
    P173 ("root-mean-square normalization"); eps reading C3; S53."""
    x = np.asarray(x, dtype=np.float64)
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * g


def group_rms_norm(taps, scales, eps):
    """Grouped RMS Norm (P177): RMSNorm over the last dim of each of the 4 tap
    slices with its own scale vector, then reshape [.., 4, d] -> [.., 4d]
    (I_Cat, Eq.8 second line P186). taps: [4, T, d]; scales: [4, d] -> [T, 4d]."""
    return np.concatenate([rms_norm(taps[g], scales[g], eps) for g in range(taps.shape[0])], axis=-1)


def rope(x, pos, theta):
    """Rotary embedding, rotate-half convention (reading C5): pair (i, i + hd/2),
    angle = pos * theta^(-2i/hd). x: [T, H, hd]; pos: [T] absolute 0-based."""
    hd = x.shape[-1]
    half = hd // 2
    inv = theta ** (-2.0 * np.arange(half, dtype=np.float64) / hd)
    ang = np.asarray(pos, dtype=np.float64)[:, None] * inv[None, :]
    cos, sin = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * cos - x2 * sin, x2 * cos + x1 * sin], axis=-1)


def attention_dense_masked(q, k, v, mask):
    """softmax(q k^T / sqrt(hd) + M) v with M = -inf where mask is False (S77-81).
    q: [nq, hd]; k, v: [nk, hd]; mask: [nq, nk] bool (True = visible). A fully
    masked row is an error (reading C22)."""
    mask = np.asarray(mask, dtype=bool)
    if not mask.any(axis=1).all():
        raise ValueError("fully-masked attention row")
    s = (q @ k.T) / np.sqrt(q.shape[-1])
    s = np.where(mask, s, -np.inf)
    s = s - s.max(axis=1, keepdims=True)
    p = np.exp(s)
    p = p / p.sum(axis=1, keepdims=True)
    return p @ v


def silu(z):
    return z / (1.0 + np.exp(-z))


def swiglu(x, w_gate, w_up, w_down):
    """SwiGLU FFN: W_down (silu(W_gate x) * (W_up x)) (P197; S86-89)."""
    return (silu(x @ w_gate.T) * (x @ w_up.T)) @ w_down.T


def argmax_lowest(v):
    """Greedy token: argmax with ties broken toward the lowest id (reading C13; S180-188).
    np.argmax returns the first maximum. Non-finite input is an error (S26)."""
    v = np.asarray(v)
    if not np.all(np.isfinite(v)):
        raise FloatingPointError("non-finite logits")
    return int(np.argmax(v))


def taps_index(L):
    """Hook layers HS[0], HS[L/2], HS[L-1], HS[L] (P175) with floor(L/2) (reading C1)."""
    return (0, L // 2, L - 1, L)


# --------------------------------------------------------------------------- KV cache
class KVCache:
    """Dense per-layer K/V (layers 0..L-1 base, layer L = SpecFormer context layer,
    "an additional (L+1)-th layer of the LLM", P177). Each layer keeps its own length;
    rollback is truncation (S198-206)."""

    def __init__(self, n_layers_total, n_kv_heads, head_dim):
        self.K = [np.zeros((n_kv_heads, 0, head_dim)) for _ in range(n_layers_total)]
        self.V = [np.zeros((n_kv_heads, 0, head_dim)) for _ in range(n_layers_total)]

    def length(self, layer):
        return self.K[layer].shape[1]

    def append(self, layer, k_new, v_new, pos0):
        """k_new, v_new: [T, Hkv, hd] at positions pos0..pos0+T-1."""
        if self.length(layer) != pos0:
            raise ValueError(f"cache misalignment: layer {layer} len {self.length(layer)} != pos {pos0}")
        self.K[layer] = np.concatenate([self.K[layer], k_new.transpose(1, 0, 2)], axis=1)
        self.V[layer] = np.concatenate([self.V[layer], v_new.transpose(1, 0, 2)], axis=1)

    def truncate(self, layers, n):
        for l in layers:
            if n > self.length(l):
                raise ValueError("truncate beyond length")
            self.K[l] = self.K[l][:, :n]
            self.V[l] = self.V[l][:, :n]


def _attn(W, prefix, x, pos, cache, layer, causal=True, slot_causal=False, ctx_prefix=None):
    """Multi-head attention sub-block on normalised input x [T, d].
    With `cache`: RoPE at absolute positions, append K/V, attend causally over the
    cached prefix + the new rows (query i at position p_i sees keys at <= p_i).
    Without cache (draft block, P204): no RoPE, all-to-all over the T rows -- or, with
    slot_causal (the "+Att Mask" ablation, T4 P497-514), row i sees rows <= i only.
    ctx_prefix = (K, V, n) (the BIDIR_PREFIX draft variant): the T draft slots sit
    at positions n..n+T-1 (queries and keys rotated there) and every slot sees the n cached
    context-layer keys [Hkv, n, hd] (positions 0..n-1) and all T slots.
    GQA: query head h reads kv head floor(h * Hkv / Hq)."""
    c = W.cfg
    T = x.shape[0]
    hq, hkv, hd = c.n_heads, c.n_kv_heads, c.head_dim
    q = (x @ W[prefix + "wq"].T).reshape(T, hq, hd)
    k = (x @ W[prefix + "wk"].T).reshape(T, hkv, hd)
    v = (x @ W[prefix + "wv"].T).reshape(T, hkv, hd)
    if ctx_prefix is not None:
        PK, PV, n = ctx_prefix
        spos = n + np.arange(T)
        q = rope(q, spos, c.rope_theta)
        k = rope(k, spos, c.rope_theta)
        K = np.concatenate([PK[:, :n], k.transpose(1, 0, 2)], axis=1)
        V = np.concatenate([PV[:, :n], v.transpose(1, 0, 2)], axis=1)
        mask = np.ones((T, n + T), dtype=bool)
    elif cache is not None:
        q = rope(q, pos, c.rope_theta)
        k = rope(k, pos, c.rope_theta)
        cache.append(layer, k, v, int(pos[0]))
        K, V = cache.K[layer], cache.V[layer]
        keypos = np.arange(K.shape[1])
        mask = keypos[None, :] <= np.asarray(pos)[:, None]
    else:
        K, V = k.transpose(1, 0, 2), v.transpose(1, 0, 2)
        mask = np.tril(np.ones((T, T), dtype=bool)) if slot_causal else np.ones((T, T), dtype=bool)
    out = np.empty((T, hq, hd))
    for h in range(hq):
        g = (h * hkv) // hq
        out[:, h, :] = attention_dense_masked(q[:, h, :], K[g], V[g], mask)
    return out.reshape(T, hq * hd) @ W[prefix + "wo"].T


# --------------------------------------------------------------------------- base model
def decoder_layer(W, l, h, pos, cache):
    """Base decoder layer l (0-based) on the residual stream h [T, d] at positions pos: the
    pre-norm block of Eq.7 (P160-165), h += Attn(RMS(h)); h += SwiGLU(RMS(h)). Returns HS[l+1]."""
    eps = W.cfg.rms_eps
    p = f"layers.{l}."
    h = h + _attn(W, p, rms_norm(h, W[p + "attn_norm"], eps), pos, cache, l)
    return h + swiglu(rms_norm(h, W[p + "ffn_norm"], eps), W[p + "w_gate"], W[p + "w_up"], W[p + "w_down"])


def base_forward(W, tokens, pos0, cache):
    """Base decoder forward over `tokens` at positions pos0.. (pre-norm blocks, Eq.7
    P160-165: h += Attn(RMS(h)); h += SwiGLU(RMS(h))). Returns (logits [T, V],
    taps [4, T, d]) with HS[0] = Embedding, HS[l] = residual after layer l, taps
    per P175 / reading C1, HS[L] taken before the final norm (reading C2)."""
    c = W.cfg
    L, eps = c.n_layers, c.rms_eps
    tokens = np.asarray(tokens, dtype=np.int64)
    T = tokens.shape[0]
    pos = pos0 + np.arange(T)
    h = W["embed"][tokens].copy()
    hs = [h.copy()]
    for l in range(L):
        h = decoder_layer(W, l, h, pos, cache)
        hs.append(h.copy())
    logits = rms_norm(h, W["final_norm"], eps) @ W["lm_head"].T
    taps = np.stack([hs[i] for i in taps_index(L)])
    return logits, taps


# --------------------------------------------------------------------------- SpecFormer
def context_layer(W, taps, pos0, cache):
    """Context Causal Attention, Eq.8 (P179-188):
        I_Cat = GroupRMS(HS[0, L/2, L-1, L]);  X = W_D I_Cat (no bias, P177);
        I_D = (MSA . RMS + I)(X) = X + MSA(RMS(X)),
    MSA causal over context positions with its own KV cache = layer L (P177), RoPE at
    the base positions (reading C5), base head layout (C4). taps: [4, T, d]."""
    c = W.cfg
    eps = c.rms_eps
    T = taps.shape[1]
    pos = pos0 + np.arange(T)
    icat = group_rms_norm(taps, W["sf.group_scale"], eps)
    X = icat @ W["sf.w_d"].T
    return X + _attn(W, "sf.ctx_", rms_norm(X, W["sf.ctx_norm"], eps), pos, cache, c.n_layers)


def positional_ffn(W, i_d):
    """Positional FFN, Eq.9 (P189-193): D = W_P RMS(I_D) + b_P, W_P: d -> l_d*d,
    reshaped so slot j takes output rows [j*d, (j+1)*d). i_d: [d] -> D: [k, d].
    cfg.no_pos_ffn (the T4 "-Pos" ablation, P499 / P189 -- DESIGN.md §3 reading): W_P removed, each
    slot gets the same normalised row plus its own position vector, D_j = RMS(I_D) + b_P[j]
    ("assigning a basic mask per position")."""
    c = W.cfg
    r = rms_norm(i_d, W["sf.pos_norm"], c.rms_eps)
    if getattr(c, "no_pos_ffn", False):
        return np.tile(r, c.draft_len).reshape(c.draft_len, c.d_model) + W["sf.b_p"].reshape(c.draft_len, c.d_model)
    y = W["sf.w_p"] @ r + W["sf.b_p"]
    return y.reshape(c.draft_len, c.d_model)


def draft_block(W, D, slot_causal=False, ctx_prefix=None):
    """Draft Bi-directional Attention layer, Eq.10 (P197-204):
        E = (SwiGLU . RMS + I)((SA . RMS + I)(D)),
    SA unmasked along the l_d draft slots, no positional encoding (reading C6).
    slot_causal: the T4 "+Att Mask" ablation (P497-514) -- slot j attends slots <= j.
    cfg.draft_blocks > 1: the T4 "+Larger" ablation read as that many such layers applied in turn
    (weights sf.blk_* then sf.blk<i>_*). ctx_prefix: the BIDIR_PREFIX variant (see _attn).
    D: [k, d] -> E: [k, d]."""
    eps = W.cfg.rms_eps
    E = D
    for i in range(max(1, getattr(W.cfg, "draft_blocks", 1))):
        b = "sf.blk_" if i == 0 else f"sf.blk{i}_"
        Y = E + _attn(W, b, rms_norm(E, W[b + "attn_norm"], eps), None, None, None, slot_causal=slot_causal,
                      ctx_prefix=ctx_prefix)
        E = Y + swiglu(rms_norm(Y, W[b + "ffn_norm"], eps), W[b + "w_gate"], W[b + "w_up"], W[b + "w_down"])
    return E


def draft_logits(W, i_d, slot_causal=False, ctx_prefix=None):
    """Draft logits for one context row: positional FFN -> draft block -> frozen base
    final norm + LM head, shared (reading C8). Returns [k, V]."""
    E = draft_block(W, positional_ffn(W, i_d), slot_causal, ctx_prefix)
    return rms_norm(E, W["final_norm"], W.cfg.rms_eps) @ W["lm_head"].T


def draft_tokens(W, i_d):
    """Chain draft of k tokens in parallel (P6, P37: no prefix tree)."""
    return [argmax_lowest(r) for r in draft_logits(W, i_d)]


# --------------------------------------------------------------------------- accept
def accept(draft, greedy):
    """Lossless greedy acceptance (P23, P25: "only draft tokens that exactly match the
    outputs of the large model"). draft: k ints; greedy: k+1 ints (greedy[i] is the
    base prediction after verify input i). m = length of the longest prefix with
    draft[i] == greedy[i]; emitted = greedy[0..m] (m matches + the bonus token)."""
    m = 0
    while m < len(draft) and int(draft[m]) == int(greedy[m]):
        m += 1
    return m, [int(t) for t in greedy[: m + 1]]


# --------------------------------------------------------------------------- loops
def _new_cache(c):
    return KVCache(c.n_layers + 1, c.n_kv_heads, c.head_dim)


def _ctx_prefix(W, cache, n):
    """The BIDIR_PREFIX draft variant's prefix: the context layer's (layer L) cached K / V of the n
    committed positions; None for the paper's draft block."""
    if not getattr(W.cfg, "draft_prefix", False):
        return None
    L = W.cfg.n_layers
    return cache.K[L][:, :n], cache.V[L][:, :n], n


def prefill(W, prompt, cache):
    """Setup pass (reading C11): base forward over the P prompt tokens, context layer
    over all P rows. Returns (g0, I_D row P-1, logits [P, V])."""
    logits, taps = base_forward(W, prompt, 0, cache)
    i_d = context_layer(W, taps, 0, cache)
    return argmax_lowest(logits[-1]), i_d[-1], logits


def decode_greedy(W, prompt, n_tokens):
    """Plain autoregressive greedy decoding of the base model: the result lossless SD
    must reproduce exactly (P25-26; S189-197)."""
    c = W.cfg
    cache = _new_cache(c)
    P = len(prompt)
    if n_tokens == 0:
        return []
    logits, _ = base_forward(W, prompt, 0, cache)
    out = [argmax_lowest(logits[-1])]
    while len(out) < n_tokens:
        logits, _ = base_forward(W, [out[-1]], P + len(out) - 1, cache)
        out.append(argmax_lowest(logits[0]))
    return out


def sd_decode(W, prompt, n_tokens, draft_fn=None, record=False, step_times=None):
    """SpecFormer speculative decoding, the three-step protocol of P20-23:
      1. draft k tokens from the context layer's row for the newest committed position
         (draft_fn(step, n, out) may override, e.g. perfect or adversarial drafts);
      2. verify [last_token, d_1..d_k] in ONE base forward at positions n..n+k, keeping
         its hidden-state taps ("extracting and storing information for the next round");
      3. accept (m, emitted); commit n += m + 1 (rollback = truncation of layers 0..L-1),
         run the context layer over the m+1 committed verify rows (C14), next draft row
         = I_D[m].
    Stops once >= n_tokens are emitted and trims the overshoot (reading C15; S400).
    Returns (tokens, steps) where steps lists per-step dicts when record=True. step_times (a list,
    optional; bench.py's CPU baseline) receives each step's wall time -- timing only, no arithmetic."""
    c = W.cfg
    L = c.n_layers
    cache = _new_cache(c)
    P = len(prompt)
    g0, i_d, _ = prefill(W, prompt, cache)
    out, n, last = [g0], P, g0
    steps = []
    while len(out) < n_tokens:
        t_step = time.perf_counter() if step_times is not None else 0.0
        dl = None
        if draft_fn is None:
            dl = draft_logits(W, i_d, ctx_prefix=_ctx_prefix(W, cache, n))
            dr = [argmax_lowest(r) for r in dl]
        else:
            dr = [int(t) for t in draft_fn(len(steps), n, list(out))]
        logits, taps = base_forward(W, [last] + dr, n, cache)
        greedy = [argmax_lowest(r) for r in logits]
        m, emitted = accept(dr, greedy)
        cache.truncate(range(L), n + m + 1)
        i_d = context_layer(W, taps[:, : m + 1], n, cache)[m]
        if record:
            steps.append(dict(n=n, draft=dr, greedy=greedy, m=m, logits=logits, draft_logits=dl, i_d=i_d))
        else:
            steps.append(dict(m=m))
        out += emitted
        last = greedy[m]
        n += m + 1
        if step_times is not None:
            step_times.append(time.perf_counter() - t_step)
    return out[:n_tokens], steps


def replay(W, prompt, gpu_steps, slot_causal=False):
    """Teacher-forced oracle along a trajectory produced elsewhere (the GPU's).
    gpu_steps: list of dicts with 'draft' (k ints), 'm' (accept length) and 'last'
    (the verify block's first token). At each step the oracle verifies the SAME block,
    returns its own logits / greedy tokens, its own draft logits for that step (from
    its own context-layer row), then commits the GPU's m. Returns (g0 oracle logits row,
    list of per-step dicts)."""
    c = W.cfg
    L = c.n_layers
    cache = _new_cache(c)
    P = len(prompt)
    g0, i_d, plog = prefill(W, prompt, cache)
    n = P
    res = []
    for st in gpu_steps:
        dl = draft_logits(W, i_d, slot_causal, _ctx_prefix(W, cache, n))
        dr = [int(t) for t in st["draft"]]
        logits, taps = base_forward(W, [int(st["last"])] + dr, n, cache)
        m = int(st["m"])
        cache.truncate(range(L), n + m + 1)
        i_d = context_layer(W, taps[:, : m + 1], n, cache)[m]
        res.append(dict(n=n, logits=logits, greedy=[argmax_lowest(r) for r in logits], draft_logits=dl))
        n += m + 1
    return plog[-1], res


def top2_margin(row):
    """top-1 minus top-2 logit (the margin rule of reading C21)."""
    s = np.sort(np.asarray(row, dtype=np.float64))
    return float(s[-1] - s[-2])
