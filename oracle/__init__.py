"""TEST INFRASTRUCTURE ONLY -- the fp64 CPU oracle of SpecFormer speculative decoding.

A plain, slow, obviously-correct NumPy float64 implementation of what the hot path
computes, written from PAPER.md (arXiv 2511.20340) and the readings listed in
DESIGN.md §3. Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import it. The product path
(`paper_2511_20340_b200`) never imports it and shares no code with it; the only
shared module is `synth/` (seeded random inputs, no arithmetic of the method).

Parity-pin status: every function here is pinned by a `-m "not gpu"`
test against closed forms, SPEC.md worked examples, brute force or the
losslessness invariant, EXCEPT the draft head's numerics on random weights
(`draft_logits` composed end to end), which is "parity unpinned" beyond its
per-piece pins (residual identities, W_P = 0 => D = b_P, permutation equivariance).
"""
from .model import (  # noqa: F401
    Weights, rms_norm, group_rms_norm, rope, attention_dense_masked, swiglu, argmax_lowest,
    taps_index, KVCache, decoder_layer, base_forward, context_layer, positional_ffn, draft_block, top2_margin,
    draft_logits, draft_tokens, accept, decode_greedy, sd_decode, replay, prefill,
)
from . import analytics  # noqa: F401
