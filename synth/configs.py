"""Shape presets from BASELINE.json:configs (Tiny, Small, 7B-, 13B-, 70B-shaped).

Pure data: layer counts, widths, head layout, vocabulary, draft length k (= l_d,
PAPER.md P101-105 Eq.5 with k = l_d), batch, prompt and generation lengths.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass


@dataclass(frozen=True)
class ModelConfig:
    name: str
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    d_ff: int
    vocab: int
    draft_len: int          # k = l_d
    dtype: str              # "fp32" | "bf16"
    batch: int
    prompt_len: int
    gen_len: int
    kv_block: int = 16
    draft_blocks: int = 1   # NEXT-2 "+Larger" (T4): stacked draft blocks, weights sf.blk<i>_* for i >= 1
    no_pos_ffn: bool = False   # NEXT-2 "-Pos" (T4): no W_P, D_j = RMS(I_D) + b_P[j]
    draft_prefix: bool = False  # NEXT-2 BIDIR_PREFIX: draft slots also attend the context layer's cache
    rope_theta: float = 10000.0
    rms_eps: float = 1e-6

    def replace(self, **kw) -> "ModelConfig":
        return dataclasses.replace(self, **kw)

    @property
    def max_seq(self) -> int:
        # prompt + generated + one verify block of overshoot (k+1), rounded to kv_block
        n = self.prompt_len + self.gen_len + self.draft_len + 1
        return ((n + self.kv_block - 1) // self.kv_block) * self.kv_block


PRESETS = {
    # BASELINE.json configs[0]
    "tiny": ModelConfig("tiny", 2, 64, 4, 4, 16, 256, 512, 4, "fp32", 1, 16, 32),
    # configs[1]
    "small": ModelConfig("small", 12, 768, 12, 12, 64, 3072, 32000, 4, "bf16", 8, 128, 128),
    # configs[2] (batch swept 1/16/64)
    "7b": ModelConfig("7b", 32, 4096, 32, 32, 128, 11008, 32000, 4, "bf16", 64, 512, 256),
    # configs[3] (k swept 4/6/8)
    "13b": ModelConfig("13b", 40, 5120, 40, 40, 128, 13824, 32000, 4, "bf16", 64, 1024, 256),
    # configs[4] (GQA; tensor-parallel in the paper-free build plan)
    "70b": ModelConfig("70b", 80, 8192, 64, 8, 128, 28672, 32000, 4, "bf16", 128, 2048, 128),
}


def get_config(name: str, **overrides) -> ModelConfig:
    cfg = PRESETS[name]
    return cfg.replace(**overrides) if overrides else cfg
