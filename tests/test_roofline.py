"""The bench's algorithmic byte / FLOP model (paper_2511_20340_b200/roofline.py) against the per-step
totals SURVEY §8(a) derives independently ("Totals per step" table: weights once per pass, KV once
per (sequence, layer), fp32 logits written and read once)."""
import pytest

from paper_2511_20340_b200 import roofline as R
from synth import get_config


def test_weight_bytes_7b():
    c = get_config("7b")
    w = (R.base_linear_params(c) + c.vocab * c.d_model) * 2 + (R.head_params(c, 4) + c.vocab * c.d_model) * 2
    assert w == pytest.approx(14.28e9, rel=2e-3)  # 14.28 GB of weights per step


@pytest.mark.parametrize("name,B,k,n,total,logits", [("7b", 1, 4, 655, 14.64e9, 2.3e6),
                                                     ("13b", 64, 4, 1152, 89.6e9, 147.5e6)])
def test_step_bytes_match_survey(name, B, k, n, total, logits):
    c = get_config(name)
    lens = [n] * B
    assert R.step_bytes(c, B, k, lens, lens) == pytest.approx(total, rel=2e-3)
    kv = R.attention_kv_bytes(c, lens, lens, k)
    w = (R.base_linear_params(c) + R.head_params(c, k) + 2 * c.vocab * c.d_model) * 2
    assert R.step_bytes(c, B, k, lens, lens) - w - kv == pytest.approx(logits, rel=1e-2)


def test_kv_bytes_per_token_and_layer():
    c = get_config("7b")
    assert R.kv_bytes_per_token_layer(c) == 16 * 1024  # K and V, 32 heads x 128 dims, bf16
    # verify over L base layers at n_b + k + 1 keys, context layer at n_prev + k + 1
    assert R.attention_kv_bytes(c, [10], [7], 4) == 16 * 1024 * (32 * 15 + 12)


def test_step_flops_dominated_by_2TNK():
    c = get_config("7b")
    B, k = 64, 4
    f = R.step_flops(c, B, k, [640] * B)
    lin = 2 * B * (k + 1) * (R.base_linear_params(c) + c.vocab * c.d_model)
    assert lin < f < 1.2 * lin  # 4.61 TF at 7B, B = 64
    assert f == pytest.approx(4.61e12, rel=3e-2)


def test_step_bytes_without_logits():
    """SF_FLAG_NO_LOGITS (fused LM-head argmax): the verify + draft rows' fp32 logits round trip is
    replaced by one 8-byte key per row, written and read."""
    c = get_config("7b")
    B, k, lens = 16, 4, [700] * 16
    rows = B * (k + 1) + B * k
    full, fused = R.step_bytes(c, B, k, lens, lens), R.step_bytes(c, B, k, lens, lens, logits=False)
    assert full - fused == rows * c.vocab * 4 * 2 - rows * 8 * 2
