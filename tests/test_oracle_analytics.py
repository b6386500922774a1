"""Pins of the paper's evaluation calculus (§AI, P68-105) against printed values."""
import json
import os

import pytest

from oracle import analytics as A
from synth import get_config

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_eq1_ai_model():
    assert A.ai_model(7e9, 2) == GOLD["ai_model_bf16"]["value"]
    assert A.ai_model(123, 4) == 0.5


def test_eq2_ai_chip_a100():
    g = GOLD["ai_chip_a100"]
    assert abs(A.ai_chip(g["peak_tflops"] * 1e12, g["bw_tbs"] * 1e12) - g["value"]) < g["tol"]
    rho = A.redundancy(A.ai_chip(311.84e12, 2.04e12), A.ai_model(1, 2))
    assert abs(rho - 152.86) < 0.005


def test_eq3_budget():
    rho = 311.84 / 2.04
    assert A.gain_and_budget(2, 1, 1, 8, rho, 16)[2] is True     # 8 <= 9.55
    assert A.gain_and_budget(2, 1, 1, 8, rho, 32)[2] is False    # 8 > 4.78
    assert A.gain_and_budget(2, 1, 1, 4, rho, 1)[0] == 2


def test_eq4_overhead():
    assert A.overhead_factor(1000, 100, 25, 4) == pytest.approx(1.2)
    assert A.overhead_factor(10, 0, 0, 8) == 1.0


@pytest.mark.parametrize("row", GOLD["kappa_examples"])
def test_eq5_kappa(row):
    assert A.kappa(row["a"], row["l_d"], row["k"]) == row["kappa"]


@pytest.mark.parametrize("row", GOLD["theta_rows"])
def test_theta_table3(row):
    assert abs(A.theta(row["kappa"], row["tps_sd"], row["tps_base"]) - row["theta"]) < 0.005


def test_positional_params():
    g = GOLD["positional_params"]
    cfg = get_config("tiny").replace(d_model=g["d_h"], draft_len=g["l_d"])
    m_s, m_p = A.draft_param_counts(cfg)
    assert g["l_d"] * m_p == g["value"]
    # exhaustive shape walk of the synth weight table's sf.* tensors equals m_s + l_d m_p
    from synth import weight_shapes
    import math
    tot = sum(math.prod(s) for n, s in weight_shapes(cfg) if n.startswith("sf."))
    assert tot == m_s + cfg.draft_len * m_p
