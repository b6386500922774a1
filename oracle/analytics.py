"""TEST INFRASTRUCTURE ONLY. The paper's evaluation calculus (§AI, P68-105), as written.

Pinned by tests/test_oracle_analytics.py against the values the paper prints
(Eq.1 = 1, Eq.2 = 152.86) and Table 3 rows (theta).
"""
from __future__ import annotations


def ai_model(M, bytes_per_param):
    """Eq.1 (P72-78): AI_m = 2M / (bytes * M)."""
    if M <= 0 or bytes_per_param <= 0:
        raise ValueError("nonpositive")
    return 2.0 * M / (bytes_per_param * M)


def ai_chip(peak_flops, bandwidth):
    """Eq.2 (P81-86): AI_c = peak FLOP/s / memory bandwidth."""
    if peak_flops <= 0 or bandwidth <= 0:
        raise ValueError("nonpositive")
    return peak_flops / bandwidth


def redundancy(ai_c, ai_m):
    """rho = AI_c / AI_m (P87)."""
    return ai_c / ai_m


def overhead_factor(M, m_s, m_p, l_d):
    """Eq.4 (P96-99): p = 1 + (m_s + l_d m_p) / M."""
    if M <= 0:
        raise ValueError("M <= 0")
    return 1.0 + (m_s + l_d * m_p) / M


def gain_and_budget(a, p, ai_m, k, rho, bs):
    """Eq.3 (P91-95): r1 = (a/p) AI_m; r2 = k; feasible iff k <= rho / bs."""
    return (a / p) * ai_m, k, k <= rho / bs


def kappa(a, l_d, k):
    """Eq.5 (P101-105): kappa = a l_d / k."""
    if k < 1:
        raise ValueError("k < 1")
    return a * l_d / k


def theta(kap, tps_sd, tps_base):
    """kappa-to-TPS conversion ratio (P493; reading C18): kappa / (tps_sd / tps_base)."""
    if tps_base <= 0:
        raise ValueError("tps_base <= 0")
    return kap / (tps_sd / tps_base)


def draft_param_counts(cfg):
    """(m_s, m_p) of Eq.4 for the SpecFormer head: positional params l_d (d^2 + d)
    (P189: "l_d * d_h^2", plus the bias b_P), m_s = everything else in the head."""
    d, F, hq, hkv, hd = cfg.d_model, cfg.d_ff, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    attn = d * hq * hd + 2 * d * hkv * hd + hq * hd * d
    m_s = 4 * d + 4 * d * d + d + attn + d + d + attn + d + 3 * d * F
    m_p = d * d + d
    return m_s, m_p
