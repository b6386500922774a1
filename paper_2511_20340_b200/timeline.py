"""Kernel timeline analysis (host side, numpy only).

Every kernel of the hot path carries a probe (csrc/common.cuh KtScope / kt_item) that, when the
timeline is on (sf_debug_ktrace_enable / SF_KTRACE=1), appends one 40-byte record per CTA:
{kind << 24 | param, smid, start_ns, dependency_resolved_ns, end_ns, 0} (%globaltimer). This module
groups the records into launches and attributes the step's critical path to them: a launch's
*exposed* time is the part of [dependency resolved, end] that does not overlap the launches before
it, so the exposed times plus the idle gaps add up to the traced span.
"""
from __future__ import annotations

import collections

import numpy as np

KIND = {1: "gemm", 2: "resid_norm", 3: "rope", 4: "attn", 5: "rmsnorm", 6: "group_rms", 7: "embed", 8: "argmax_p",
        9: "argmax_f", 10: "accept", 11: "bidir", 12: "gather", 13: "rows", 14: "gemm_simt", 15: "attn_part",
        16: "attn_comb", 17: "misc", 18: "item", 19: "gemm_seq"}
KT_ITEM = 18
REC = np.dtype([("kid", "<u4"), ("sm", "<u4"), ("t0", "<u8"), ("tw", "<u8"), ("t1", "<u8"), ("pad", "<u8")])
# kernel classes of the bench roofline (same split as sf_profile_read)
CLASS = {"gemm": "gemm", "gemm_simt": "gemm", "gemm_seq": "gemm", "attn": "attention", "rope": "attention", "attn_part": "attention",
         "attn_comb": "attention", "resid_norm": "norm", "rmsnorm": "norm", "group_rms": "norm", "embed": "norm",
         "gather": "norm", "rows": "norm"}


def name(kid: int) -> str:
    k, p = kid >> 24, kid & 0xFFFFFF
    n = KIND.get(k, str(k))
    return f"{n}[N={p & 0x7FFF},K={64 * (p >> 15)}]" if n == "gemm" else n


def kclass(kid: int) -> str:
    return CLASS.get(KIND.get(kid >> 24, ""), "argmax")


def launches(rec: np.ndarray) -> list[dict]:
    """CTA records (no KT_ITEM) -> launches, ordered by dependency-resolved time. Records of one
    kernel kind belong to the same launch while they overlap it (launches of one kind never overlap:
    every kernel waits for its predecessor's completion before its main work)."""
    rec = np.sort(rec, order="t0")
    open_, out = {}, []
    for r in rec:
        k = int(r["kid"])
        L = open_.get(k)
        if L is None or r["t0"] > L["t1"]:
            L = {"kid": k, "t0": int(r["t0"]), "tw": int(r["tw"]), "t1": int(r["t1"]), "n": 0}
            open_[k] = L
            out.append(L)
        L["tw"] = min(L["tw"], int(r["tw"]))
        L["t1"] = max(L["t1"], int(r["t1"]))
        L["n"] += 1
    return sorted(out, key=lambda L: L["tw"])


def critical_path(rec: np.ndarray, key=name) -> dict:
    """Exposed time (us), dependency->end duration (us) and count per key, idle gaps, span."""
    rec = rec[(rec["kid"] >> 24) != KT_ITEM]
    Ls = launches(rec)
    if not Ls:
        return {"span_us": 0.0, "gap_us": 0.0, "exposed": {}, "dur": {}, "count": {}, "launches": 0}
    t_first = Ls[0]["tw"]
    exposed, dur, cnt = collections.defaultdict(float), collections.defaultdict(float), collections.Counter()
    gap, run_end = 0.0, t_first
    for L in Ls:
        s = max(L["tw"], run_end)
        if L["tw"] > run_end:
            gap += (L["tw"] - run_end) / 1e3
        kk = key(L["kid"])
        exposed[kk] += max(0, L["t1"] - s) / 1e3
        dur[kk] += (L["t1"] - L["tw"]) / 1e3
        cnt[kk] += 1
        run_end = max(run_end, L["t1"])
    span = (max(L["t1"] for L in Ls) - t_first) / 1e3
    return {"span_us": span, "gap_us": gap, "exposed": dict(exposed), "dur": dict(dur), "count": dict(cnt),
            "launches": len(Ls), "_launches": Ls, "_t_first": t_first}


def spans_between(rec: np.ndarray, start_kid: int, end_kind: int) -> list[float]:
    """Per occurrence: dependency release of a launch with kid == start_kid -> dependency release of
    the next launch of kind end_kind (us). E.g. the verify forward of a decode step: the verify-row
    builder (kind 13, param 0) to the accept kernel (kind 10)."""
    Ls = launches(rec[(rec["kid"] >> 24) != KT_ITEM])
    out, start = [], None
    for L in Ls:
        if L["kid"] == start_kid:
            start = L["tw"]
        elif (L["kid"] >> 24) == end_kind and start is not None:
            out.append((L["tw"] - start) / 1e3)
            start = None
    return out
