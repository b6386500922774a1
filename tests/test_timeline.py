"""Host-side kernel-timeline attribution (paper_2511_20340_b200/timeline.py), no GPU."""
import numpy as np

from paper_2511_20340_b200 import timeline as tl


def _rec(rows):
    r = np.zeros(len(rows), dtype=tl.REC)
    for i, (kind, param, t0, tw, t1) in enumerate(rows):
        r[i] = ((kind << 24) | param, 0, t0, tw, t1, 0)
    return r


def test_critical_path_partitions_span():
    # gemm launch (2 CTAs) 0..10us, overlapping resid_norm 8..14 (exposed 4), gap 14..15, attn 15..20,
    # a second gemm launch of the same kind 21..30 after another gap; an item record is ignored
    us = 1000
    g = 4096 | (64 << 15)  # gemm N = 4096, K = 4096
    rec = _rec([(1, g, 0, 0, 9 * us), (1, g, 1 * us, 1 * us, 10 * us), (2, 0, 5 * us, 8 * us, 14 * us),
                (4, 0, 15 * us, 15 * us, 20 * us), (1, g, 21 * us, 21 * us, 30 * us),
                (18, 7, 16 * us, 17 * us, 18 * us)])
    cp = tl.critical_path(rec)
    assert cp["launches"] == 4
    assert abs(cp["span_us"] - 30) < 1e-9 and abs(cp["gap_us"] - 2) < 1e-9
    assert abs(cp["exposed"]["gemm[N=4096,K=4096]"] - 19) < 1e-9 and cp["count"]["gemm[N=4096,K=4096]"] == 2
    assert abs(cp["exposed"]["resid_norm"] - 4) < 1e-9 and abs(cp["dur"]["resid_norm"] - 6) < 1e-9
    assert abs(sum(cp["exposed"].values()) + cp["gap_us"] - cp["span_us"]) < 1e-9
    by_class = tl.critical_path(rec, key=tl.kclass)
    assert set(by_class["exposed"]) == {"gemm", "norm", "attention"}


def test_spans_between():
    us = 1000
    rows, acc = 13 << 24, 10 << 24
    rec = _rec([(13, 0, 0, 1 * us, 2 * us), (1, 4096 | (64 << 15), 2 * us, 2 * us, 9 * us), (10, 4, 9 * us, 10 * us, 11 * us),
                (13, 1, 11 * us, 11 * us, 12 * us),  # prefill row builder: not a verify start
                (13, 0, 20 * us, 20 * us, 21 * us), (10, 4, 24 * us, 25 * us, 26 * us)])
    assert tl.spans_between(rec, rows, acc >> 24) == [9.0, 5.0]
