"""NEXT-3 host-side model check of the fused all-reduce's exchange protocol.

The device path (csrc/gemm.cu: EPI_STORE_ACT with GemmEpi::out_sel, tp_signal_kernel, resid_norm_kernel
with a TpSrc) runs, per rank and per all-reduce i, in stream order:

  GEMM_i    writes this rank's slot (ctr + 1) & 1            (ctr = epochs published so far)
  signal_i  ctr += 1; publishes epoch ctr into every peer's flag for this rank
  consume_i waits until every peer's flag >= ctr, then reads every rank's slot ctr & 1

This test executes that program for tp ranks under random interleavings (one step of one rank at a time,
a rank's consumer blocked until its wait is satisfied) and checks the two properties the two-slot design
relies on: no rank ever overwrites a slot that a peer has not finished reading for an earlier all-reduce,
and every consumer reads exactly the values the ranks produced for the same all-reduce. A one-slot variant
must violate the first property (so the check is not vacuous)."""
import random

import pytest


def _run(tp, n_ar, seed, n_slots=2):
    rng = random.Random(seed)
    slot_val = [[None] * n_slots for _ in range(tp)]      # slot contents: (rank, all-reduce index)
    readers = [[set() for _ in range(n_slots)] for _ in range(tp)]  # (reader, i) still to read slot
    flags = [[0] * tp for _ in range(tp)]                 # flags[owner][q]: epoch rank q published to owner
    ctr = [0] * tp
    pc = [0] * tp                                         # next op: 3 i + {0 GEMM, 1 signal, 2 consume}
    violations = []
    while any(p < 3 * n_ar for p in pc):
        r = rng.choice([q for q in range(tp) if pc[q] < 3 * n_ar])
        i, op = divmod(pc[r], 3)
        if op == 0:                                       # GEMM_i: this rank's slot of the coming epoch
            s = ((ctr[r] + 1) & 1) if n_slots == 2 else 0
            for (reader, j) in readers[r][s]:
                if j < i:
                    violations.append(("overwrite", r, i, reader, j))
            slot_val[r][s] = (r, i)
            readers[r][s] = {(q, i) for q in range(tp)}
        elif op == 1:                                     # signal_i
            ctr[r] += 1
            for q in range(tp):
                flags[q][r] = ctr[r]
        else:                                             # consume_i: blocked until every peer published
            e = ctr[r]
            if any(flags[r][q] < e for q in range(tp) if q != r):
                continue
            s = (e & 1) if n_slots == 2 else 0
            got = [slot_val[q][s] for q in range(tp)]
            if got != [(q, i) for q in range(tp)]:
                violations.append(("read", r, i, got))
            for q in range(tp):
                readers[q][s].discard((r, i))
        pc[r] += 1
    return violations


@pytest.mark.parametrize("tp", [2, 3, 4, 8])
def test_two_slot_exchange_is_safe(tp):
    for seed in range(200):
        assert _run(tp, n_ar=7, seed=seed) == []  # 7: an odd count, as in a decode step (2 L + 5)


def test_one_slot_exchange_races():
    assert any(_run(2, n_ar=7, seed=s, n_slots=1) for s in range(200))
