"""CPU oracle for the per-round hot path of EqSpec / EXSpec (arXiv 2510.22876).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_2510_22876_b200/)
may import, call or execute anything under oracle/.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg use it.

Plain, slow, obviously-correct numpy (fp64 where floating point is involved),
written from the paper's definitions in the paper's order:

    verify.py   Alg. 1 BatchVerify + the BatchRepad plan
    align.py    Alg. 2 Phase 3 unpad-append-repad + Realign,
                §3.1 invariants
    pool.py     Alg. 3 GetBatch / RefillWindow / write-back,
                §3.2
    toy_lm.py   SPEC.md toy_lm: fp64, left-to-right sums
    loops.py    Alg. 2 EqSpec and Alg. 3 EXSpec driven by the toy LM, plus the
                per-sequence autoregressive greedy reference
    metrics.py  §3.1 closed form, §4.1 exact/partial match

Shares no code with the CUDA path.  Pins live in tests/test_oracle_*.py and
tests/test_golden.py (hand-worked fixtures in tests/golden/).
Parity pin status per function is listed in DESIGN.md §"Oracle pins".
"""
