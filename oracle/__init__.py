"""CPU oracle for the zkLLM tlookup prover hot path (arXiv 2404.16109).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s cpu_baseline / `--impl reference` leg may import, call, link or
execute anything under `oracle/`.  The product path
(`paper_2404_16109_b200/`) never imports it and shares no code with it: no
kernels, headers, helpers, constants or pre/post-processing.

Two tiers:

* `oracle.field`, `oracle.mle`, `oracle.tlookup` — plain Python big integers,
  the definitions written out (PAPER.md:164-170 Eq. MLE; PAPER.md:231-250
  Lemma / Eq. hab22-coefs / hab22-invs / tlookup-sumcheck; PAPER.md:181-183
  sumcheck).  Inverses use the library routine `pow(x, -1, r)`; round
  polynomials are evaluated directly at t = 0, 1, 2, 3 from D-sized vectors.
* `oracle.c` (C, 4 x 64-bit limbs, `unsigned __int128`) — the same algorithm
  for sizes Python cannot reach (C2..C5), cross-checked against the Python
  tier in `tests/test_oracle_c.py`.

Parity pins (what fixes the oracle to something other than itself) are listed
in DESIGN.md §4 and tested under `-m "not gpu"`.
"""
