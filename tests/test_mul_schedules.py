"""Design checks of the two aligned-pair Montgomery schedules (csrc/fr.cuh fr_mul, csrc/g1.cuh fq_mul), host only:
the word-level simulators in tools/ model every PTX carry chain with 32-bit words and a carry flag, assert that the
chains whose carry-out the kernels drop never carry, and compare a b R^-1 mod p with Python integers on random and
extreme operands (a, b < p; the F_q schedule is not valid for an unreduced left operand, which is why the hash to
the field keeps the portable multiplication, fq_mul_wide_a)."""
import os
import random
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import sim_fq_mul  # noqa: E402
import sim_fr_mul  # noqa: E402


def test_fr_schedule():
    sim_fr_mul.main(400)


def test_fq_schedule():
    sim_fq_mul.main(400)


def test_fq_schedule_needs_reduced_operands():
    """a >= q (left operand unreduced) breaks the dropped-carry bound for some inputs: kept out of fq_mul."""
    rng = random.Random(3)
    Q = sim_fq_mul.Q
    failures = 0
    for _ in range(600):
        a, b = rng.randrange(Q, 1 << 384), rng.randrange(Q)
        try:
            ok = sim_fq_mul.mul(sim_fq_mul.words(a), sim_fq_mul.words(b)) == a * b * pow(1 << 384, -1, Q) % Q
        except AssertionError:
            ok = False
        failures += not ok
    assert failures > 0
