"""Hyrax / Pedersen commitments on the GPU against oracle/hyrax.py.

Generators (hash to the curve) point by point; row commitments point by point on small matrices, with and without
blinds, including zero rows (the point at infinity), all-ones-digit scalars (r - 1) and tiny scalars; at a larger
size every row is checked through the homomorphism Com(S1) + Com(S2) = Com(S1 + S2) and two rows
against the definition; ProveEval's w and y against the oracle, and the oracle verifier accepts on the GPU's
commitments."""
import random

import pytest

from oracle import hyrax as HX
from oracle import mle
from oracle.field import R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2404_16109_b200 import zkl
    c = zkl.Context(0)
    yield c
    c.close()


@pytest.fixture(scope="module")
def pp8(ctx):
    return ctx.hyrax_setup(8)


def test_generators_match_oracle(ctx, pp8):
    G, Hb = ctx.hyrax_generators(pp8)
    oG, oH = HX.generators(8)
    assert G == oG and Hb == oH
    assert all(HX.on_curve(P) for P in G + [Hb])


@pytest.mark.parametrize("blind", [False, True])
def test_commit_small_matches_oracle(ctx, pp8, blind):
    from paper_2404_16109_b200 import zkl
    rng = random.Random(3 + blind)
    cols, rows = 8, 4
    S = [rng.randrange(R) for _ in range(rows * cols)]
    S[0:8] = [0] * 8                                # a zero row -> infinity (without blind)
    S[8:16] = [R - 1, 1, 2, 15, 16, 0, R - 1, 255]  # digit extremes
    rho = [rng.randrange(R) for _ in range(rows)] if blind else None
    ctx.reserve(1 << 12, 1 << 4)
    Sv = ctx.import_canon(zkl.ints_to_canon(S))
    C = ctx.hyrax_commit(pp8, Sv, rows * cols, rho)
    G, Hb = HX.generators(cols)
    assert C == HX.commit(S, cols, G, Hb, rho)
    if not blind:
        assert C[0] is None


def test_commit_homomorphism_and_rows(ctx):
    from paper_2404_16109_b200 import zkl
    rng = random.Random(9)
    cols, rows = 64, 64
    D = rows * cols
    pp = ctx.hyrax_setup(cols)
    S1 = [rng.randrange(R) for _ in range(D)]
    S2 = [rng.randrange(R) for _ in range(D)]
    r1 = [rng.randrange(R) for _ in range(rows)]
    r2 = [rng.randrange(R) for _ in range(rows)]
    C1 = ctx.hyrax_commit(pp, ctx.import_canon(zkl.ints_to_canon(S1)), D, r1)
    C2 = ctx.hyrax_commit(pp, ctx.import_canon(zkl.ints_to_canon(S2)), D, r2)
    C12 = ctx.hyrax_commit(pp, ctx.import_canon(zkl.ints_to_canon([(a + b) % R for a, b in zip(S1, S2)])), D,
                           [(a + b) % R for a, b in zip(r1, r2)])
    assert C12 == [HX.add(a, b) for a, b in zip(C1, C2)]
    G, Hb = ctx.hyrax_generators(pp)
    for j in (0, 37):
        assert C1[j] == HX.add(HX.msm(S1[j * cols:(j + 1) * cols], G), HX.mul(r1[j], Hb))


def test_prove_eval(ctx):
    from paper_2404_16109_b200 import zkl
    rng = random.Random(5)
    rows, cols = 16, 16
    D = rows * cols
    pp = ctx.hyrax_setup(cols)
    S = [rng.randrange(R) for _ in range(D)]
    rho = [rng.randrange(R) for _ in range(rows)]
    Sv = ctx.import_canon(zkl.ints_to_canon(S))
    C = ctx.hyrax_commit(pp, Sv, D, rho)
    v = [rng.randrange(R) for _ in range(8)]
    w, y = ctx.hyrax_prove_eval(Sv, D, cols, v)
    ow, oy = HX.prove_eval(S, cols, v[:4], v[4:])
    assert ctx.export_ints(w) == ow and y == oy == mle.mle_eval(S, v)
    G, Hb = ctx.hyrax_generators(pp)
    assert HX.verify_eval(C, cols, G, Hb, v[:4], v[4:], ow, oy, rho)


def test_commit_signed_magnitude_boundaries(ctx, pp8):
    """k_hx_canon commits s > (r-1)/2 as -(r - s) (the table point negated): scalars on both sides of the split,
    small negatives (one 32-bit chunk), and rows that are all small (no Horner doublings) equal the oracle's."""
    from paper_2404_16109_b200 import zkl
    h = (R - 1) // 2
    cols, rows = 8, 4
    S = [h, h + 1, h - 1, h + 2, R - 1, R - 2, 1, 0,                          # around the split
         R - 5, 7, R - (1 << 31), (1 << 31) - 1, R - (1 << 32) + 1, (1 << 32) - 1, R - 255, 3,   # small signed
         R - 1, R - 1, R - 1, R - 1, R - 1, R - 1, R - 1, R - 1,             # all -1: one negated chunk each
         (1 << 254), R - (1 << 254), h + (1 << 200), h - (1 << 200), 2, R - 2, 1 << 40, R - (1 << 40)]
    ctx.reserve(1 << 12, 1 << 4)
    Sv = ctx.import_canon(zkl.ints_to_canon(S))
    C = ctx.hyrax_commit(pp8, Sv, rows * cols, None)
    G, H = HX.generators(cols)
    assert C == HX.commit(S, cols, G, H)
