"""Pins for the Hyrax/Pedersen oracle, CPU only.

The curve constants are pinned to the BLS12-381 family formulas (z, r = z^4 - z^2 + 1, q = (z-1)^2 r/3 + z,
#E = q + 1 - (z + 1) = h r); the group law to the group axioms and to the generator's order; the commitment to
its definition (a sum of scalar multiples), to Com(e_i) = G_i, and to the homomorphism PAPER.md:203 states;
ProveEval to the MLE definition and to the verifier's check."""
import random

import pytest

from oracle import hyrax as HX
from oracle import mle
from oracle.field import R

Z = -0xD201000000010000


def test_curve_constants_from_the_family_formulas():
    assert Z ** 4 - Z ** 2 + 1 == R
    assert (Z - 1) ** 2 * R % 3 == 0 and (Z - 1) ** 2 * R // 3 + Z == HX.Q
    n = HX.Q + 1 - (Z + 1)
    assert n == HX.H_COFACTOR * R
    assert HX.Q % 4 == 3                      # the sqrt exponent (q+1)/4 of the hash to the curve


def test_generator_on_curve_and_of_order_r():
    G = HX.G1_GEN
    assert HX.on_curve(G)
    assert HX.mul(R, G) is None
    assert HX.mul(R - 1, G) == HX.neg(G)


def test_group_law_axioms():
    rng = random.Random(1)
    G = HX.G1_GEN
    P, Qp, S = (HX.mul(rng.randrange(1, R), G) for _ in range(3))
    assert HX.add(P, Qp) == HX.add(Qp, P)
    assert HX.add(HX.add(P, Qp), S) == HX.add(P, HX.add(Qp, S))
    assert HX.add(P, None) == P and HX.add(P, HX.neg(P)) is None
    assert HX.add(P, P) == HX.mul(2, P)
    a, b = rng.randrange(R), rng.randrange(R)
    assert HX.mul((a + b) % R, G) == HX.add(HX.mul(a, G), HX.mul(b, G))
    assert all(HX.on_curve(X) for X in (P, Qp, S))


def test_hash_to_curve_lands_in_the_subgroup():
    G, Hb = HX.generators(4)
    for X in G + [Hb]:
        assert X is not None and HX.on_curve(X)
        assert HX.mul(R, X) is None
    assert len({X for X in G + [Hb]}) == 5
    assert HX.hash_to_curve(b"zkl-hyrax-G", 2) == G[2]


def test_commit_definition_unit_vectors_and_homomorphism():
    rng = random.Random(2)
    cols, rows = 4, 2
    G, Hb = HX.generators(cols)
    e = [0] * (rows * cols)
    e[1 * cols + 2] = 1
    C = HX.commit(e, cols, G, Hb)
    assert C[0] is None and C[1] == G[2]
    S1 = [rng.randrange(R) for _ in range(rows * cols)]
    S2 = [rng.randrange(R) for _ in range(rows * cols)]
    r1 = [rng.randrange(R) for _ in range(rows)]
    r2 = [rng.randrange(R) for _ in range(rows)]
    C1, C2 = HX.commit(S1, cols, G, Hb, r1), HX.commit(S2, cols, G, Hb, r2)
    C12 = HX.commit([(a + b) % R for a, b in zip(S1, S2)], cols, G, Hb, [(a + b) % R for a, b in zip(r1, r2)])
    assert C12 == [HX.add(a, b) for a, b in zip(C1, C2)]
    # the definition, term by term
    assert C1[0] == HX.add(HX.add(HX.add(HX.add(HX.mul(S1[0], G[0]), HX.mul(S1[1], G[1])), HX.mul(S1[2], G[2])),
                                  HX.mul(S1[3], G[3])), HX.mul(r1[0], Hb))


def test_prove_eval_matches_mle_and_verifies():
    rng = random.Random(3)
    rows, cols = 4, 4
    G, Hb = HX.generators(cols)
    S = [rng.randrange(R) for _ in range(rows * cols)]
    rho = [rng.randrange(R) for _ in range(rows)]
    C = HX.commit(S, cols, G, Hb, rho)
    vr = [rng.randrange(R) for _ in range(2)]
    vc = [rng.randrange(R) for _ in range(2)]
    w, y = HX.prove_eval(S, cols, vr, vc)
    assert y == mle.mle_eval(S, vr + vc)
    assert HX.verify_eval(C, cols, G, Hb, vr, vc, w, y, rho)
    bad = list(w)
    bad[1] = (bad[1] + 1) % R
    assert not HX.verify_eval(C, cols, G, Hb, vr, vc, bad, y, rho)
    assert not HX.verify_eval(C, cols, G, Hb, vr, vc, w, (y + 1) % R, rho)
