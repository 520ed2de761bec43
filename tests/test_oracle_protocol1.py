"""Pins of the Protocol-1 oracle (oracle/protocol1.py): an honest proof verifies; every message is
bound into the transcript before the challenge after it (one changed lookup changes alpha_f and beta); tampered
finals, evaluation proofs or commitments are rejected; both variants."""
import random

import pytest

from oracle import hyrax as HX
from oracle import protocol1 as P1
from oracle import tlookup as TL

R = TL.R


def _instance(D, N, seed):
    rng = random.Random(seed)
    tx = list(range(-N // 2, N // 2))
    ty = [rng.randrange(-2 ** 20, 2 ** 20) for _ in range(N)]
    pick = [rng.randrange(N) for _ in range(D)]
    return [tx[i] for i in pick], [ty[i] for i in pick], tx, ty


@pytest.fixture(scope="module")
def gens():
    return HX.generators(4)


@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
def test_honest_proof_verifies(gens, variant):
    G, H = gens
    x, y, tx, ty = _instance(64, 8, 1 + variant)
    pf = P1.prove(x, y, tx, ty, b"\x07" * 32, 4, variant, G, H)
    assert P1.verify(pf, G, H)
    # the sumcheck claim is the paper's (alpha1 + alpha2, or alpha1 for LOGUP) and S = X + alpha_f Y
    ch = pf["challenges"]
    g1 = pf["evals"][0]
    assert (g1[0] + g1[1]) % R == TL.claimed_sum(ch.alpha1, ch.alpha2, variant)


def test_transcript_binds_the_lookups(gens):
    G, H = gens
    x, y, tx, ty = _instance(64, 8, 5)
    a = P1.prove(x, y, tx, ty, bytes(32), 4, TL.PAPER, G, H)
    x2, y2 = list(x), list(y)
    j = next(i for i in range(8) if tx[i] != x[10])
    x2[10], y2[10] = tx[j], ty[j]                  # one lookup moved to another table entry
    b = P1.prove(x2, y2, tx, ty, bytes(32), 4, TL.PAPER, G, H)
    assert a["C"]["X"] != b["C"]["X"]
    assert a["alpha_f"] != b["alpha_f"] and a["challenges"].beta != b["challenges"].beta
    assert P1.verify(b, G, H)


def test_tampering_is_rejected(gens):
    G, H = gens
    x, y, tx, ty = _instance(64, 8, 9)
    pf = P1.prove(x, y, tx, ty, bytes(32), 4, TL.PAPER, G, H)
    bad = dict(pf, finals=dict(pf["finals"], A=(pf["finals"]["A"] + 1) % R))
    assert not P1.verify(bad, G, H)
    w, yv = pf["eval_proofs"]["m"]
    bad = dict(pf, eval_proofs=dict(pf["eval_proofs"], m=([(w[0] + 1) % R] + w[1:], yv)))
    assert not P1.verify(bad, G, H)
    C = dict(pf["C"])
    C["B"] = [HX.add(C["B"][0], G[0])] + C["B"][1:]
    assert not P1.verify(dict(pf, C=C), G, H)
    ev = [list(e) for e in pf["evals"]]
    ev[2][3] = (ev[2][3] + 1) % R
    assert not P1.verify(dict(pf, evals=ev), G, H)
