"""Protocol 1 with its commitments on the GPU (zkl_tlookup_prove_p1) against the oracle
(oracle/protocol1.py): the commitments, the transcript's challenges, every round polynomial, the finals and the
proofs of evaluation are equal to the oracle's, the oracle's verifier accepts the GPU's proof, and the transcript
binds the lookups (one changed lookup changes alpha_f and beta)."""
import random

import pytest

from oracle import hyrax as HX
from oracle import protocol1 as P1
from oracle import tlookup as TL

pytestmark = pytest.mark.gpu
R = TL.R


@pytest.fixture(scope="module")
def ctx():
    from paper_2404_16109_b200 import zkl
    c = zkl.Context(0)
    yield c
    c.close()


def _instance(D, N, seed):
    rng = random.Random(seed)
    tx = list(range(-N // 2, N // 2))
    ty = [rng.randrange(-2 ** 20, 2 ** 20) for _ in range(N)]
    pick = [rng.randrange(N) for _ in range(D)]
    return [tx[i] for i in pick], [ty[i] for i in pick], tx, ty


@pytest.mark.parametrize("D,N,cols,variant", [(1 << 8, 1 << 4, 4, TL.PAPER), (1 << 10, 1 << 6, 16, TL.LOGUP)])
def test_p1_equals_oracle(ctx, D, N, cols, variant):
    x, y, tx, ty = _instance(D, N, D + variant)
    seed = bytes(range(32))
    G, H = HX.generators(cols)
    ref = P1.prove(x, y, tx, ty, seed, cols, variant, G, H)
    ctx.reserve(D, N)
    pp = ctx.hyrax_setup(cols)
    got = ctx.prove_p1(pp, x, y, tx, ty, seed, variant)
    assert got["C"] == ref["C"]
    assert got["alpha_f"] == ref["alpha_f"]
    ch = ref["challenges"]
    assert got["derived"] == {"beta": ch.beta, "alpha1": ch.alpha1, "alpha2": ch.alpha2, "u": ch.u, "r": ch.r}
    assert got["evals"] == ref["evals"] and got["finals"] == ref["finals"]
    assert got["eval_proofs"] == {k: (list(w), yv) for k, (w, yv) in ref["eval_proofs"].items()}
    assert P1.verify(got, G, H)


def test_p1_binds_the_statement(ctx):
    D, N, cols = 1 << 8, 1 << 4, 4
    x, y, tx, ty = _instance(D, N, 3)
    ctx.reserve(D, N)
    pp = ctx.hyrax_setup(cols)
    a = ctx.prove_p1(pp, x, y, tx, ty, bytes(32), TL.PAPER)
    j = next(i for i in range(N) if tx[i] != x[77])
    x2, y2 = list(x), list(y)
    x2[77], y2[77] = tx[j], ty[j]
    b = ctx.prove_p1(pp, x2, y2, tx, ty, bytes(32), TL.PAPER)
    assert a["alpha_f"] != b["alpha_f"] and a["derived"]["beta"] != b["derived"]["beta"]
    G, H = HX.generators(cols)
    assert P1.verify(b, G, H)
    bad = dict(b, finals=dict(b["finals"], m=(b["finals"]["m"] + 1) % R))
    assert not P1.verify(bad, G, H)


def test_p1_larger_instance_verifies(ctx):
    """D = 2^16 lookups into N = 2^8 with rows of 2^8: the GPU proof passes the oracle's verifier."""
    D, N, cols = 1 << 16, 1 << 8, 1 << 8
    x, y, tx, ty = _instance(D, N, 16)
    ctx.reserve(D, N)
    pp = ctx.hyrax_setup(cols)
    pf = ctx.prove_p1(pp, x, y, tx, ty, b"\x11" * 32, TL.PAPER)
    G, H = HX.generators(cols)
    assert P1.verify(pf, G, H)
