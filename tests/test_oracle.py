"""Pins for the Python oracle (CPU only): each test checks the oracle against something
other than itself — closed forms, the paper's identities, worked examples, brute force
through the MLE definition, and the survey's independently computed known answers."""
import hashlib
import json
import os
import random
import struct

import pytest

import workloads as W
from oracle import field as F
from oracle import mle
from oracle import tlookup as TL

R = F.R
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- Fr

def test_modulus_is_prime_with_2adicity_32():
    # Miller-Rabin with fixed bases: r prime (BLS12-381 scalar field)
    n, d, s = R, R - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    assert s == 32
    for a in [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41]:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            pytest.fail(f"witness {a}")
    assert R.bit_length() == 255
    limbs = [(R >> (32 * i)) & 0xFFFFFFFF for i in range(8)]
    assert limbs == [0x00000001, 0xFFFFFFFF, 0xFFFE5BFE, 0x53BDA402, 0x09A1D805, 0x3339D808, 0x299D7D48, 0x73EDA753]


def test_field_closed_forms():
    assert F.inv(2) == (R + 1) // 2
    assert F.mul(R - 1, R - 1) == 1
    assert F.fr(-1) == R - 1 and F.fr(-32768) == R - 32768
    rng = random.Random(1)
    for _ in range(200):
        a = rng.randrange(1, R)
        assert F.mul(a, F.inv(a)) == 1
        b = rng.randrange(R)
        assert F.sub(F.add(a, b), b) == a
    with pytest.raises(F.NotInvertible):
        F.inv(0)


# ---------------------------------------------------------------- MLE / eq

def test_spec_examples_mle_eq():
    g = _load("spec_examples.json")
    for ex in g["mle"]:
        assert mle.mle_eval(ex["vals"], ex["point"]) == ex["value"] % R
    for ex in g["eq"]:
        assert mle.eq(ex["u"], ex["v"]) == ex["value"]
    for ex in g["eq_table"]:
        assert mle.eq_table(ex["u"]) == ex["table"]


def test_eq_is_indicator_on_cube_and_sums_to_one():
    d = 4
    for a in range(1 << d):
        for b in range(1 << d):
            assert mle.eq(mle.bits_msb_first(a, d), mle.bits_msb_first(b, d)) == (1 if a == b else 0)
    rng = random.Random(2)
    u = [rng.randrange(R) for _ in range(6)]
    assert sum(mle.eq_table(u)) % R == 1


def test_mle_msb_first_convention():
    # coordinate 0 is the MSB of the row-major flat index (reading 3)
    vals = [10, 20, 30, 40]          # S[i0, i1] row-major
    assert mle.mle_eval(vals, [0, 1]) == 20
    assert mle.mle_eval(vals, [1, 0]) == 30


# ---------------------------------------------------------------- m, A, B

def test_multiplicity_examples_and_invariants():
    g = _load("spec_examples.json")
    for ex in g["multiplicities"]:
        assert TL.multiplicities(ex["S"], ex["T"]) == ex["m"]
    T = list(range(16))
    assert TL.multiplicities(T, T) == [1] * 16
    assert TL.multiplicities([5] * 32, list(range(5, 21))) == [32] + [0] * 15
    rng = random.Random(3)
    S = [rng.choice(T) for _ in range(64)]
    m = TL.multiplicities(S, T)
    assert sum(m) == 64
    assert m == [S.count(t) for t in T]


def test_identity_worked_example():
    g = _load("spec_examples.json")["identity"]
    m = TL.multiplicities(g["S"], g["T"])
    A, B = TL.inverses(g["S"], g["T"], g["beta"], m)
    lhs = sum(A) % R
    rhs = sum(mi * b for mi, b in zip(m, B)) % R
    assert lhs == rhs == int(g["hex"], 16) == 9 * F.inv(10) % R


@pytest.mark.parametrize("seed", range(5))
def test_identity_random(seed):
    wl = W.random_instance(64, 16, seed)
    S, T = TL.field_inputs(wl)
    ch = TL.challenges_from(wl.chal)
    m = TL.multiplicities(S, T)
    A, B = TL.inverses(S, T, ch.beta, m)
    for a, s in zip(A, S):
        assert a * (s + ch.beta) % R == 1
    assert sum(A) % R == sum(mi * b for mi, b in zip(m, B)) % R      # Eq. hab22-check
    A2, B2 = TL.inverses(S, T, ch.beta, m, TL.LOGUP)
    assert A2 == A and sum(A) % R == sum(B2) % R                       # north-star form
    for b, t, mi in zip(B2, T, m):
        assert b * (t + ch.beta) % R == mi


def test_errors_smallest_index():
    with pytest.raises(TL.NotInTable) as e:
        TL.multiplicities([1, 2, 9, 3, 8], [1, 2, 3, 4])
    assert e.value.index == 2
    with pytest.raises(TL.DupTable) as e:
        TL.check_table([4, 7, 1, 7, 4, 4])
    assert e.value.index == 3
    with pytest.raises(TL.DivZero) as e:                 # T is checked first
        TL.inverses([R - 5, 1], [1, R - 5, R - 1], 5, [1, 1, 0])
    assert e.value.index == 1 and e.value.side == "T"
    with pytest.raises(TL.DivZero) as e:
        TL.inverses([1, 2, R - 5, R - 5], [1, 2], 5, [1, 1])
    assert e.value.index == 2 and e.value.side == "S"
    for D, N in [(3, 1), (4, 8), (0, 1), (8, 3)]:
        with pytest.raises(TL.ShapeError):
            TL.check_shapes(D, N)
    with pytest.raises(TL.NonCanonical) as e:
        TL.check_canonical([0, R - 1, R, 5])
    assert e.value.index == 2


# ---------------------------------------------------------------- sumcheck

@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
def test_known_answer_transcript(variant):
    g = _load("kat_d2.json")
    inp = g["inputs"]
    ch = TL.Challenges(inp["beta"], inp["alpha1"], inp["alpha2"], inp["u"], inp["r"])
    p = TL.prove(inp["S"], inp["T"], ch, variant)
    key = "PAPER" if variant == TL.PAPER else "LOGUP"
    assert p.m == g["m"]
    h = lambda xs: [int(x, 16) for x in xs]
    if variant == TL.PAPER:
        assert p.A == h(g["PAPER"]["A"])
    else:
        assert p.B == h(g["LOGUP"]["B"])
    assert p.transcript.evals[0] == h(g[key]["g1"])
    assert p.transcript.evals[1] == h(g[key]["g2"])
    assert p.transcript.finals == {k: int(v, 16) for k, v in g[key]["finals"].items()}


def _digest_fr(xs):
    return hashlib.sha256(b"".join(x.to_bytes(32, "little") for x in xs)).hexdigest()


@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
def test_c1_golden_digests(variant):
    g = _load("c1_digests.json")
    key = "PAPER" if variant == TL.PAPER else "LOGUP"
    wl = W.range_check()
    assert [int(v) for v in wl.s[:8]] == g["S_head"]
    S, T = TL.field_inputs(wl)
    ch = TL.challenges_from(wl.chal)
    assert ch.beta == int(g["challenges"]["beta"], 16) and ch.r[0] == int(g["challenges"]["r1"], 16)
    p = TL.prove(S, T, ch, variant)
    assert p.m[:8] == g["m_head"]
    assert hashlib.sha256(b"".join(struct.pack("<I", x) for x in p.m)).hexdigest() == g[key]["m"]
    assert _digest_fr(p.A) == g[key]["A"]
    assert _digest_fr(p.B) == g[key]["B"]
    assert _digest_fr([x for e in p.transcript.evals for x in e]) == g[key]["evals"]
    assert p.transcript.evals[0][0] == int(g[key]["g1_0"], 16)
    assert p.transcript.finals == {k: int(v, 16) for k, v in g[key]["finals"].items()}


def _rand_case(d, n, seed, tamper=False):
    rng = random.Random(seed)
    D, N = 1 << d, 1 << n
    T = [rng.randrange(R) for _ in range(N)]
    S = [rng.choice(T) for _ in range(D)]
    ch = TL.Challenges(rng.randrange(R), rng.randrange(R), 0, [rng.randrange(R) for _ in range(d)],
                       [rng.randrange(R) for _ in range(d)])
    ch.alpha2 = ch.alpha1 * ch.alpha1 % R
    m = TL.multiplicities(S, T)
    A, B = TL.inverses(S, T, ch.beta, m)
    if tamper:               # arbitrary vectors: the transcript must still be the true round polys
        A = [rng.randrange(R) for _ in range(D)]
        m = [rng.randrange(5) for _ in range(N)]
    return S, T, m, A, B, ch


CASES = [(1, 0), (1, 1), (2, 0), (3, 1), (3, 3), (4, 4), (5, 3), (5, 2), (3, 0)]


@pytest.mark.parametrize("d,n", CASES)
@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
@pytest.mark.parametrize("tamper", [False, True])
def test_linear_prover_equals_brute_force(d, n, variant, tamper):
    S, T, m, A, B, ch = _rand_case(d, n, 100 * d + 10 * n + variant + 7 * tamper, tamper)
    if variant == TL.LOGUP and not tamper:
        _, B = TL.inverses(S, T, ch.beta, m, TL.LOGUP)
    lin = TL.sumcheck_prove(A, S, B, T, m, ch, variant)
    bf = TL.brute_force_round_polys(A, S, B, T, m, ch, variant)
    assert lin.evals == bf.evals
    assert lin.finals == bf.finals


@pytest.mark.parametrize("d,n", [(1, 0), (4, 2), (5, 5), (6, 3)])
@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
def test_claim_and_verifier_accept(d, n, variant):
    rng = random.Random(d * 7 + n)
    D, N = 1 << d, 1 << n
    T = [rng.randrange(R) for _ in range(N)]
    S = [rng.choice(T) for _ in range(D)]
    ch = TL.Challenges(rng.randrange(R), rng.randrange(R), 0, [rng.randrange(R) for _ in range(d)],
                       [rng.randrange(R) for _ in range(d)])
    ch.alpha2 = ch.alpha1 * ch.alpha1 % R
    p = TL.prove(S, T, ch, variant)
    g1 = p.transcript.evals[0]
    assert (g1[0] + g1[1]) % R == TL.claimed_sum(ch.alpha1, ch.alpha2, variant)
    assert TL.verify(p.transcript, D, N, ch, variant)


@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
def test_soundness_tamper_rejected(variant):
    """Thm 3 as a test: a prover that deviates is rejected."""
    rng = random.Random(99 + variant)
    d, n = 6, 3
    D, N = 1 << d, 1 << n
    for trial in range(20):
        T = [rng.randrange(R) for _ in range(N)]
        S = [rng.choice(T) for _ in range(D)]
        ch = TL.Challenges(rng.randrange(R), rng.randrange(R), 0, [rng.randrange(R) for _ in range(d)],
                           [rng.randrange(R) for _ in range(d)])
        ch.alpha2 = ch.alpha1 * ch.alpha1 % R
        m = TL.multiplicities(S, T)
        kind = trial % 3
        if kind == 0:                                  # m[0] + 1
            m_bad = list(m)
            m_bad[0] += 1
            A, B = TL.inverses(S, T, ch.beta, m_bad, variant)
            tr = TL.sumcheck_prove(A, S, B, T, m_bad, ch, variant)
        elif kind == 1:                                # S_i replaced by a non-member, stale m
            S_bad = list(S)
            S_bad[rng.randrange(D)] = rng.randrange(R)
            A, B = TL.inverses(S_bad, T, ch.beta, m, variant)
            tr = TL.sumcheck_prove(A, S_bad, B, T, m, ch, variant)
        else:                                          # honest proof, one evaluation perturbed
            p = TL.prove(S, T, ch, variant)
            tr = p.transcript
            k = rng.randrange(d)
            tr.evals[k][rng.randrange(4)] += 1
        assert not TL.verify(tr, D, N, ch, variant)
    p = TL.prove(S, T, ch, variant)
    p.transcript.finals["A"] = (p.transcript.finals["A"] + 1) % R
    assert not TL.verify(p.transcript, D, N, ch, variant)


@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
def test_degenerate_challenges(variant):
    """alpha1 = 0, u_c in {0, 1}, r_k in {0, 1} are legal inputs (reading 19)."""
    rng = random.Random(5)
    d, n = 5, 2
    T = [rng.randrange(R) for _ in range(1 << n)]
    S = [rng.choice(T) for _ in range(1 << d)]
    for u, r, a1 in [([0, 1, 0, 1, 1], [1, 0, 0, 1, 1], 0),
                     ([1] * 5, [0] * 5, 7),
                     ([rng.randrange(R) for _ in range(5)], [1, 1, 0, 0, 1], 3)]:
        ch = TL.Challenges(rng.randrange(R), a1, a1 * a1 % R, u, r)
        p = TL.prove(S, T, ch, variant)
        bf = TL.brute_force_round_polys(p.A, S, p.B, T, p.m, ch, variant)
        assert p.transcript.evals == bf.evals and p.transcript.finals == bf.finals
        assert TL.verify(p.transcript, 1 << d, 1 << n, ch, variant)


def test_function_lookup_inputs():
    """Y = f(X) becomes X + alpha_f Y in T_X + alpha_f T_Y."""
    wl = W.activation("2", D=1 << 8)
    S, T = TL.field_inputs(wl)
    m = TL.multiplicities(S, T)
    assert sum(m) == 256
    xs = [int(x) for x in wl.x]
    for j, c in enumerate(m):
        assert c == xs.count(j - 32768)
