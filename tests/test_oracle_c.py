"""Cross-checks of the C oracle tier against the Python tier (itself pinned in test_oracle.py)."""
import random

import numpy as np
import pytest

import workloads as W
from oracle import c_oracle as C
from oracle import tlookup as TL

R = TL.R


def test_field_ops_match_python():
    rng = random.Random(11)
    edge = [0, 1, 2, R - 1, R - 2, (1 << 255) % R, (1 << 254), (1 << 64) - 1, (1 << 128) + 5]
    vals = edge + [rng.randrange(R) for _ in range(300)]
    for i, a in enumerate(vals):
        b = vals[(i * 7 + 3) % len(vals)]
        assert C.fr_binop("mul", a, b) == a * b % R
        assert C.fr_binop("add", a, b) == (a + b) % R
        assert C.fr_binop("sub", a, b) == (a - b) % R
        if a:
            assert C.fr_inv(a) == pow(a, -1, R)


def _chal(ch):
    return C.chal_array(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)


@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
@pytest.mark.parametrize("d,n", [(1, 0), (1, 1), (2, 0), (3, 3), (4, 1), (5, 3), (6, 6), (7, 2), (8, 4), (14, 3),
                                 (15, 9)])
def test_c_equals_python(d, n, variant):
    rng = random.Random(d * 31 + n + variant)
    D, N = 1 << d, 1 << n
    T = [rng.randrange(R) for _ in range(N)]
    S = [rng.choice(T) for _ in range(D)]
    ch = TL.Challenges(rng.randrange(R), rng.randrange(R), 0, [rng.randrange(R) for _ in range(d)],
                       [rng.randrange(R) for _ in range(d)])
    ch.alpha2 = ch.alpha1 ** 2 % R
    py = TL.prove(S, T, ch, variant)
    c = C.prove(C.ints_to_limbs(S), C.ints_to_limbs(T), _chal(ch), variant)
    assert list(c.m) == py.m
    assert C.limbs_to_ints(c.A) == py.A
    assert C.limbs_to_ints(c.B) == py.B
    assert c.evals == py.transcript.evals
    assert c.finals == py.transcript.finals


@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
def test_c_sumcheck_tampered_equals_python(variant):
    rng = random.Random(77)
    d, n = 6, 3
    D, N = 1 << d, 1 << n
    A = [rng.randrange(R) for _ in range(D)]
    S = [rng.randrange(R) for _ in range(D)]
    B = [rng.randrange(R) for _ in range(N)]
    T = [rng.randrange(R) for _ in range(N)]
    m = [rng.randrange(100) for _ in range(N)]
    ch = TL.Challenges(5, 7, 49, [rng.randrange(R) for _ in range(d)], [rng.randrange(R) for _ in range(d)])
    py = TL.sumcheck_prove(A, S, B, T, m, ch, variant)
    c = C.sumcheck(*(C.ints_to_limbs(v) for v in (A, S, B, T)), np.array(m, np.uint32), _chal(ch), variant)
    assert c.evals == py.evals and c.finals == py.finals


def test_c1_workload_c_equals_python():
    wl = W.range_check()
    S, T = C.inputs_from_workload(wl)
    Sp, Tp = TL.field_inputs(wl)
    assert C.limbs_to_ints(S) == Sp and C.limbs_to_ints(T) == Tp
    ch = TL.challenges_from(wl.chal)
    for variant in (0, 1):
        c = C.prove(S, T, _chal(ch), variant)
        py = TL.prove(Sp, Tp, ch, variant)
        assert c.evals == py.transcript.evals and c.finals == py.transcript.finals


def test_pair_inputs_match_python():
    wl = W.activation("2", D=1 << 16)
    S, T = C.inputs_from_workload(wl)
    Sp, Tp = TL.field_inputs(wl)
    assert C.limbs_to_ints(S) == Sp and C.limbs_to_ints(T) == Tp
    ch = TL.challenges_from(wl.chal)
    c = C.prove(S, T, _chal(ch), 0, want_A=False)
    assert sum(c.m) == wl.D


def test_c_errors():
    T = C.ints_to_limbs([1, 2, 3, 4])
    ch = C.chal_array(5, 1, 1, [1, 2, 3], [1, 2, 3])
    with pytest.raises(C.OracleError) as e:
        C.prove(C.ints_to_limbs([1, 2, 9, 3, 8, 1, 1, 1]), T, ch)
    assert e.value.name == "E_NOT_IN_TABLE" and e.value.index == 2
    with pytest.raises(C.OracleError) as e:
        C.prove(C.ints_to_limbs([1] * 8), C.ints_to_limbs([4, 7, 1, 7]), ch)
    assert e.value.name == "E_DUP_TABLE" and e.value.index == 3
    with pytest.raises(C.OracleError) as e:
        C.prove(C.ints_to_limbs([1] * 8), C.ints_to_limbs([1, R - 5, 3, 4]), ch)
    assert e.value.name == "E_DIV_ZERO_T" and e.value.index == 1
    with pytest.raises(C.OracleError) as e:
        C.prove(C.ints_to_limbs([1] * 8), C.ints_to_limbs([1, R, 3, 4]), ch)
    assert e.value.name == "E_NONCANONICAL" and e.value.index == 1


@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
@pytest.mark.parametrize("d,n,s", [(1, 0, 0), (1, 1, 1), (3, 3, 2), (5, 2, 0), (5, 2, 3), (5, 2, 5), (8, 4, 4),
                                   (12, 8, 1), (12, 8, 6), (13, 13, 4)])
def test_stream_tier_equals_c_tier(d, n, s, variant):
    """The bounded-memory streaming tier (pair inputs, first s rounds per block of 2^s) against zko_tlookup."""
    rng = np.random.default_rng(d * 100 + n * 10 + s + variant)
    D, N = 1 << d, 1 << n
    tx = (np.arange(N) - N // 2).astype(np.int32)              # a range X column, as the activation tables
    ty = rng.integers(-2 ** 31, 2 ** 31, N, dtype=np.int64).astype(np.int32)
    pick = rng.integers(0, N, D)
    x, y = tx[pick], ty[pick]
    ch = W.challenges(f"stream{d}.{n}.{s}", d)
    chal = _chal(ch)
    wl = W.Workload("t", D, N, "pair", ch, x=x, y=y, tx=tx, ty=ty)
    S, T = C.inputs_from_workload(wl)
    ref = C.prove(S, T, chal, variant, want_A=False)
    got = C.prove_pair_stream(x, y, tx, ty, ch.alpha_f, chal, variant, s)
    assert np.array_equal(got.m, ref.m)
    assert C.limbs_to_ints(got.B) == C.limbs_to_ints(ref.B)
    assert got.evals == ref.evals
    assert got.finals == ref.finals


def test_stream_tier_errors():
    tx = np.arange(8, dtype=np.int32)
    ty = np.zeros(8, dtype=np.int32)
    ch = W.challenges("stream-err", 4)
    chal = _chal(ch)
    x = np.array([1, 2, 3, 4, 5, 6, 7, 9, 0, 1, 2, 3, 9, 5, 6, 7], dtype=np.int32)   # 9 is not in T (first at 7)
    with pytest.raises(C.OracleError) as e:
        C.prove_pair_stream(x, np.zeros(16, np.int32), tx, ty, ch.alpha_f, chal, 0, 2)
    assert e.value.name == "E_NOT_IN_TABLE" and e.value.index == 7
    txd = tx.copy()
    txd[5] = 2                                                                      # T_5 = T_2: duplicate 5
    with pytest.raises(C.OracleError) as e:
        C.prove_pair_stream(np.zeros(16, np.int32), np.zeros(16, np.int32), txd, ty, ch.alpha_f, chal, 0, 2)
    assert e.value.name == "E_DUP_TABLE" and e.value.index == 5
    # beta = -T_3: DIV_ZERO_T(3) (checked before S)
    bad = C.chal_array((-3) % R, ch.alpha1, ch.alpha2, ch.u, ch.r)
    with pytest.raises(C.OracleError) as e:
        C.prove_pair_stream(np.zeros(16, np.int32), np.zeros(16, np.int32), tx, ty, ch.alpha_f, bad, 0, 2)
    assert e.value.name == "E_DIV_ZERO_T" and e.value.index == 3
