"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, bit-exact.

Every field element, the m vector and every round polynomial must match (BASELINE.json north star).
Small cases use the Python big-integer oracle; larger ones the C tier (itself pinned to the Python tier
in test_oracle_c.py).
"""
import random

import numpy as np
import pytest

import workloads as W
from oracle import c_oracle as C
from oracle import tlookup as TL

pytestmark = pytest.mark.gpu
R = TL.R


@pytest.fixture(scope="module")
def ctx():
    from paper_2404_16109_b200 import zkl
    c = zkl.Context(0)
    c.reserve(1 << 12, 1 << 12)
    yield c
    c.close()


def zkl_mod():
    from paper_2404_16109_b200 import zkl
    return zkl


def _chal_gpu(ch):
    return zkl_mod().Context.challenges(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)


def _canon(xs):
    return zkl_mod().ints_to_canon(xs)


# ------------------------------------------------------------------ a1 boundary encode
def test_import_export_roundtrip(ctx):
    rng = random.Random(1)
    vals = [0, 1, 2, R - 1, R - 2, (1 << 255) % R, (1 << 64) - 1] + [rng.randrange(R) for _ in range(1017)]
    v = ctx.import_canon(_canon(vals))
    assert ctx.export_ints(v) == vals


def test_import_noncanonical(ctx):
    zkl = zkl_mod()
    vals = [5, 7, R, R + 3, 9, 1 << 255, 3, 4]
    with pytest.raises(zkl.ZklError) as e:
        ctx.import_canon(_canon([v % (1 << 256) for v in vals]))
    assert e.value.name == "ZKL_E_NONCANONICAL" and e.value.index == 2


def test_import_pair_and_ints(ctx):
    wl = W.activation("2", D=1 << 16)
    S, T = TL.field_inputs(wl)
    v = ctx.import_pair(wl.x, wl.y, wl.chal.alpha_f)
    assert ctx.export_ints(v) == S
    ints = [0, -1, 5, -32768, 32767, -(1 << 40), (1 << 62), -(1 << 63) + 1]
    v = ctx.import_ints(np.array(ints, dtype=np.int64))
    assert ctx.export_ints(v) == [x % R for x in ints]


def test_fr_mul_via_pair_import(ctx):
    """x + alpha*y exercises the device Montgomery multiplication on random/extreme operands."""
    rng = np.random.default_rng(3)
    n = 1 << 14
    x = rng.integers(-(1 << 31), (1 << 31) - 1, n, dtype=np.int64).astype(np.int32)
    y = rng.integers(-(1 << 31), (1 << 31) - 1, n, dtype=np.int64).astype(np.int32)
    y[:4] = [-1, 0, 1, -(1 << 31)]
    for alpha in [R - 1, 1, (1 << 255) % R, random.Random(4).randrange(R)]:
        v = ctx.import_pair(x, y, alpha)
        got = ctx.export_ints(v)
        want = [(int(a) + alpha * int(b)) % R for a, b in zip(x, y)]
        assert got == want


# ------------------------------------------------------------------ a2/a3 table and m
def _table_from_ints(ctx, t_ints):
    T = ctx.import_canon(_canon([x % R for x in t_ints]))
    return T, ctx.table(T)


@pytest.mark.parametrize("D,N,seed", [(1 << 10, 1 << 8, 1), (1 << 12, 1 << 4, 2), (1 << 13, 1 << 13, 3),
                                      (1 << 14, 1, 4), (1 << 15, 1 << 10, 5), (4, 2, 6), (1, 1, 7)])
def test_multiplicities(ctx, D, N, seed):
    wl = W.random_instance(D, N, seed)
    S, T = TL.field_inputs(wl)
    ctx.reserve(D, N)
    Sv = ctx.import_canon(_canon(S))
    _, tab = _table_from_ints(ctx, T)
    m = ctx.prepare(Sv, D, tab).cpu().numpy().astype(np.uint32)
    assert list(m) == TL.multiplicities(S, T)


def test_multiplicities_skew(ctx):
    """All-equal S (one bin gets everything) and a causal-mask-like spike."""
    D, N = 1 << 16, 1 << 8
    ctx.reserve(D, N)
    T = list(range(N))
    _, tab = _table_from_ints(ctx, T)
    S = [17] * D
    m = ctx.prepare(ctx.import_ints(np.array(S)), D, tab).cpu().numpy()
    assert m[17] == D and m.sum() == D
    rng = np.random.default_rng(5)
    S = np.where(rng.random(D) < 0.5, 255, rng.integers(0, N, D)).astype(np.int64)
    m = ctx.prepare(ctx.import_ints(S), D, tab).cpu().numpy()
    assert list(m) == list(np.bincount(S, minlength=N))


def test_prepare_pair_not_in_table(ctx):
    zkl = zkl_mod()
    D, N = 1 << 14, 1 << 8
    ctx.reserve(D, N)
    tx = np.arange(N, dtype=np.int32) - 128
    ty = tx * 3 + 1
    tab = ctx.table(ctx.import_pair(tx, ty, 12345))
    rng = np.random.default_rng(1)
    x = rng.integers(-128, 128, D).astype(np.int32)
    y = (x * 3 + 1).astype(np.int32)
    S, m = ctx.prepare_pair(x, y, 12345, D, tab)
    assert list(m.cpu().numpy()) == list(np.bincount(x.astype(np.int64) + 128, minlength=N))
    y[9000] += 1             # (x, y) no longer on the function's graph
    y[12000] += 1
    with pytest.raises(zkl.ZklError) as e:
        ctx.prepare_pair(x, y, 12345, D, tab)
    assert e.value.name == "ZKL_E_NOT_IN_TABLE" and e.value.index == 9000


def test_not_in_table_and_dup(ctx):
    zkl = zkl_mod()
    D, N = 1 << 13, 1 << 6
    ctx.reserve(D, N)
    _, tab = _table_from_ints(ctx, list(range(N)))
    S = np.arange(D) % N
    S[5000] = 999
    S[7000] = -3
    with pytest.raises(zkl.ZklError) as e:
        ctx.prepare(ctx.import_ints(S), D, tab)
    assert e.value.name == "ZKL_E_NOT_IN_TABLE" and e.value.index == 5000
    T = list(range(N))
    T[40] = 7
    T[50] = 7
    T[60] = 3
    with pytest.raises(zkl.ZklError) as e:
        _table_from_ints(ctx, T)
    assert e.value.name == "ZKL_E_DUP_TABLE" and e.value.index == 40   # smallest later duplicate


# ------------------------------------------------------------------ a4-a9 full proof
def _gpu_prove(ctx, S, T, ch, variant, D, N):
    ctx.reserve(D, N)
    Sv = ctx.import_canon(_canon(S))
    _, tab = _table_from_ints(ctx, T)
    m = ctx.prepare(Sv, D, tab)
    pf = ctx.prove(Sv, D, tab, m, _chal_gpu(ch), variant, want_A=True, want_B=True)
    return m.cpu().numpy().astype(np.uint32), pf


@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
def test_c1_full_transcript(ctx, variant):
    wl = W.range_check()
    S, T = TL.field_inputs(wl)
    ch = TL.challenges_from(wl.chal)
    ref = TL.prove(S, T, ch, variant)
    m, pf = _gpu_prove(ctx, S, T, ch, variant, wl.D, wl.N)
    assert list(m) == ref.m
    assert ctx.export_ints(pf.A) == ref.A
    assert ctx.export_ints(pf.B) == ref.B
    assert pf.evals == ref.transcript.evals
    assert pf.finals == ref.transcript.finals


CASES = [(1, 0), (1, 1), (2, 1), (3, 3), (5, 2), (11, 4), (12, 4), (12, 12), (13, 5), (14, 8), (15, 0), (16, 16),
         (17, 11)]


@pytest.mark.parametrize("d,n", CASES)
@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
def test_prove_random(ctx, d, n, variant):
    rng = random.Random(1000 * d + n + variant)
    D, N = 1 << d, 1 << n
    T = [rng.randrange(R) for _ in range(N)]
    S = [T[rng.randrange(N)] for _ in range(D)]
    ch = TL.Challenges(rng.randrange(R), rng.randrange(R), 0, [rng.randrange(R) for _ in range(d)],
                       [rng.randrange(R) for _ in range(d)])
    ch.alpha2 = ch.alpha1 ** 2 % R
    m, pf = _gpu_prove(ctx, S, T, ch, variant, D, N)
    ref = C.prove(C.ints_to_limbs(S), C.ints_to_limbs(T),
                  C.chal_array(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r), variant)
    assert list(m) == list(ref.m)
    assert ctx.export_ints(pf.A) == C.limbs_to_ints(ref.A)
    assert ctx.export_ints(pf.B) == C.limbs_to_ints(ref.B)
    assert pf.evals == ref.evals
    assert pf.finals == ref.finals


@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
@pytest.mark.parametrize("d", [5, 13])
def test_prove_degenerate_challenges(ctx, variant, d):
    rng = random.Random(d + variant)
    n = 3
    D, N = 1 << d, 1 << n
    T = [rng.randrange(R) for _ in range(N)]
    S = [T[rng.randrange(N)] for _ in range(D)]
    for u, r, a1 in [([0, 1] * d, [1, 0, 0] * d, 0),
                     ([1] * d, [0] * d, 7),
                     ([rng.randrange(R) if c % 3 else 0 for c in range(d)], [1, 1, 0, 5] * d, 3)]:
        ch = TL.Challenges(rng.randrange(R), a1, a1 * a1 % R, u[:d], r[:d])
        m, pf = _gpu_prove(ctx, S, T, ch, variant, D, N)
        ref = C.prove(C.ints_to_limbs(S), C.ints_to_limbs(T),
                      C.chal_array(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r), variant)
        assert pf.evals == ref.evals and pf.finals == ref.finals


@pytest.mark.parametrize("d,n", [(4, 2), (12, 3), (14, 6)])
@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
def test_sumcheck_prove_tampered(ctx, d, n, variant):
    """zkl_sumcheck_prove on arbitrary vectors: the true round polynomials of the given data."""
    rng = random.Random(7 * d + n + variant)
    D, N = 1 << d, 1 << n
    A = [rng.randrange(R) for _ in range(D)]
    S = [rng.randrange(R) for _ in range(D)]
    B = [rng.randrange(R) for _ in range(N)]
    T = [rng.randrange(R) for _ in range(N)]
    m = [rng.randrange(1000) for _ in range(N)]
    ch = TL.Challenges(rng.randrange(R), rng.randrange(R), rng.randrange(R), [rng.randrange(R) for _ in range(d)],
                       [rng.randrange(R) for _ in range(d)])
    ctx.reserve(D, N)
    vs = [ctx.import_canon(_canon(v)) for v in (A, S, B, T, m)]
    pf = ctx.sumcheck(vs[0], vs[1], D, vs[2], vs[3], vs[4], _chal_gpu(ch), variant)
    ref = C.sumcheck(*(C.ints_to_limbs(v) for v in (A, S, B, T)), np.array(m, np.uint32),
                     C.chal_array(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r), variant)
    assert pf.evals == ref.evals and pf.finals == ref.finals


def test_div_zero(ctx):
    zkl = zkl_mod()
    d, n = 12, 4
    D, N = 1 << d, 1 << n
    rng = random.Random(9)
    T = [rng.randrange(R) for _ in range(N)]
    S = [T[rng.randrange(N)] for _ in range(D)]
    ch = TL.Challenges((R - T[9]) % R, 3, 9, [rng.randrange(R) for _ in range(d)], [rng.randrange(R) for _ in range(d)])
    with pytest.raises(zkl.ZklError) as e:
        _gpu_prove(ctx, S, T, ch, TL.PAPER, D, N)
    assert e.value.name == "ZKL_E_DIV_ZERO_T" and e.value.index == 9
    # S side: prove does not re-check membership; an S value outside T with beta = -S_i
    ctx.reserve(D, N)
    Sv = ctx.import_canon(_canon(S))
    _, tab = _table_from_ints(ctx, T)
    m = ctx.prepare(Sv, D, tab)
    bad = list(S)
    s_star = rng.randrange(R)
    for i in (3000, 1234, 4000):
        bad[i] = s_star
    ch.beta = (R - s_star) % R
    with pytest.raises(zkl.ZklError) as e:
        ctx.prove(ctx.import_canon(_canon(bad)), D, tab, m, _chal_gpu(ch), TL.PAPER)
    assert e.value.name == "ZKL_E_DIV_ZERO_S" and e.value.index == 1234


@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
def test_prove_unprepared_nonmember_falls_back(ctx, variant):
    """prove on an S with an element outside T (a tamper trial): the gather path A_i = B_j(i) cannot apply,
    the library redoes the proof with the batched inversion; the transcript is that of the given data."""
    rng = random.Random(31 + variant)
    d, n = 14, 5
    D, N = 1 << d, 1 << n
    T = [rng.randrange(R) for _ in range(N)]
    S = [T[rng.randrange(N)] for _ in range(D)]
    ch = TL.Challenges(rng.randrange(R), rng.randrange(R), 0, [rng.randrange(R) for _ in range(d)],
                       [rng.randrange(R) for _ in range(d)])
    ch.alpha2 = ch.alpha1 ** 2 % R
    ctx.reserve(D, N)
    _, tab = _table_from_ints(ctx, T)
    m = ctx.prepare(ctx.import_canon(_canon(S)), D, tab)
    bad = list(S)
    bad[777] = rng.randrange(R)
    pf = ctx.prove(ctx.import_canon(_canon(bad)), D, tab, m, _chal_gpu(ch), variant, want_A=True, want_B=True)
    mm = m.cpu().numpy().astype(np.uint32)
    A = [pow((ch.beta + s) % R, -1, R) for s in bad]
    B = [pow((ch.beta + t) % R, -1, R) for t in T]
    if variant == TL.LOGUP:
        B = [b * int(c) % R for b, c in zip(B, mm)]
    ref = C.sumcheck(*(C.ints_to_limbs(v) for v in (A, bad, B, T)), mm,
                     C.chal_array(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r), variant)
    assert ctx.export_ints(pf.A) == A
    assert ctx.export_ints(pf.B) == B
    assert pf.evals == ref.evals and pf.finals == ref.finals


@pytest.mark.parametrize("y", [1, 2, 3, 1 << 31, 1 << 32, (1 << 32) + 1, 1 << 64, 5 << 96, (1 << 200) + 7,
                               (1 << 254) + 1, R - 1, R - 2, (R + 1) // 2, 0xffffffff, (1 << 64) - 1])
def test_inverse_edge_values(ctx, y):
    """The single-thread inversion at the top of every batched inversion (binary extended Euclid on the
    Montgomery integer yR... here chosen directly): N = 1 makes the table side invert beta + T_0 = beta alone, and
    beta = y R^-1 puts the integer y into the routine -- powers of two (whole zero words), 1, r - 1."""
    zkl = zkl_mod()
    Rinv = pow(1 << 256, -1, R)
    beta = y * Rinv % R
    ctx.reserve(2, 1)
    _, tab = _table_from_ints(ctx, [0])
    Sv = ctx.import_canon(_canon([0, 0]))
    m = ctx.prepare(Sv, 2, tab)
    pf = ctx.prove(Sv, 2, tab, m, zkl.Context.challenges(beta, 1, 1, [1], [1]), TL.PAPER, want_A=True, want_B=True)
    inv = pow(beta, -1, R)
    assert ctx.export_ints(pf.B) == [inv]
    assert ctx.export_ints(pf.A) == [inv, inv]


def test_shape_errors(ctx):
    zkl = zkl_mod()
    ctx.reserve(1 << 10, 1 << 4)
    Sv = ctx.import_ints(np.zeros(1 << 10, dtype=np.int64))
    _, tab = _table_from_ints(ctx, list(range(16)))
    with pytest.raises(zkl.ZklError) as e:
        ctx.prepare(Sv, 3 << 8, tab)
    assert e.value.name in ("ZKL_E_SHAPE",)
    _, big = _table_from_ints(ctx, list(range(1 << 11)))
    with pytest.raises(zkl.ZklError) as e:
        ctx.prepare(Sv, 1 << 10, big)
    assert e.value.name == "ZKL_E_SHAPE"


# ------------------------------------------------------------------ config-shaped inputs
@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
def test_c2_activation_full(ctx, variant):
    """C2: GELU activation lookup D = 2^20 into N = 2^16 (full transcript vs the C oracle)."""
    wl = W.activation("2")
    S, T = C.inputs_from_workload(wl)
    ch = TL.challenges_from(wl.chal)
    ref = C.prove(S, T, C.chal_array(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r), variant, want_A=False)
    ctx.reserve(wl.D, wl.N)
    Tv = ctx.import_pair(wl.tx, wl.ty, wl.chal.alpha_f)
    tab = ctx.table(Tv)
    if variant == TL.PAPER:      # the fused a1 + a3 entry point
        Sv, m = ctx.prepare_pair(wl.x, wl.y, wl.chal.alpha_f, wl.D, tab)
    else:
        Sv = ctx.import_pair(wl.x, wl.y, wl.chal.alpha_f)
        m = ctx.prepare(Sv, wl.D, tab)
    assert ctx.export_ints(Sv) == C.limbs_to_ints(S)
    assert np.array_equal(m.cpu().numpy().astype(np.uint32), ref.m)
    pf = ctx.prove(Sv, wl.D, tab, m, _chal_gpu(ch), variant, want_B=True)
    assert ctx.export_ints(pf.B) == C.limbs_to_ints(ref.B)
    assert pf.evals == ref.evals
    assert pf.finals == ref.finals


@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
def test_big_table_rounds(ctx, variant):
    """N = 2^14: the chunked table rounds (k_tab_chunk, 2^14 <= 2^17 entries) + the one-block tail."""
    rng = random.Random(4242 + variant)
    d, n = 15, 14
    D, N = 1 << d, 1 << n
    T = [rng.randrange(R) for _ in range(N)]
    S = [T[rng.randrange(N)] for _ in range(D)]
    ch = TL.Challenges(rng.randrange(R), rng.randrange(R), 0, [rng.randrange(R) for _ in range(d)],
                       [rng.randrange(R) for _ in range(d)])
    ch.alpha2 = ch.alpha1 ** 2 % R
    m, pf = _gpu_prove(ctx, S, T, ch, variant, D, N)
    ref = C.prove(C.ints_to_limbs(S), C.ints_to_limbs(T), C.chal_array(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r),
                  variant)
    assert ctx.export_ints(pf.B) == C.limbs_to_ints(ref.B)
    assert pf.evals == ref.evals and pf.finals == ref.finals


@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
def test_table_rounds_above_2p17(ctx, variant):
    """N = 2^18 > 2^17 entries: the multi-block table round k_tab_round runs (round 1) before the chunked table
    rounds; D = 2^19 function lookups through the virtual-S path, against the streaming C oracle."""
    d, n = 19, 18
    D, N = 1 << d, 1 << n
    rng = np.random.default_rng(1818 + variant)
    tx = (np.arange(N) - N // 2).astype(np.int32)
    ty = rng.integers(-2 ** 31, 2 ** 31, N, dtype=np.int64).astype(np.int32)
    pick = rng.integers(0, N, D)
    x, y = tx[pick], ty[pick]
    ch = W.challenges(f"bigtab{variant}", d)
    chal = C.chal_array(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)
    ref = C.prove_pair_stream(x, y, tx, ty, ch.alpha_f, chal, variant, 2)
    ctx.reserve(D, N)
    tab = ctx.table(ctx.import_pair(tx, ty, ch.alpha_f))
    assert ctx.table_attach_pair(tab, tx, ty, ch.alpha_f)
    ctx.set_profiling(True)
    try:
        _, m = ctx.prepare_pair(x, y, ch.alpha_f, D, tab, virtual_s=True)
        pf = ctx.prove(None, D, tab, m, _chal_gpu(ch), variant, want_B=True)
        names = [rec[0] for rec in ctx.profile_read()]
    finally:
        ctx.set_profiling(False)
    assert "k_tab_round" in names, names
    assert np.array_equal(m.cpu().numpy().astype(np.uint32), ref.m)
    assert ctx.export_ints(pf.B) == C.limbs_to_ints(ref.B)
    assert pf.evals == ref.evals and pf.finals == ref.finals
