"""tlookup (Protocol 1 of PAPER.md §4) as a plain CPU computation (TEST INFRASTRUCTURE ONLY).

Each function follows one passage of PAPER.md, in the paper's order and notation:

  multiplicities   PAPER.md:238-239  Eq. hab22-coefs   m_i = |{j : S_j = T_i}|
  inverses         PAPER.md:240-241  Eq. hab22-invs    A = 1/(beta+S), B = 1/(beta+T)
  tlookup_poly     PAPER.md:244-250  Eq. tlookup-sumcheck (the summand f)
  sumcheck_prove   PAPER.md:181-183  Eq. sumcheck, round by round, LSB first
  verify           PAPER.md:181-183, 547-557 (round consistency; final claim f(v))

Readings of silent / garbled points used here:
  * coordinate 0 = MSB of the row-major index; table index j = x mod N, the
    table slice of u is u[log2(D/N):] (the LAST n coordinates) (readings 3-5);
  * round k binds coordinate d-k (LSB first), pairs (2y, 2y+1) (reading 6);
  * round polynomial g_k given by its values at t = 0, 1, 2, 3 (reading 7);
  * weights (1, alpha1, alpha2), alpha2 = alpha^2 for the paper (reading 8);
  * claim alpha1 + alpha2 (PAPER) / alpha1 (LOGUP) (reading 9);
  * variant LOGUP: B = m/(beta+T), the north-star wording (reading 10);
  * duplicate table entries, S not in T, beta in -S u -T, shapes: errors with
    the smallest offending index (readings 11-14, 16).

No blocking, fusion, eq factoring or derived evaluations: every vector lives on
the D-sized hypercube and every g_k(t) is summed directly.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Sequence

from . import field as F
from .mle import bits_msb_first, eq, eq_table, mle_eval

R = F.R
PAPER = 0
LOGUP = 1


class TlookupError(Exception):
    code = "ERR"

    def __init__(self, index: int = -1, msg: str = ""):
        super().__init__(f"{self.code}({index}) {msg}")
        self.index = index


class ShapeError(TlookupError):
    code = "E_SHAPE"


class NonCanonical(TlookupError):
    code = "E_NONCANONICAL"


class DupTable(TlookupError):
    code = "E_DUP_TABLE"


class NotInTable(TlookupError):
    code = "E_NOT_IN_TABLE"


class DivZero(TlookupError):
    code = "E_DIV_ZERO"

    def __init__(self, index: int = -1, msg: str = "", side: str = "S"):
        super().__init__(index, msg)
        self.side = side            # "T": beta + T_j = 0 (checked first), "S": beta + S_i = 0


def log2_exact(x: int) -> int:
    if x < 1 or x & (x - 1):
        raise ShapeError(-1, f"{x} is not a power of two")
    return x.bit_length() - 1


def check_shapes(D: int, N: int) -> None:
    """PAPER.md:258 (Protocol 1 Require): N, D powers of 2 and N | D."""
    log2_exact(D)
    log2_exact(N)
    if N > D:
        raise ShapeError(-1, "N must divide D")


def check_canonical(v: Sequence[int]) -> None:
    for i, x in enumerate(v):
        if not 0 <= x < R:
            raise NonCanonical(i)


def check_table(T: Sequence[int]) -> None:
    """Reading 11: a table with repeated entries is rejected; index = smallest later duplicate j'."""
    seen = set()
    for j, t in enumerate(T):
        if t in seen:
            raise DupTable(j)
        seen.add(t)


def multiplicities(S: Sequence[int], T: Sequence[int]) -> List[int]:
    """Eq. hab22-coefs: m_i <- |{j : S_j = T_i}| by straightforward counting
    (PAPER.md:83).  S_j not in T: NotInTable(smallest j) (reading 12)."""
    where = {t: i for i, t in enumerate(T)}
    m = [0] * len(T)
    for j, s in enumerate(S):
        i = where.get(s)
        if i is None:
            raise NotInTable(j)
        m[i] += 1
    return m


def inverses(S: Sequence[int], T: Sequence[int], beta: int, m: Sequence[int], variant: int = PAPER):
    """Eq. hab22-invs: A = (1/(beta+S_i))_i, B = (1/(beta+T_i))_i.

    LOGUP variant (north star): B_i = m_i / (beta+T_i).  beta in -T (checked first) or
    -S: DivZero(smallest index) — the completeness error of Thm 2.
    """
    for j, t in enumerate(T):
        if (beta + t) % R == 0:
            raise DivZero(j, "beta + T_j = 0", side="T")
    for i, s in enumerate(S):
        if (beta + s) % R == 0:
            raise DivZero(i, "beta + S_i = 0", side="S")
    A = [F.inv(F.add(beta, s)) for s in S]
    B = [F.inv(F.add(beta, t)) for t in T]
    if variant == LOGUP:
        B = [F.mul(mi % R, b) for mi, b in zip(m, B)]
    return A, B


def claimed_sum(alpha1: int, alpha2: int, variant: int = PAPER) -> int:
    """Left side of Eq. tlookup-sumcheck: alpha + alpha^2 (reading 9)."""
    return F.add(alpha1, alpha2) if variant == PAPER else alpha1 % R


def tlookup_poly(a, s, e, b, t, mm, e2, beta, alpha1, alpha2, w, variant=PAPER):
    """The summand of Eq. tlookup-sumcheck at one point, from the values there
    of A~, S~, e~(u,.), B~, T~, m~, e~(u[log2(D/N):], .) and w = N D^{-1}:

        PAPER: A (alpha1 e (S + beta) + 1) + w B (alpha2 e2 (T + beta) - m)
        LOGUP: A (alpha1 e (S + beta) + 1) + w (-B + alpha2 e2 (B (T + beta) - m))
    """
    d_side = a * ((alpha1 * e % R) * ((s + beta) % R) % R + 1) % R
    if variant == PAPER:
        t_side = b * ((alpha2 * e2 % R) * ((t + beta) % R) % R - mm) % R
    else:
        t_side = (-b + (alpha2 * e2 % R) * ((b * ((t + beta) % R) - mm) % R)) % R
    return (d_side + w * t_side) % R


@dataclass
class Challenges:
    beta: int
    alpha1: int
    alpha2: int
    u: List[int]
    r: List[int]


@dataclass
class Transcript:
    evals: List[List[int]]          # evals[k-1][t] = g_k(t), t = 0..3
    finals: Dict[str, int]          # A(v), S(v), B(v'), T(v'), m(v')


def lagrange_0123(g: Sequence[int], x: int) -> int:
    """Value at x of the degree-3 polynomial with values g[0..3] at 0, 1, 2, 3."""
    nodes = [0, 1, 2, 3]
    acc = 0
    for i, xi in enumerate(nodes):
        num, den = 1, 1
        for j, xj in enumerate(nodes):
            if j != i:
                num = num * (x - xj) % R
                den = den * (xi - xj) % R
        acc = (acc + g[i] * num % R * F.inv(den)) % R
    return acc


def sumcheck_prove(A, S, B, T, m, ch: Challenges, variant: int = PAPER, next_r=None) -> Transcript:
    """Sumcheck on Eq. tlookup-sumcheck, linear time.

    All seven multilinear vectors are laid out on the D-point hypercube (the table
    terms repeat with period N: j = x mod N, reading 5).  Round k (1-based) binds
    coordinate d-k: for each pair (2y, 2y+1) every vector V is evaluated at
    t in {0,1,2,3} as V_t = V_0 + t (V_1 - V_0) (multilinearity), the summand is
    evaluated there and summed over y; then every vector is folded with r_k as
    V' = V_0 + r_k (V_1 - V_0).

    next_r(k, g_k) -> r_k (optional): a Fiat-Shamir transcript supplies r_k once g_k is known (it is appended to
    ch.r); by default r_k = ch.r[k-1].
    """
    D, N = len(A), len(B)
    check_shapes(D, N)
    d, n = log2_exact(D), log2_exact(N)
    assert len(S) == D and len(T) == N and len(m) == N
    assert len(ch.u) == d and (len(ch.r) == d or next_r is not None)
    w = N * F.inv(D) % R
    E = eq_table(ch.u)
    E2 = eq_table(ch.u[d - n:])
    vecs = [list(A), list(S), E,
            [B[x % N] for x in range(D)], [T[x % N] for x in range(D)],
            [m[x % N] % R for x in range(D)], [E2[x % N] for x in range(D)]]
    evals = []
    for k in range(1, d + 1):
        half = len(vecs[0]) // 2
        g = [0, 0, 0, 0]
        for y in range(half):
            for tt in range(4):
                vals = [(v[2 * y] + tt * (v[2 * y + 1] - v[2 * y])) % R for v in vecs]
                g[tt] = (g[tt] + tlookup_poly(*vals, ch.beta, ch.alpha1, ch.alpha2, w, variant)) % R
        evals.append(g)
        if next_r is not None:
            ch.r.append(next_r(k, g) % R)
        rk = ch.r[k - 1]
        vecs = [[(v[2 * y] + rk * (v[2 * y + 1] - v[2 * y])) % R for y in range(half)] for v in vecs]
    finals = {"A": vecs[0][0], "S": vecs[1][0], "B": vecs[3][0], "T": vecs[4][0], "m": vecs[5][0]}
    return Transcript(evals, finals)


def bound_point(ch_r: Sequence[int], d: int, k: int, t: int, z: int) -> List[int]:
    """Point of g_k(t)'s z-th term: coords 0..d-k-1 = bits of z, coord d-k = t, coord c > d-k = r_{d-c}."""
    free = bits_msb_first(z, d - k) if d - k > 0 else []
    return free + [t] + [ch_r[d - c - 1] for c in range(d - k + 1, d)]


def brute_force_round_polys(A, S, B, T, m, ch: Challenges, variant: int = PAPER):
    """g_k(t) = sum_{z in {0,1}^{d-k}} f~(z, t, r_{k-1}, ..., r_1), every MLE evaluated by its
    definition and e~ by its product formula.  Exponential; d <= 6."""
    D, N = len(A), len(B)
    d, n = log2_exact(D), log2_exact(N)
    w = N * F.inv(D) % R
    mf = [x % R for x in m]
    evals = []
    for k in range(1, d + 1):
        g = []
        for t in range(4):
            acc = 0
            for z in range(1 << (d - k)):
                p = bound_point(ch.r, d, k, t, z)
                pt = p[d - n:]
                acc += tlookup_poly(mle_eval(A, p), mle_eval(S, p), eq(ch.u, p),
                                    mle_eval(B, pt), mle_eval(T, pt), mle_eval(mf, pt),
                                    eq(ch.u[d - n:], pt), ch.beta, ch.alpha1, ch.alpha2, w, variant)
            g.append(acc % R)
        evals.append(g)
    v = [ch.r[d - c - 1] for c in range(d)]
    vt = v[d - n:]
    finals = {"A": mle_eval(A, v), "S": mle_eval(S, v), "B": mle_eval(B, vt),
              "T": mle_eval(T, vt), "m": mle_eval(mf, vt)}
    return Transcript(evals, finals)


def verify(tr: Transcript, D: int, N: int, ch: Challenges, variant: int = PAPER) -> bool:
    """Sumcheck verifier: g_1(0)+g_1(1) = claim, g_k(0)+g_k(1) = g_{k-1}(r_{k-1}),
    and g_d(r_d) = f(v) from the final evaluations (the proofs of evaluation of PAPER.md:277 are
    out of scope; the finals are taken as the committed values)."""
    d, n = log2_exact(D), log2_exact(N)
    if len(tr.evals) != d:
        return False
    claim = claimed_sum(ch.alpha1, ch.alpha2, variant)
    for k in range(d):
        g = tr.evals[k]
        if (g[0] + g[1]) % R != claim:
            return False
        claim = lagrange_0123(g, ch.r[k])
    v = [ch.r[d - c - 1] for c in range(d)]
    w = N * F.inv(D) % R
    f = tr.finals
    fv = tlookup_poly(f["A"], f["S"], eq(ch.u, v), f["B"], f["T"], f["m"], eq(ch.u[d - n:], v[d - n:]),
                      ch.beta, ch.alpha1, ch.alpha2, w, variant)
    return fv == claim


@dataclass
class Proof:
    m: List[int]
    A: List[int]
    B: List[int]
    transcript: Transcript


def prove(S: Sequence[int], T: Sequence[int], ch: Challenges, variant: int = PAPER) -> Proof:
    """Protocol 1 without the commitments: Prep (m), then Prove (A, B, sumcheck)."""
    D, N = len(S), len(T)
    check_shapes(D, N)
    check_canonical(T)
    check_canonical(S)
    check_table(T)
    m = multiplicities(S, T)                          # tlookup-Prep
    A, B = inverses(S, T, ch.beta, m, variant)
    tr = sumcheck_prove(A, S, B, T, m, ch, variant)
    return Proof(m, A, B, tr)


def challenges_from(w) -> Challenges:
    """Adapter from workloads.Challenges (plain integers) to this module's type."""
    return Challenges(w.beta % R, w.alpha1 % R, w.alpha2 % R, [x % R for x in w.u], [x % R for x in w.r])


def field_inputs(wl):
    """Build S, T in Fr from a workloads.Workload (function lookups: X + alpha_f Y)."""
    if wl.kind == "int":
        return [F.fr(int(v)) for v in wl.s], [F.fr(int(v)) for v in wl.t]
    af = wl.chal.alpha_f % R
    S = [(F.fr(int(x)) + af * F.fr(int(y))) % R for x, y in zip(wl.x, wl.y)]
    T = [(F.fr(int(x)) + af * F.fr(int(y))) % R for x, y in zip(wl.tx, wl.ty)]
    return S, T
