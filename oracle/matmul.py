"""Matrix-multiplication sumcheck — TEST INFRASTRUCTURE ONLY.

PAPER.md:463-467 (§5.1.1, "Matrix multiplications"): to confirm C = A B with A in F^{m x n}, B in F^{n x p},
prover and verifier run a sumcheck on

    C~(u, v) = sum_{i in {0,1}^{log2 n}} A~(u, i) B~(i, v)                       (Eq. matmul)

with u in F^{log2 m}, v in F^{log2 p} chosen by the verifier; prover time O(mn + np).

Readings: matrices are row-major, the row index is the high part of the flat index, so
A~(u, i) is the MLE of the flat vector A at the point (u, bits(i)) (coordinate 0 = MSB, as for tlookup);
the sumcheck binds the coordinates of i least significant first (round k binds coordinate log2(n) - k,
pairs (2y, 2y+1)), exactly as the tlookup sumcheck; the summand has degree 2, so each round sends
g_k(0), g_k(1), g_k(2).  Entries are quantised integers mapped into F (negative x -> r - |x|).
"""
from dataclasses import dataclass
from typing import List, Sequence

from . import field as F
from .field import R
from .mle import bits_msb_first, eq, eq_table, mle_eval


def log2_exact(x: int) -> int:
    if x < 1 or x & (x - 1):
        raise ValueError(f"{x} is not a power of two")
    return x.bit_length() - 1


@dataclass
class MatmulProof:
    a: List[int]            # a_i = A~(u, i), i in [n]
    b: List[int]            # b_i = B~(i, v)
    claim: int              # sum_i a_i b_i = C~(u, v)
    evals: List[List[int]]  # evals[k-1] = [g_k(0), g_k(1), g_k(2)]
    finals: List[int]       # [a~(w), b~(w)] at the bound point w


def restrict_rows(A: Sequence[Sequence[int]], u: Sequence[int]) -> List[int]:
    """a_i = A~(u, i) = sum_r e~(u, bits(r)) A[r][i]: Eq. MLE with the column bits fixed."""
    m, n = len(A), len(A[0])
    assert len(u) == log2_exact(m)
    E = eq_table(u)
    return [sum(E[r] * A[r][i] for r in range(m)) % R for i in range(n)]


def restrict_cols(B: Sequence[Sequence[int]], v: Sequence[int]) -> List[int]:
    """b_i = B~(i, v) = sum_c e~(v, bits(c)) B[i][c]."""
    n, p = len(B), len(B[0])
    assert len(v) == log2_exact(p)
    E = eq_table(v)
    return [sum(E[c] * B[i][c] for c in range(p)) % R for i in range(n)]


def sumcheck_prove(a: Sequence[int], b: Sequence[int], r: Sequence[int]):
    """Sumcheck of sum_i a~(i) b~(i): round k evaluates, for every pair (2y, 2y+1),
    a_t = a_0 + t (a_1 - a_0) and b_t likewise at t = 0, 1, 2 and sums a_t b_t; then folds both with r_k."""
    n = len(a)
    L = log2_exact(n)
    assert len(b) == n and len(r) == L
    va, vb = [x % R for x in a], [x % R for x in b]
    evals = []
    for k in range(1, L + 1):
        half = len(va) // 2
        g = [0, 0, 0]
        for y in range(half):
            for t in range(3):
                at = (va[2 * y] + t * (va[2 * y + 1] - va[2 * y])) % R
                bt = (vb[2 * y] + t * (vb[2 * y + 1] - vb[2 * y])) % R
                g[t] = (g[t] + at * bt) % R
        evals.append(g)
        rk = r[k - 1]
        va = [(va[2 * y] + rk * (va[2 * y + 1] - va[2 * y])) % R for y in range(half)]
        vb = [(vb[2 * y] + rk * (vb[2 * y + 1] - vb[2 * y])) % R for y in range(half)]
    return evals, [va[0], vb[0]]


def prove(A, B, u, v, r) -> MatmulProof:
    """The prover of Eq. matmul: restrictions a, b (O(mn + np)), the claim, the log2(n)-round sumcheck."""
    a = restrict_rows(A, u)
    b = restrict_cols(B, v)
    claim = sum(x * y for x, y in zip(a, b)) % R
    evals, finals = sumcheck_prove(a, b, r)
    return MatmulProof(a, b, claim, evals, finals)


def lagrange_012(g: Sequence[int], x: int) -> int:
    """Value at x of the degree-2 polynomial with values g[0..2] at 0, 1, 2."""
    nodes = [0, 1, 2]
    acc = 0
    for i, xi in enumerate(nodes):
        num, den = 1, 1
        for j, xj in enumerate(nodes):
            if j != i:
                num = num * (x - xj) % R
                den = den * (xi - xj) % R
        acc = (acc + g[i] * num % R * F.inv(den)) % R
    return acc


def verify(claim: int, evals, finals, n: int, r: Sequence[int]) -> bool:
    """g_1(0)+g_1(1) = claim, g_k(0)+g_k(1) = g_{k-1}(r_{k-1}), g_L(r_L) = a~(w) b~(w)."""
    L = log2_exact(n)
    if len(evals) != L:
        return False
    cur = claim % R
    for k in range(L):
        g = evals[k]
        if (g[0] + g[1]) % R != cur:
            return False
        cur = lagrange_012(g, r[k])
    return cur == finals[0] * finals[1] % R


def bound_w(r: Sequence[int], L: int) -> List[int]:
    """The point the sumcheck binds: coordinate c gets r_{L-c} (round k binds coordinate L - k)."""
    return [r[L - c - 1] for c in range(L)]


def brute_force_round_polys(a: Sequence[int], b: Sequence[int], r: Sequence[int]):
    """g_k(t) = sum_{z in {0,1}^{L-k}} a~(z, t, r_{k-1}..r_1) b~(same), each MLE by its definition.  L <= 6."""
    n = len(a)
    L = log2_exact(n)
    evals = []
    for k in range(1, L + 1):
        g = []
        for t in range(3):
            acc = 0
            for z in range(1 << (L - k)):
                free = bits_msb_first(z, L - k) if L - k > 0 else []
                pt = free + [t] + [r[L - c - 1] for c in range(L - k + 1, L)]
                acc += mle_eval(a, pt) * mle_eval(b, pt)
            g.append(acc % R)
        evals.append(g)
    w = bound_w(r, L)
    return evals, [mle_eval(a, w), mle_eval(b, w)]


def matmul(A, B):
    """C = A B over F (the plain definition)."""
    m, n, p = len(A), len(B), len(B[0])
    return [[sum(A[i][k] * B[k][j] for k in range(n)) % R for j in range(p)] for i in range(m)]


def flat(M):
    return [x for row in M for x in row]


def eval_matrix_mle(M, u_rows: Sequence[int], v_cols: Sequence[int]) -> int:
    """M~(u, v): the MLE of the row-major flat vector at the point (u, v) (rows = high bits)."""
    return mle_eval(flat(M), list(u_rows) + list(v_cols))


def field_matrix(ints) -> List[List[int]]:
    """Quantised integers -> F (x < 0 -> r - |x|)."""
    return [[F.fr(int(x)) for x in row] for row in ints]
