"""Pins for the matmul-sumcheck oracle, CPU only.

Each check ties the oracle to something other than itself: Eq. matmul evaluated through C = A B and the MLE
definition, the boolean-point special case (e~ is the equality indicator), the identity matrix, brute force
through the MLE definition for every round polynomial, and verifier acceptance / rejection."""
import random

import pytest

from oracle import matmul as MM
from oracle import mle
from oracle.field import R


def _rand_matrix(rng, rows, cols, lo=-(1 << 15), hi=(1 << 15)):
    return [[rng.randrange(lo, hi) for _ in range(cols)] for _ in range(rows)]


@pytest.mark.parametrize("m,n,p,seed", [(1, 1, 1, 0), (2, 4, 2, 1), (4, 8, 2, 2), (8, 4, 16, 3), (2, 16, 4, 4)])
def test_claim_is_C_mle(m, n, p, seed):
    """Eq. matmul: sum_i A~(u,i) B~(i,v) equals C~(u,v) of the product C = A B."""
    rng = random.Random(seed)
    A = MM.field_matrix(_rand_matrix(rng, m, n))
    B = MM.field_matrix(_rand_matrix(rng, n, p))
    u = [rng.randrange(R) for _ in range(MM.log2_exact(m))]
    v = [rng.randrange(R) for _ in range(MM.log2_exact(p))]
    r = [rng.randrange(R) for _ in range(MM.log2_exact(n))]
    pf = MM.prove(A, B, u, v, r)
    assert pf.claim == MM.eval_matrix_mle(MM.matmul(A, B), u, v)
    if n > 1:
        assert (pf.evals[0][0] + pf.evals[0][1]) % R == pf.claim


def test_boolean_points_select_rows_and_columns():
    """At boolean u, v the restrictions are a row of A and a column of B (e~ = equality indicator)."""
    rng = random.Random(7)
    m, n, p = 8, 4, 4
    A = MM.field_matrix(_rand_matrix(rng, m, n))
    B = MM.field_matrix(_rand_matrix(rng, n, p))
    for row in range(m):
        u = mle.bits_msb_first(row, 3)
        assert MM.restrict_rows(A, u) == A[row]
    for col in range(p):
        v = mle.bits_msb_first(col, 2)
        assert MM.restrict_cols(B, v) == [B[i][col] for i in range(n)]


def test_identity_matrix():
    """A = I (m = n): C = B, so the claim is B~(u, v) and a_i = e~(u, bits(i))."""
    rng = random.Random(9)
    n, p = 8, 4
    A = [[1 if i == j else 0 for j in range(n)] for i in range(n)]
    B = MM.field_matrix(_rand_matrix(rng, n, p))
    u = [rng.randrange(R) for _ in range(3)]
    v = [rng.randrange(R) for _ in range(2)]
    pf = MM.prove(A, B, u, v, [rng.randrange(R) for _ in range(3)])
    assert pf.a == [mle.eq(u, mle.bits_msb_first(i, 3)) for i in range(n)]
    assert pf.claim == MM.eval_matrix_mle(B, u, v)


@pytest.mark.parametrize("L,seed", [(1, 0), (2, 1), (3, 2), (5, 3)])
def test_round_polys_brute_force(L, seed):
    """Every g_k(t) and both finals equal the brute-force sums through the MLE definition."""
    rng = random.Random(seed)
    n = 1 << L
    a = [rng.randrange(R) for _ in range(n)]
    b = [rng.randrange(R) for _ in range(n)]
    r = [rng.randrange(R) for _ in range(L)]
    assert MM.sumcheck_prove(a, b, r) == MM.brute_force_round_polys(a, b, r)


def test_verifier_accepts_and_rejects():
    rng = random.Random(11)
    m, n, p = 4, 16, 8
    A = MM.field_matrix(_rand_matrix(rng, m, n))
    B = MM.field_matrix(_rand_matrix(rng, n, p))
    u = [rng.randrange(R) for _ in range(2)]
    v = [rng.randrange(R) for _ in range(3)]
    r = [rng.randrange(R) for _ in range(4)]
    pf = MM.prove(A, B, u, v, r)
    assert MM.verify(pf.claim, pf.evals, pf.finals, n, r)
    assert not MM.verify((pf.claim + 1) % R, pf.evals, pf.finals, n, r)
    bad = [list(g) for g in pf.evals]
    bad[2][2] = (bad[2][2] + 1) % R
    assert not MM.verify(pf.claim, bad, pf.finals, n, r)
    assert not MM.verify(pf.claim, pf.evals, [pf.finals[0], (pf.finals[1] + 1) % R], n, r)
    # a wrong product: C' = A B + E claims a different C~(u, v)
    C = MM.matmul(A, B)
    C[1][3] = (C[1][3] + 1) % R
    assert MM.eval_matrix_mle(C, u, v) != pf.claim


def test_negative_entries_map_to_r_minus():
    """Quantised negatives are r - |x|; the restriction is linear in them."""
    A = MM.field_matrix([[-1, 2], [3, -4]])
    assert A == [[R - 1, 2], [3, R - 4]]
    u = [5]
    # a_i = (1-u) A[0][i] + u A[1][i]
    assert MM.restrict_rows(A, u) == [((1 - 5) * -1 + 5 * 3) % R, ((1 - 5) * 2 + 5 * -4) % R]
