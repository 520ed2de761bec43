"""Matmul sumcheck on the GPU against the oracle (oracle/matmul.py).

Element by element: the restrictions a = A~(u, .) and b = B~(., v), the claim, every round polynomial and both
finals, for shapes that exercise every stage (n = 1; one chunk; several chunks + the one-warp tail; the multi-block
rounds before the chunks), int32 entries over the full range (the 320-bit accumulation with the 2^31 offset), and
at LLaMA-like shapes the oracle can still do (sampled restriction entries + the verifier)."""
import random

import numpy as np
import pytest

from oracle import matmul as MM
from oracle.field import R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2404_16109_b200 import zkl
    c = zkl.Context(0)
    yield c
    c.close()


def _mats(rng, m, n, p, lo, hi):
    A = np.array([[rng.randrange(lo, hi) for _ in range(n)] for _ in range(m)], dtype=np.int64)
    B = np.array([[rng.randrange(lo, hi) for _ in range(p)] for _ in range(n)], dtype=np.int64)
    return A, B


def _ref(A, B, u, v, r):
    return MM.prove(MM.field_matrix(A.tolist()), MM.field_matrix(B.tolist()), u, v, r)


@pytest.mark.parametrize("m,n,p,lo,hi,seed", [
    (1, 1, 1, -5, 5, 0), (2, 2, 2, -(1 << 31), 1 << 31, 1), (4, 8, 2, -(1 << 15), 1 << 15, 2),
    (16, 64, 8, -(1 << 31), 1 << 31, 3), (128, 256, 64, -(1 << 15), 1 << 15, 4), (64, 2048, 16, -100, 100, 5),
    (8, 1 << 12, 4, -(1 << 31), 1 << 31, 6), (2, 1 << 14, 2, -(1 << 20), 1 << 20, 7)])
def test_matmul_parity(ctx, m, n, p, lo, hi, seed):
    rng = random.Random(seed)
    A, B = _mats(rng, m, n, p, lo, hi)
    u = [rng.randrange(R) for _ in range(MM.log2_exact(m))]
    v = [rng.randrange(R) for _ in range(MM.log2_exact(p))]
    r = [rng.randrange(R) for _ in range(MM.log2_exact(n))]
    got = ctx.matmul_prove(A.astype(np.int32), B.astype(np.int32), u, v, r, want_ab=True)
    ref = _ref(A, B, u, v, r)
    assert ctx.export_ints(got["a"]) == ref.a
    assert ctx.export_ints(got["b"]) == ref.b
    assert got["claim"] == ref.claim
    assert got["evals"] == ref.evals
    assert got["finals"] == ref.finals
    assert MM.verify(got["claim"], got["evals"], got["finals"], n, r)


def test_matmul_multiblock_rounds(ctx):
    """n = 2^18 > 2^17: the first round runs multi-block before the chunks.  The sumcheck alone is compared
    with the oracle's on the GPU's own restrictions (which are checked on a sample against the definition)."""
    rng = random.Random(11)
    m, n, p = 2, 1 << 18, 2
    A = np.array([[rng.randrange(-1000, 1000) for _ in range(n)] for _ in range(m)], dtype=np.int32)
    B = np.array([[rng.randrange(-1000, 1000) for _ in range(p)] for _ in range(n)], dtype=np.int32)
    u, v = [rng.randrange(R)], [rng.randrange(R)]
    r = [rng.randrange(R) for _ in range(18)]
    got = ctx.matmul_prove(A, B, u, v, r, want_ab=True)
    a, b = ctx.export_ints(got["a"]), ctx.export_ints(got["b"])
    for i in rng.sample(range(n), 64):
        assert a[i] == ((1 - u[0]) * int(A[0, i]) + u[0] * int(A[1, i])) % R
        assert b[i] == ((1 - v[0]) * int(B[i, 0]) + v[0] * int(B[i, 1])) % R
    evals, finals = MM.sumcheck_prove(a, b, r)
    assert got["evals"] == evals and got["finals"] == finals
    assert got["claim"] == sum(x * y for x, y in zip(a, b)) % R


def test_matmul_llama_shape_verifies(ctx):
    """A LLaMA-2-7B projection slice (m = 64 tokens, n = 4096, p = 4096, int16-range weights): the GPU transcript
    verifies, and sampled a_i / b_i equal their definitions."""
    rng = np.random.default_rng(3)
    m, n, p = 64, 4096, 4096
    A = rng.integers(-(1 << 15), 1 << 15, size=(m, n), dtype=np.int32)
    B = rng.integers(-(1 << 15), 1 << 15, size=(n, p), dtype=np.int32)
    prng = random.Random(5)
    u = [prng.randrange(R) for _ in range(6)]
    v = [prng.randrange(R) for _ in range(12)]
    r = [prng.randrange(R) for _ in range(12)]
    got = ctx.matmul_prove(A, B, u, v, r, want_ab=True)
    assert MM.verify(got["claim"], got["evals"], got["finals"], n, r)
    from oracle import mle
    Eu, Ev = mle.eq_table(u), mle.eq_table(v)
    a, b = ctx.export_ints(got["a"]), ctx.export_ints(got["b"])
    for i in prng.sample(range(n), 6):
        assert a[i] == sum(Eu[rr] * int(A[rr, i]) for rr in range(m)) % R
        assert b[i] == sum(int(B[i, c]) * Ev[c] for c in range(p)) % R
    assert got["claim"] == sum(x * y for x, y in zip(a, b)) % R


def test_matmul_errors(ctx):
    from paper_2404_16109_b200 import zkl
    with pytest.raises(zkl.ZklError) as e:
        ctx.matmul_prove(np.zeros((3, 4), np.int32), np.zeros((4, 2), np.int32), [1, 2], [1], [1, 2])
    assert e.value.name == "ZKL_E_SHAPE"
    # the C ABI itself refuses non-canonical challenges (the binding reduces mod r before the call)
    import ctypes
    A = ctx.torch.zeros((2, 2), dtype=ctx.torch.int32, device=ctx.device)
    bad = (zkl.zkl_fr * 1)()
    for i in range(8):
        bad[0].w[i] = 0xFFFFFFFF
    one = (zkl.zkl_fr * 1)()
    one[0].w[0] = 1
    claim, ev, fin = zkl.zkl_fr(), (zkl.zkl_fr * 3)(), (zkl.zkl_fr * 2)()
    st = zkl.lib().zkl_matmul_prove(ctx.h, ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(A.data_ptr()), 2, 2, 2,
                                    bad, one, one, zkl.zkl_vec(None, 2), zkl.zkl_vec(None, 2), ctypes.byref(claim),
                                    ev, fin)
    assert zkl.STATUS[st] == "ZKL_E_NONCANONICAL"
