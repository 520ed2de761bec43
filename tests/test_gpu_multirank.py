"""The P > 1 path on one GPU: P virtual ranks (host threads, one ctx + stream each) with the loopback
communicator.  Each rank holds the contiguous slice S[p D/P, (p+1) D/P) (top log2 P hypercube variables =
rank); the transcript must be bit-identical to the single-rank oracle's."""
import random
import threading

import numpy as np
import pytest

from oracle import c_oracle as C
from oracle import tlookup as TL

pytestmark = pytest.mark.gpu
R = TL.R


def _run_ranks(P, D, S, T, ch, variant, want_sumcheck=False):
    import torch
    from paper_2404_16109_b200 import zkl
    N = len(T)
    Dp = D // P
    group = zkl.LoopbackGroup(P, max_D_local=Dp, max_N=N)
    out, errs = [None] * P, []

    def rank_main(p):
        try:
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                ctx = zkl.Context(0, stream=stream, rank=p, group=group)
                ctx.reserve(Dp, N)
                Sv = ctx.import_canon(zkl.ints_to_canon(S[p * Dp:(p + 1) * Dp]))
                Tv = ctx.import_canon(zkl.ints_to_canon(T))
                tab = ctx.table(Tv)
                m = ctx.prepare(Sv, D, tab)
                chg = zkl.Context.challenges(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)
                pf = ctx.prove(Sv, D, tab, m, chg, variant, want_A=True)
                A = ctx.export_ints(pf.A)
                out[p] = (m.cpu().numpy().astype(np.uint32), pf, A)
                ctx.close()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=rank_main, args=(p,)) for p in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    group.close()
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("P,d,n", [(2, 5, 2), (2, 13, 4), (4, 14, 6), (8, 15, 3), (2, 16, 16), (8, 12, 12)])
@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
def test_loopback_ranks_match_oracle(P, d, n, variant):
    rng = random.Random(P * 100 + d * 7 + n + variant)
    D, N = 1 << d, 1 << n
    T = [rng.randrange(R) for _ in range(N)]
    S = [T[rng.randrange(N)] for _ in range(D)]
    ch = TL.Challenges(rng.randrange(R), rng.randrange(R), 0, [rng.randrange(R) for _ in range(d)],
                       [rng.randrange(R) for _ in range(d)])
    ch.alpha2 = ch.alpha1 ** 2 % R
    ref = C.prove(C.ints_to_limbs(S), C.ints_to_limbs(T), C.chal_array(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r),
                  variant)
    refA = C.limbs_to_ints(ref.A)
    out = _run_ranks(P, D, S, T, ch, variant)
    Dp = D // P
    for p, (m, pf, A) in enumerate(out):
        assert np.array_equal(m, ref.m), f"rank {p}: m"
        assert A == refA[p * Dp:(p + 1) * Dp], f"rank {p}: A slice"
        assert pf.evals == ref.evals, f"rank {p}: round polynomials"
        assert pf.finals == ref.finals, f"rank {p}: finals"


def test_loopback_not_in_table_smallest_global_index():
    import torch
    from paper_2404_16109_b200 import zkl
    P, D, N = 4, 1 << 13, 1 << 5
    S = [i % N for i in range(D)]
    S[5000] = 999       # rank 2
    S[7000] = 1000      # rank 3
    S[3000] = 1001      # rank 1: the smallest global index
    group = zkl.LoopbackGroup(P, max_D_local=D // P, max_N=N)
    res = [None] * P

    def rank_main(p):
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            ctx = zkl.Context(0, stream=stream, rank=p, group=group)
            ctx.reserve(D // P, N)
            Sv = ctx.import_ints(np.array(S[p * D // P:(p + 1) * D // P], dtype=np.int64))
            tab = ctx.table(ctx.import_ints(np.arange(N, dtype=np.int64)))
            try:
                ctx.prepare(Sv, D, tab)
                res[p] = None
            except zkl.ZklError as e:
                res[p] = (e.name, e.index)
            ctx.close()

    th = [threading.Thread(target=rank_main, args=(p,)) for p in range(P)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    group.close()
    assert all(r == ("ZKL_E_NOT_IN_TABLE", 3000) for r in res), res


@pytest.mark.parametrize("bad", [False, True])
def test_loopback_pair_range_prepare(bad):
    """P = 4 ranks, function lookups through the pair-range fast path (zkl_table_attach_pair): m summed over the
    ranks equals the global histogram; with a pair off the graph on rank 2 (and another on rank 3), every rank's
    fast path falls back to the hash index and all report NOT_IN_TABLE at the smallest global index."""
    import torch
    from paper_2404_16109_b200 import zkl
    P, D, N = 4, 1 << 14, 1 << 8
    tx = np.arange(N, dtype=np.int32) - 128
    ty = (tx * 5 - 3).astype(np.int32)
    rng = np.random.default_rng(9)
    x = rng.integers(-128, 128, D).astype(np.int32)
    y = (x * 5 - 3).astype(np.int32)
    if bad:
        y[9001] += 1        # rank 2
        y[13000] += 2       # rank 3
    group = zkl.LoopbackGroup(P, max_D_local=D // P, max_N=N)
    res = [None] * P

    def rank_main(p):
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            ctx = zkl.Context(0, stream=stream, rank=p, group=group)
            ctx.reserve(D // P, N)
            tab = ctx.table(ctx.import_pair(tx, ty, 4242))
            assert ctx.table_attach_pair(tab, tx, ty, 4242)
            sl = slice(p * D // P, (p + 1) * D // P)
            try:
                _, m = ctx.prepare_pair(x[sl], y[sl], 4242, D, tab)
                res[p] = m.cpu().numpy().astype(np.int64)
            except zkl.ZklError as e:
                res[p] = (e.name, e.index)
            ctx.close()

    th = [threading.Thread(target=rank_main, args=(p,)) for p in range(P)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    group.close()
    if bad:
        assert all(r == ("ZKL_E_NOT_IN_TABLE", 9001) for r in res), res
    else:
        ref = np.bincount(x.astype(np.int64) + 128, minlength=N)
        for r in res:
            assert np.array_equal(r, ref)
