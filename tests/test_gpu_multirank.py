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


def _run_ranks_pair(P, D, x, y, tx, ty, ch, variant):
    """P loopback ranks, each proving its slice of a function lookup through prepare_pair with a virtual S."""
    import torch
    from paper_2404_16109_b200 import zkl
    N = len(tx)
    Dp = D // P
    group = zkl.LoopbackGroup(P, max_D_local=Dp, max_N=N)
    out, errs = [None] * P, []

    def rank_main(p):
        try:
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                ctx = zkl.Context(0, stream=stream, rank=p, group=group)
                ctx.reserve(Dp, N)
                tab = ctx.table(ctx.import_pair(tx, ty, ch.alpha_f))
                assert ctx.table_attach_pair(tab, tx, ty, ch.alpha_f)
                _, m = ctx.prepare_pair(x[p * Dp:(p + 1) * Dp], y[p * Dp:(p + 1) * Dp], ch.alpha_f, D, tab,
                                        virtual_s=True)
                chg = zkl.Context.challenges(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)
                pf = ctx.prove(None, D, tab, m, chg, variant)
                out[p] = (m.cpu().numpy().astype(np.uint32), pf)
                ctx.close()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=rank_main, args=(p,)) for p in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    group.close()
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("P,dl", [(2, 19), (8, 20)])
@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
def test_loopback_big_local_rounds(P, dl, variant):
    """D_local >= 2^19: the multi-block k_round rounds (with the round-2 gather of the virtual S) and the causal
    chunked rounds run under P > 1; bit-identical to the single-rank oracle."""
    import workloads as W
    D = P << dl
    d, n = D.bit_length() - 1, 16
    N = 1 << n
    rng = np.random.default_rng(P * 1000 + dl + variant)
    tx = (np.arange(N) - N // 2).astype(np.int32)
    ty = rng.integers(-2 ** 31, 2 ** 31, N, dtype=np.int64).astype(np.int32)
    pick = np.clip(np.rint(N / 2 + rng.normal(0, N / 8, D)), 0, N - 1).astype(np.int64)
    x, y = tx[pick], ty[pick]
    ch = W.challenges(f"loop{P}.{dl}", d)
    chal = C.chal_array(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)
    ref = C.prove_pair_stream(x, y, tx, ty, ch.alpha_f, chal, variant, 2)
    out = _run_ranks_pair(P, D, x, y, tx, ty, ch, variant)
    for m, pf in out:
        assert np.array_equal(m, ref.m)
        assert pf.evals == ref.evals and pf.finals == ref.finals


def _run_ranks_pair_fs(P, D, x, y, tx, ty, alpha_f, seed, variant):
    import torch
    from paper_2404_16109_b200 import zkl
    N = len(tx)
    Dp = D // P
    group = zkl.LoopbackGroup(P, max_D_local=Dp, max_N=N)
    out, errs = [None] * P, []

    def rank_main(p):
        try:
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                ctx = zkl.Context(0, stream=stream, rank=p, group=group)
                ctx.reserve(Dp, N)
                tab = ctx.table(ctx.import_pair(tx, ty, alpha_f))
                assert ctx.table_attach_pair(tab, tx, ty, alpha_f)
                _, m = ctx.prepare_pair(x[p * Dp:(p + 1) * Dp], y[p * Dp:(p + 1) * Dp], alpha_f, D, tab,
                                        virtual_s=True)
                out[p] = ctx.prove_fs(None, D, tab, m, seed, variant)
                ctx.close()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=rank_main, args=(p,)) for p in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    group.close()
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("P,dl,n", [(2, 15, 16), (4, 18, 16), (8, 20, 16), (8, 3, 4)])
@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
def test_loopback_fiat_shamir(P, dl, n, variant):
    """Fiat-Shamir at P > 1 (one all-gather of the round sums per local round, then the replicated last log2 P
    rounds): every rank derives the same challenges, and the transcript equals the single-rank one and the oracle's
    on those challenges."""
    import hashlib
    import workloads as W
    from paper_2404_16109_b200 import zkl
    D = P << dl
    N = 1 << n
    rng = np.random.default_rng(P * 77 + dl + variant)
    tx = (np.arange(N) - N // 2).astype(np.int32)
    ty = rng.integers(-2 ** 31, 2 ** 31, N, dtype=np.int64).astype(np.int32)
    pick = np.clip(np.rint(N / 2 + rng.normal(0, N / 8, D)), 0, N - 1).astype(np.int64)
    x, y = tx[pick], ty[pick]
    alpha_f = W.chal(f"fsloop{P}", "alpha_f", 0)
    seed = hashlib.sha256(f"fs-loopback-{P}-{dl}".encode()).digest()
    out = _run_ranks_pair_fs(P, D, x, y, tx, ty, alpha_f, seed, variant)
    ctx = zkl.Context(0)
    ctx.reserve(D, N)
    tab = ctx.table(ctx.import_pair(tx, ty, alpha_f))
    _, m = ctx.prepare_pair(x, y, alpha_f, D, tab, virtual_s=True)
    ref, dref = ctx.prove_fs(None, D, tab, m, seed, variant)
    ctx.close()
    chal = C.chal_array(dref["beta"], dref["alpha1"], dref["alpha2"], dref["u"], dref["r"])
    o = C.prove_pair_stream(x, y, tx, ty, alpha_f, chal, variant, 2)
    assert ref.evals == o.evals and ref.finals == o.finals
    for pf, der in out:
        assert der == dref
        assert pf.evals == ref.evals and pf.finals == ref.finals
