"""The multi-GPU partition of SURVEY.md §8(e), on CPU with torch.distributed (gloo, world size 2 and 4).

Each rank owns S[p D/P, (p+1) D/P) — the top log2 P hypercube coordinates are its rank bits — and runs the
local rounds on its slice only; the per-round D-side sums are all-gathered and summed mod r, the table-side
term (replicated) is added once, and after the local rounds the fully folded (A, S, e) of every rank are
all-gathered so the last log2 P rounds run identically on all ranks.  This is the exchange schedule the CUDA
path implements (csrc/nccl_loader.h); the test checks that it reproduces the single-rank oracle transcript
bit for bit.  Field arithmetic comes from the oracle (test infrastructure)."""
import os
import random
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import field as F
from oracle import tlookup as TL
from oracle.mle import eq_table

R = TL.R


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allgather_ints(vals, P):
    """all-gather a list of field elements (Python ints) over gloo as 32-bit limbs."""
    t = torch.tensor([[(v >> (32 * k)) & 0xFFFFFFFF for k in range(8)] for v in vals], dtype=torch.int64)
    out = [torch.zeros_like(t) for _ in range(P)]
    dist.all_gather(out, t)
    return [[sum(int(x) << (32 * k) for k, x in enumerate(row)) for row in o.tolist()] for o in out]


def _table_term(b, t, mm, e2, ch, variant):
    if variant == TL.PAPER:
        return b * ((ch.alpha2 * e2 % R) * ((t + ch.beta) % R) % R - mm) % R
    return (-b + (ch.alpha2 * e2 % R) * ((b * ((t + ch.beta) % R) - mm) % R)) % R


def _d_side(a, s, e, ch):
    return a * ((ch.alpha1 * e % R) * ((s + ch.beta) % R) % R + 1) % R


def _fold(v, r):
    return [(v[2 * y] + r * (v[2 * y + 1] - v[2 * y])) % R for y in range(len(v) // 2)]


def _partitioned(rank, P, S, T, ch, variant):
    D, N = len(S), len(T)
    d, n, pb = D.bit_length() - 1, N.bit_length() - 1, P.bit_length() - 1
    Dp = D // P
    dl = d - pb
    Sl = S[rank * Dp:(rank + 1) * Dp]
    # prepare: local counts, all-reduced (u32 sum)
    where = {t: j for j, t in enumerate(T)}
    mloc = [0] * N
    for s in Sl:
        mloc[where[s]] += 1
    mt = torch.tensor(mloc, dtype=torch.int64)
    dist.all_reduce(mt)
    m = [int(x) for x in mt.tolist()]
    A, B = TL.inverses(Sl, T, ch.beta, m, variant)
    # this rank's slice of e~(u, .): eq(u_top, rank) * eq(u_rest, i)
    E = eq_table(ch.u)[rank * Dp:(rank + 1) * Dp]
    # table side (replicated, N-sized, weight rule of SURVEY.md §8(a8))
    tb, tt, tm, te = list(B), list(T), [x % R for x in m], eq_table(ch.u[d - n:])
    tau, scale = None, 1
    inv2 = F.inv(2)
    evals = []
    vecs = [A, list(Sl), E]

    def table_round(k):
        nonlocal tb, tt, tm, te, tau, scale
        if k <= n:
            g = [0] * 4
            for y in range(len(tb) // 2):
                for q in range(4):
                    v = [(w[2 * y] + q * (w[2 * y + 1] - w[2 * y])) % R for w in (tb, tt, tm, te)]
                    g[q] = (g[q] + _table_term(*v, ch, variant)) % R
            rk = ch.r[k - 1]
            tb, tt, tm, te = _fold(tb, rk), _fold(tt, rk), _fold(tm, rk), _fold(te, rk)
            if k == n:
                tau = _table_term(tb[0], tt[0], tm[0], te[0], ch, variant)
            return g
        if tau is None:
            tau = _table_term(tb[0], tt[0], tm[0], te[0], ch, variant)
        scale = scale * inv2 % R
        return [tau * scale % R] * 4

    for k in range(1, d + 1):
        if k == dl + 1:   # gather the folded local values; the remaining rounds are replicated
            fins = _allgather_ints([vecs[0][0], vecs[1][0], vecs[2][0]], P)
            vecs = [[f[i] for f in fins] for i in range(3)]
        local = k <= dl
        g = [0] * 4
        for y in range(len(vecs[0]) // 2):
            for q in range(4):
                v = [(w[2 * y] + q * (w[2 * y + 1] - w[2 * y])) % R for w in vecs]
                g[q] = (g[q] + _d_side(*v, ch)) % R
        if local:
            g = [sum(col) % R for col in zip(*_allgather_ints(g, P))]
        tg = table_round(k)
        evals.append([(x + y) % R for x, y in zip(g, tg)])
        vecs = [_fold(v, ch.r[k - 1]) for v in vecs]
    if dl == d:   # P == 1
        pass
    finals = {"A": vecs[0][0], "S": vecs[1][0], "B": tb[0], "T": tt[0], "m": tm[0]}
    return evals, finals, m


def _worker(rank, P, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=P)
    S, T, ch = case
    res = [_partitioned(rank, P, S, T, ch, variant) for variant in (TL.PAPER, TL.LOGUP)]
    q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("P,d,n", [(2, 4, 2), (2, 5, 5), (4, 5, 3), (4, 6, 1), (2, 3, 0)])
def test_partitioned_transcript_equals_single_rank(P, d, n):
    rng = random.Random(P * 31 + d * 7 + n)
    D, N = 1 << d, 1 << n
    T = [rng.randrange(R) for _ in range(N)]
    S = [T[rng.randrange(N)] for _ in range(D)]
    ch = TL.Challenges(rng.randrange(R), rng.randrange(R), 0, [rng.randrange(R) for _ in range(d)],
                       [rng.randrange(R) for _ in range(d)])
    ch.alpha2 = ch.alpha1 ** 2 % R
    refs = [TL.prove(S, T, ch, variant) for variant in (TL.PAPER, TL.LOGUP)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, P, port, (S, T, ch), q)) for r in range(P)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(P))
    for p in procs:
        p.join(timeout=60)
    for r in range(P):
        for (evals, finals, m), ref in zip(results[r], refs):
            assert m == ref.m
            assert evals == ref.transcript.evals, f"rank {r}"
            assert finals == ref.transcript.finals, f"rank {r}"
