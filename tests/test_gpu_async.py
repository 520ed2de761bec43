"""Many instances in flight: async mode on K contexts, each with its own CUDA stream.

Every instance's m, transcript and finals must equal the C oracle's, whatever the interleaving of the K
streams; errors come back from wait() with the failing call's index; a proof whose prepared keys miss
falls back to the inversion inside wait(); an FS proof completes through wait() as well."""
import hashlib
import random

import numpy as np
import pytest

from oracle import c_oracle as C
from oracle import tlookup as TL
from tests.fs_transcript import derive

pytestmark = pytest.mark.gpu
R = TL.R


def _instance(rng, d, n):
    T = [rng.randrange(R) for _ in range(1 << n)]
    hot = rng.randrange(1 << n)
    S = [T[hot] if rng.random() < 0.3 else T[rng.randrange(1 << n)] for _ in range(1 << d)]
    u = [rng.randrange(R) for _ in range(d)]
    r = [rng.randrange(R) for _ in range(d)]
    return T, S, (rng.randrange(R), rng.randrange(R), rng.randrange(R), u, r)


@pytest.fixture(scope="module")
def ctxs():
    import torch
    from paper_2404_16109_b200 import zkl
    cs = [zkl.Context(0, stream=torch.cuda.Stream()) for _ in range(4)]
    yield cs
    for c in cs:
        c.close()


@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
def test_async_instances_match_oracle(ctxs, variant):
    import torch
    from paper_2404_16109_b200 import zkl
    rng = random.Random(11 + variant)
    shapes = [(12, 6), (15, 10), (13, 13), (16, 8), (11, 3), (14, 12), (17, 9), (12, 12)]
    insts = [_instance(rng, d, n) for d, n in shapes]
    for c in ctxs:
        c.reserve(1 << 17, 1 << 13)
    results = [None] * len(insts)
    # rounds of len(ctxs) instances in flight
    for base in range(0, len(insts), len(ctxs)):
        live = []
        for c, idx in zip(ctxs, range(base, min(base + len(ctxs), len(insts)))):
            T, S, (beta, a1, a2, u, r) = insts[idx]
            D = len(S)
            with torch.cuda.stream(c.stream):
                tab = c.table(c.import_canon(zkl.ints_to_canon(T)))
                Sv = c.import_canon(zkl.ints_to_canon(S))
            c.set_async(True)
            m = c.prepare(Sv, D, tab)
            pf = c.prove(Sv, D, tab, m, zkl.Context.challenges(beta, a1, a2, u, r), variant)
            live.append((c, idx, m, pf, tab))
        for c, idx, m, pf, tab in live:
            c.wait()
            c.set_async(False)
            results[idx] = (m.cpu().numpy().astype(np.uint32), pf.result())
    for (T, S, (beta, a1, a2, u, r)), (m, pf) in zip(insts, results):
        ref = C.prove(C.ints_to_limbs(S), C.ints_to_limbs(T), C.chal_array(beta, a1, a2, u, r), variant)
        assert np.array_equal(m, ref.m)
        assert pf.evals == ref.evals and pf.finals == ref.finals


def test_async_errors_and_fallback(ctxs):
    import torch
    from paper_2404_16109_b200 import zkl
    rng = random.Random(3)
    c0, c1 = ctxs[0], ctxs[1]
    d, n = 13, 7
    T, S, (beta, a1, a2, u, r) = _instance(rng, d, n)
    D = len(S)
    for c in (c0, c1):
        c.reserve(D, 1 << n)
    # c0: NOT_IN_TABLE at index 777 reported by wait(); the pending proof's result is not delivered
    bad = list(S)
    bad[777] = rng.randrange(R)
    bad[900] = rng.randrange(R)
    with torch.cuda.stream(c0.stream):
        tab0 = c0.table(c0.import_canon(zkl.ints_to_canon(T)))
        Sb = c0.import_canon(zkl.ints_to_canon(bad))
    # c1: prepared on S, then S overwritten IN PLACE by S' (one element replaced by another table entry): the
    # cached keys miss at that element, so wait() reruns the proof through the inversion path
    S2 = list(S)
    S2[5] = T[(T.index(S[5]) + 1) % len(T)]
    with torch.cuda.stream(c1.stream):
        tab1 = c1.table(c1.import_canon(zkl.ints_to_canon(T)))
        Sv = c1.import_canon(zkl.ints_to_canon(S))
    c0.set_async(True)
    c1.set_async(True)
    c0.prepare(Sb, D, tab0)
    pf0 = c0.prove(Sb, D, tab0, torch.zeros(1 << n, dtype=torch.int32, device=c0.device),
                   zkl.Context.challenges(beta, a1, a2, u, r))
    with pytest.raises(zkl.ZklError) as ei:   # a second pending prove on one ctx
        c0.prove(Sb, D, tab0, torch.zeros(1 << n, dtype=torch.int32, device=c0.device),
                 zkl.Context.challenges(beta, a1, a2, u, r))
    assert ei.value.name == "ZKL_E_STATE"
    m1 = c1.prepare(Sv, D, tab1)
    c1.wait()                                   # completes the prepare of S
    m_S = m1.cpu().numpy().astype(np.uint32)
    c1.import_canon(zkl.ints_to_canon(S2), dst=Sv)
    m2 = torch.from_numpy(np.bincount([T.index(s) for s in S2], minlength=1 << n).astype(np.int32)).to(c1.device)
    pf1 = c1.prove(Sv, D, tab1, m2, zkl.Context.challenges(beta, a1, a2, u, r))
    with pytest.raises(zkl.ZklError) as ei:
        c0.wait()
    assert ei.value.name == "ZKL_E_NOT_IN_TABLE" and ei.value.index == 777
    assert not pf0.done
    c1.wait()
    ref = C.prove(C.ints_to_limbs(S2), C.ints_to_limbs(T), C.chal_array(beta, a1, a2, u, r), TL.PAPER)
    assert np.array_equal(m2.cpu().numpy().astype(np.uint32), ref.m)
    assert pf1.result().evals == ref.evals and pf1.result().finals == ref.finals
    assert np.array_equal(m_S, np.bincount([T.index(s) for s in S], minlength=1 << n).astype(np.uint32))
    for c in (c0, c1):
        c.set_async(False)


def test_async_fs(ctxs):
    import torch
    from paper_2404_16109_b200 import zkl
    rng = random.Random(19)
    c = ctxs[2]
    d, n = 14, 6
    T, S, _ = _instance(rng, d, n)
    D, N = len(S), len(T)
    c.reserve(D, N)
    with torch.cuda.stream(c.stream):
        tab = c.table(c.import_canon(zkl.ints_to_canon(T)))
        Sv = c.import_canon(zkl.ints_to_canon(S))
    seed = hashlib.sha256(b"async-fs").digest()
    c.set_async(True)
    m = c.prepare(Sv, D, tab)
    res = c.prove_fs(Sv, D, tab, m, seed, TL.LOGUP)
    c.wait()
    c.set_async(False)
    pf, der = res.result()
    assert der == derive(seed, D, N, TL.LOGUP, pf.evals)
    ref = C.prove(C.ints_to_limbs(S), C.ints_to_limbs(T),
                  C.chal_array(der["beta"], der["alpha1"], der["alpha2"], der["u"], der["r"]), TL.LOGUP)
    assert pf.evals == ref.evals and pf.finals == ref.finals
