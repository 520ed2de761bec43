"""Fiat-Shamir mode: the device derives every challenge from a SHA-256 transcript.

Checks: (1) the derived challenges replay exactly from the transcript with hashlib (the verifier's side);
(2) with those challenges the transcript, finals, A and B equal the oracle's; (3) the oracle verifier accepts,
and a tampered round polynomial changes every later challenge (so a replayed transcript no longer matches)."""
import hashlib
import random

import numpy as np
import pytest

from oracle import c_oracle as C
from oracle import tlookup as TL
from tests.fs_transcript import derive

pytestmark = pytest.mark.gpu
R = TL.R


@pytest.fixture(scope="module")
def ctx():
    from paper_2404_16109_b200 import zkl
    c = zkl.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("d,n", [(1, 0), (3, 2), (10, 8), (13, 5), (14, 14), (16, 10), (21, 10)])
@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
def test_fs_transcript(ctx, d, n, variant):
    """d >= 21: rounds with >= 2^20 elements derive H(1) from the running claim (k_fs_inv on the side stream)."""
    from paper_2404_16109_b200 import zkl
    rng = random.Random(d * 131 + n + variant)
    D, N = 1 << d, 1 << n
    T = [rng.randrange(R) for _ in range(N)]
    S = [T[rng.randrange(N)] for _ in range(D)]
    seed = hashlib.sha256(f"seed-{d}-{n}-{variant}".encode()).digest()
    ctx.reserve(D, N)
    Sv = ctx.import_canon(zkl.ints_to_canon(S))
    tab = ctx.table(ctx.import_canon(zkl.ints_to_canon(T)))
    m = ctx.prepare(Sv, D, tab)
    pf, der = ctx.prove_fs(Sv, D, tab, m, seed, variant, want_A=True, want_B=True)
    replay = derive(seed, D, N, variant, pf.evals)
    assert der == replay
    ref = C.prove(C.ints_to_limbs(S), C.ints_to_limbs(T),
                  C.chal_array(der["beta"], der["alpha1"], der["alpha2"], der["u"], der["r"]), variant)
    assert np.array_equal(m.cpu().numpy().astype(np.uint32), ref.m)
    assert ctx.export_ints(pf.A) == C.limbs_to_ints(ref.A)
    assert ctx.export_ints(pf.B) == C.limbs_to_ints(ref.B)
    assert pf.evals == ref.evals and pf.finals == ref.finals
    ch = TL.Challenges(der["beta"], der["alpha1"], der["alpha2"], der["u"], der["r"])
    assert TL.verify(TL.Transcript(pf.evals, pf.finals), D, N, ch, variant)
    if d >= 2:
        bad = [list(e) for e in pf.evals]
        bad[0][1] = (bad[0][1] + 1) % R
        assert derive(seed, D, N, variant, bad)["r"][1:] != der["r"][1:]


def test_fs_unprepared_falls_back(ctx):
    """An S that was not prepared, with one element outside T: the gather cannot apply, the inversion does."""
    from paper_2404_16109_b200 import zkl
    rng = random.Random(5)
    d, n = 13, 4
    D, N = 1 << d, 1 << n
    T = [rng.randrange(R) for _ in range(N)]
    S = [T[rng.randrange(N)] for _ in range(D)]
    ctx.reserve(D, N)
    tab = ctx.table(ctx.import_canon(zkl.ints_to_canon(T)))
    m = ctx.prepare(ctx.import_canon(zkl.ints_to_canon(S)), D, tab)
    bad = list(S)
    bad[100] = rng.randrange(R)
    seed = bytes(range(32))
    pf, der = ctx.prove_fs(ctx.import_canon(zkl.ints_to_canon(bad)), D, tab, m, seed, TL.PAPER, want_A=True)
    assert der == derive(seed, D, N, TL.PAPER, pf.evals)
    A = [pow((der["beta"] + s) % R, -1, R) for s in bad]
    B = [pow((der["beta"] + t) % R, -1, R) for t in T]
    assert ctx.export_ints(pf.A) == A
    ref = C.sumcheck(*(C.ints_to_limbs(v) for v in (A, bad, B, T)), m.cpu().numpy().astype(np.uint32),
                     C.chal_array(der["beta"], der["alpha1"], der["alpha2"], der["u"], der["r"]), TL.PAPER)
    assert pf.evals == ref.evals and pf.finals == ref.finals


@pytest.mark.parametrize("fs", [False, True])
def test_prepared_takes_gather_path(ctx, fs):
    """After prepare, prove / prove_fs gather A from the cached index keys in ONE pass: no D-side inversion
    kernels and no rerun (a workspace-layout mismatch between plans once made every key miss)."""
    from paper_2404_16109_b200 import zkl
    rng = random.Random(7 + fs)
    d, n = 15, 9
    D, N = 1 << d, 1 << n
    T = [rng.randrange(R) for _ in range(N)]
    S = [T[rng.randrange(N)] for _ in range(D)]
    ctx.reserve(D, N)
    Sv = ctx.import_canon(zkl.ints_to_canon(S))
    tab = ctx.table(ctx.import_canon(zkl.ints_to_canon(T)))
    m = ctx.prepare(Sv, D, tab)
    ctx.set_profiling(True)
    try:
        if fs:
            ctx.prove_fs(Sv, D, tab, m, bytes(32), TL.PAPER)
        else:
            u = [rng.randrange(R) for _ in range(d)]
            r = [rng.randrange(R) for _ in range(d)]
            ctx.prove(Sv, D, tab, m, zkl.Context.challenges(5, 7, 49, u, r))
        names = [rec[0] for rec in ctx.profile_read()]
    finally:
        ctx.set_profiling(False)
    assert sum(n.startswith("(k_round1_keys<true") for n in names) == 1, names
    assert not any(nm.startswith(("k_inv_fwd", "k_inv_bwd")) for nm in names), names   # N < 4096: no tiled inversion


@pytest.mark.parametrize("fs", [False, True])
def test_prepared_then_rewritten_in_place(ctx, fs):
    """prepare(S), then S overwritten in place by S' (every element still in T, one moved to another entry): the
    cached keys no longer describe S'; the per-element check against T sends the proof through the inversion path, so the
    transcript is that of S' (with the m of S', which the caller passes)."""
    from paper_2404_16109_b200 import zkl
    rng = random.Random(23 + fs)
    d, n = 14, 7
    D, N = 1 << d, 1 << n
    T = [rng.randrange(R) for _ in range(N)]
    S = [T[rng.randrange(N)] for _ in range(D)]
    S2 = list(S)
    S2[4097] = T[(T.index(S[4097]) + 3) % N]
    ctx.reserve(D, N)
    Sv = ctx.import_canon(zkl.ints_to_canon(S))
    tab = ctx.table(ctx.import_canon(zkl.ints_to_canon(T)))
    ctx.prepare(Sv, D, tab)
    ctx.import_canon(zkl.ints_to_canon(S2), dst=Sv)
    import torch
    m2 = torch.from_numpy(np.bincount([T.index(s) for s in S2], minlength=N).astype(np.int32)).to(ctx.device)
    if fs:
        seed = bytes(range(1, 33))
        pf, der = ctx.prove_fs(Sv, D, tab, m2, seed, TL.PAPER)
        ch = (der["beta"], der["alpha1"], der["alpha2"], der["u"], der["r"])
    else:
        ch = (rng.randrange(R), rng.randrange(R), rng.randrange(R), [rng.randrange(R) for _ in range(d)],
              [rng.randrange(R) for _ in range(d)])
        pf = ctx.prove(Sv, D, tab, m2, zkl.Context.challenges(*ch))
    ref = C.prove(C.ints_to_limbs(S2), C.ints_to_limbs(T), C.chal_array(*ch), TL.PAPER)
    assert pf.evals == ref.evals and pf.finals == ref.finals
