"""Parity at the BASELINE.json configurations' sizes, in the launch configuration bench.py times.

H (2^26) and C3 (2^25, padded) : full transcript, m and B vs the C oracle; A sampled vs pow(x, -1, r).
C2 is in test_gpu_parity.py (full A as well).  C4 : the K = 5 zkAttn digit instances (2 heads = 2^23 each).
C5 (2^30) : the oracle cannot reach it in test time, so properties that hold at any size are checked:
exact m against an independent integer bincount of X, sampled A_i (beta + S_i) = 1, the verifier accepting
the transcript (round consistency and g_d(r_d) = f(v) from the finals), and a tampered evaluation rejected.
"""
import random

import numpy as np
import pytest

import workloads as W
from oracle import c_oracle as C
from oracle import tlookup as TL

pytestmark = pytest.mark.gpu
R = TL.R


def _gpu(ctx_holder={}):
    from paper_2404_16109_b200 import zkl
    if "ctx" not in ctx_holder:
        ctx_holder["ctx"] = zkl.Context(0)
    return ctx_holder["ctx"], zkl


def _sample_A(ctx, zkl, Av, idx):
    import torch
    planes = Av.data.view(8, Av.n)
    sel = torch.as_tensor(np.asarray(idx, dtype=np.int64), device=planes.device)
    sub = planes.index_select(1, sel).contiguous()
    return ctx.export_ints(zkl.Vec(sub.view(-1), len(idx)))


def _check_against_c_oracle(wl, variant=TL.PAPER, n_sample=512):
    ctx, zkl = _gpu()
    S, T = C.inputs_from_workload(wl)
    ch = TL.challenges_from(wl.chal)
    ref = C.prove(S, T, C.chal_array(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r), variant, want_A=False)
    ctx.reserve(wl.D, wl.N)
    if wl.kind == "pair":
        Sv = ctx.import_pair(wl.x, wl.y, wl.chal.alpha_f)
        Tv = ctx.import_pair(wl.tx, wl.ty, wl.chal.alpha_f)
    else:
        Sv = ctx.import_ints(np.asarray(wl.s, dtype=np.int64))
        Tv = ctx.import_ints(np.asarray(wl.t, dtype=np.int64))
    tab = ctx.table(Tv)
    m = ctx.prepare(Sv, wl.D, tab)
    assert np.array_equal(m.cpu().numpy().astype(np.uint32), ref.m)
    pf = ctx.prove(Sv, wl.D, tab, m, zkl.Context.challenges(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r), variant,
                   want_A=True, want_B=True)
    assert pf.evals == ref.evals
    assert pf.finals == ref.finals
    assert ctx.export_ints(pf.B) == C.limbs_to_ints(ref.B)
    rng = random.Random(wl.D)
    idx = sorted(rng.sample(range(wl.D), n_sample))
    got = _sample_A(ctx, zkl, pf.A, idx)
    Sints = C.limbs_to_ints(S[idx])
    for a, s in zip(got, Sints):
        assert a * (s + ch.beta) % R == 1


def test_h_full_transcript():
    """H: the bench workload itself (2^26 SiLU lookups into N = 2^16)."""
    _check_against_c_oracle(W.activation("H"))


def test_c3_padded_full_transcript():
    wl = W.activation("3")
    assert wl.D == 1 << 25 and wl.meta["real"] == 2048 * 11008
    _check_against_c_oracle(wl, TL.LOGUP)


@pytest.mark.parametrize("k", [0, 1, 2, 3, 4])
def test_c4_zkattn_digit_instances(k):
    _check_against_c_oracle(W.zkattn_digits(k, heads=2), TL.PAPER, n_sample=128)


def test_c5_properties_full_size():
    import torch
    ctx, zkl = _gpu()
    D, N = 1 << 30, 1 << 16
    real = D
    tx, ty = W.activation_table("silu")
    ch = W.challenges("5", 30)
    dev = torch.device("cuda", 0)
    xd = torch.empty(D, dtype=torch.int32, device=dev)
    yd = torch.empty(D, dtype=torch.int32, device=dev)
    counts = np.zeros(N, dtype=np.int64)
    chunk = 1 << 26
    for start in range(0, D, chunk):
        x = W.activation_x("5", start, chunk, real)
        counts += np.bincount(x.astype(np.int64) + 32768, minlength=N)
        xd[start:start + chunk] = torch.from_numpy(x).to(dev)
        yd[start:start + chunk] = torch.from_numpy(ty[x.astype(np.int64) + 32768].astype(np.int32)).to(dev)
    rng = random.Random(5)
    idx = sorted(rng.sample(range(D), 256))
    xs = xd[idx].cpu().numpy()
    ys = yd[idx].cpu().numpy()
    Sv = ctx.vec(D)
    ctx.import_pair(xd, yd, ch.alpha_f, Sv)
    del xd, yd
    torch.cuda.empty_cache()
    ctx.reserve(D, N)
    Tv = ctx.import_pair(tx.astype(np.int32), ty.astype(np.int32), ch.alpha_f)
    tab = ctx.table(Tv)
    m = ctx.prepare(Sv, D, tab).cpu().numpy().astype(np.int64)
    assert np.array_equal(m, counts)
    chl = TL.challenges_from(ch)
    pf = ctx.prove(Sv, D, tab, torch.as_tensor(m.astype(np.int32), device=dev),
                   zkl.Context.challenges(chl.beta, chl.alpha1, chl.alpha2, chl.u, chl.r), TL.PAPER, want_A=True)
    assert TL.verify(TL.Transcript(pf.evals, pf.finals), D, N, chl, TL.PAPER)
    bad = TL.Transcript([list(e) for e in pf.evals], dict(pf.finals))
    bad.evals[17][2] = (bad.evals[17][2] + 1) % R
    assert not TL.verify(bad, D, N, chl, TL.PAPER)
    # sampled A_i (beta + S_i) = 1 with S_i recomputed independently from X_i, Y_i
    got = _sample_A(ctx, zkl, pf.A, idx)
    af = ch.alpha_f % R
    for a, x, y in zip(got, xs, ys):
        s = (int(x) + af * int(y)) % R
        assert a * (s + chl.beta) % R == 1
    # table finals: T(v') and m(v') against the MLE of the (N-sized) table vectors
    from oracle.mle import mle_eval
    d = 30
    v = [chl.r[d - c - 1] for c in range(d)]
    vt = v[d - 16:]
    T_ints = [(int(a) + af * int(b)) % R for a, b in zip(tx, ty)]
    assert pf.finals["T"] == mle_eval(T_ints, vt)
    assert pf.finals["m"] == mle_eval([int(c) for c in m], vt)
