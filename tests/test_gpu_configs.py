"""Parity at the BASELINE.json configurations' full sizes, in the launch configuration bench.py times.

Every configuration is compared element by element with a golden the CPU oracle wrote ahead of time
(tools/make_goldens.py, which imports only oracle/ and workloads/: the streaming C tier zko_tlookup_pair_stream).
A golden holds the SHA-256 of the generated inputs (checked first, so generator drift cannot pass), the digests of
m and B, all log2(D) x 4 round evaluations and the five finals.

H (2^26, materialised S; the bench's virtual-S step is in test_gpu_virtual.py), C3 (2^25 padded, LOGUP),
C4 (the K = 5 zkAttn digit instances at the full 32 heads x 2048 x 2048 = 2^27 each), C5 (2^30, virtual S).
A is sampled against A_i (beta + S_i) = 1 where it is materialised.
"""
import hashlib
import json
import os
import random

import numpy as np
import pytest

import workloads as W
from oracle import c_oracle as C
from oracle import tlookup as TL

pytestmark = pytest.mark.gpu
R = TL.R
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _golden(cfg):
    with open(os.path.join(ROOT, "tests", "golden", f"full_{cfg}.json")) as f:
        return json.load(f)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _assert_golden(g, m, pf, ctx):
    assert _sha(np.asarray(m, dtype="<u4")) == g["m_sha256"], "m"
    if pf.B is not None:
        B = np.asarray(C.ints_to_limbs(ctx.export_ints(pf.B)), dtype="<u8")
        assert _sha(B) == g["B_sha256"], "B"
    assert [[hex(v) for v in e] for e in pf.evals] == g["evals"], "round evaluations"
    assert {k: hex(v) for k, v in pf.finals.items()} == g["finals"], "finals"


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


def _check_against_golden(cfg, wl, variant, n_sample=512):
    """Materialised S through zkl_vec_import_* + zkl_tlookup_prepare + zkl_tlookup_prove, against the golden."""
    ctx, zkl = _gpu()
    g = _golden(cfg)
    assert g["variant"] == ("paper" if variant == TL.PAPER else "logup")
    if wl.kind == "pair":
        assert _sha(wl.x.astype("<i4")) == g["inputs_sha256"]["x"] and _sha(wl.y.astype("<i4")) == g["inputs_sha256"]["y"]
    else:
        assert _sha(wl.s.astype("<i4")) == g["inputs_sha256"]["x"]
    ch = TL.challenges_from(wl.chal)
    ctx.reserve(wl.D, wl.N)
    if wl.kind == "pair":
        Sv = ctx.import_pair(wl.x, wl.y, wl.chal.alpha_f)
        Tv = ctx.import_pair(wl.tx, wl.ty, wl.chal.alpha_f)
    else:
        Sv = ctx.import_ints(np.asarray(wl.s, dtype=np.int64))
        Tv = ctx.import_ints(np.asarray(wl.t, dtype=np.int64))
    tab = ctx.table(Tv)
    m = ctx.prepare(Sv, wl.D, tab)
    pf = ctx.prove(Sv, wl.D, tab, m, zkl.Context.challenges(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r), variant,
                   want_A=True, want_B=True)
    _assert_golden(g, m.cpu().numpy().astype(np.uint32), pf, ctx)
    rng = random.Random(wl.D)
    idx = sorted(rng.sample(range(wl.D), n_sample))
    got = _sample_A(ctx, zkl, pf.A, idx)
    if wl.kind == "pair":
        af = wl.chal.alpha_f % R
        Sints = [(int(wl.x[i]) + af * int(wl.y[i])) % R for i in idx]
    else:
        Sints = [int(wl.s[i]) % R for i in idx]
    for a, sv in zip(got, Sints):
        assert a * (sv + ch.beta) % R == 1


def _check_virtual_against_golden(cfg, wl, variant):
    """Function lookup through the bench path: pair-range table, prepare_pair with a virtual S, prove."""
    ctx, zkl = _gpu()
    g = _golden(cfg)
    assert _sha(wl.x.astype("<i4")) == g["inputs_sha256"]["x"] and _sha(wl.y.astype("<i4")) == g["inputs_sha256"]["y"]
    ch = TL.challenges_from(wl.chal)
    ctx.reserve(wl.D, wl.N)
    tab = ctx.table(ctx.import_pair(wl.tx, wl.ty, wl.chal.alpha_f))
    assert ctx.table_attach_pair(tab, wl.tx, wl.ty, wl.chal.alpha_f)
    _, m = ctx.prepare_pair(wl.x, wl.y, wl.chal.alpha_f, wl.D, tab, virtual_s=True)
    pf = ctx.prove(None, wl.D, tab, m, zkl.Context.challenges(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r), variant,
                   want_B=True)
    _assert_golden(g, m.cpu().numpy().astype(np.uint32), pf, ctx)


def test_h_full_transcript():
    """H: the bench workload (2^26 SiLU lookups into N = 2^16), materialised S, A sampled."""
    _check_against_golden("H", W.activation("H"), TL.PAPER)


def test_c3_padded_full_transcript():
    wl = W.activation("3")
    assert wl.D == 1 << 25 and wl.meta["real"] == 2048 * 11008
    _check_against_golden("3", wl, TL.LOGUP)


@pytest.mark.parametrize("k", [0, 1, 2, 3, 4])
def test_c4_zkattn_digit_instances_full(k):
    """C4 at the full 32 heads x 2048 x 2048 = 2^27 per instance: range instances (k <= 2) with a materialised S,
    function instances (k = 3, 4) through the virtual-S bench path."""
    wl = W.zkattn_digits(k, heads=32)
    if wl.kind == "int":
        _check_against_golden(f"4.{k}", wl, TL.PAPER, n_sample=128)
    else:
        _check_virtual_against_golden(f"4.{k}", wl, TL.PAPER)


def test_c5_full_transcript_2p30():
    """C5 (2^30 SiLU lookups on one B200) through the bench path (virtual S), against the oracle's golden."""
    import torch
    ctx, zkl = _gpu()
    g = _golden("5")
    D, N = 1 << 30, 1 << 16
    tx, ty = W.activation_table("silu")
    ch = W.challenges("5", 30)
    dev = torch.device("cuda", 0)
    xd = torch.empty(D, dtype=torch.int32, device=dev)
    yd = torch.empty(D, dtype=torch.int32, device=dev)
    hx, hy = hashlib.sha256(), hashlib.sha256()
    chunk = 1 << 26
    for start in range(0, D, chunk):
        x = W.activation_x("5", start, chunk, D)
        y = ty[x.astype(np.int64) + 32768].astype(np.int32)
        hx.update(x.astype("<i4").tobytes())
        hy.update(y.astype("<i4").tobytes())
        xd[start:start + chunk] = torch.from_numpy(x).to(dev)
        yd[start:start + chunk] = torch.from_numpy(y).to(dev)
    assert hx.hexdigest() == g["inputs_sha256"]["x"] and hy.hexdigest() == g["inputs_sha256"]["y"]
    ctx.reserve(D, N)
    tab = ctx.table(ctx.import_pair(tx.astype(np.int32), ty.astype(np.int32), ch.alpha_f))
    assert ctx.table_attach_pair(tab, tx.astype(np.int32), ty.astype(np.int32), ch.alpha_f)
    _, m = ctx.prepare_pair(xd, yd, ch.alpha_f, D, tab, virtual_s=True)
    chl = TL.challenges_from(ch)
    pf = ctx.prove(None, D, tab, m, zkl.Context.challenges(chl.beta, chl.alpha1, chl.alpha2, chl.u, chl.r), TL.PAPER,
                   want_B=True)
    _assert_golden(g, m.cpu().numpy().astype(np.uint32), pf, ctx)
    assert TL.verify(TL.Transcript(pf.evals, pf.finals), D, N, chl, TL.PAPER)
    del xd, yd
    torch.cuda.empty_cache()


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
