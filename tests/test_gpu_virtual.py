"""Virtual S: prepare_pair without S_local_out keeps only the table
keys, round 1 gathers A_i = B_key and S_i = T_key from the (B, T) records and round 2 gathers them again, so S and
A never cross HBM.  Every transcript here is compared element by element with the CPU oracle (the C tier; the bench
workload H against the stored golden written by tools/make_goldens.py from oracle/ only).

Sizes cover each branch of the host logic: D_local < 4096 (one-CTA prove, S materialised from the keys),
4096 <= D_local <= 2^18 (chunked rounds from round 2, S materialised), D_local > 2^18 (round-2 gather), plus the
async mode with the background histogram, Fiat-Shamir, both variants, A requested or not, and the errors.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import workloads as W
from oracle import c_oracle as C
from oracle import tlookup as TL

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ctx():
    from paper_2404_16109_b200 import zkl
    c = zkl.Context(0)
    yield c
    c.close()


def _chal(ch):
    from paper_2404_16109_b200 import zkl
    return zkl.Context.challenges(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)


def _pair_workload(d, n, seed):
    rng = np.random.default_rng(seed)
    D, N = 1 << d, 1 << n
    tx = (np.arange(N) - N // 2).astype(np.int32)
    ty = rng.integers(-2 ** 31, 2 ** 31, N, dtype=np.int64).astype(np.int32)
    # activation-like: a peaked index distribution plus a uniform part, so some keys repeat and some never occur
    pick = np.clip(np.rint(N / 2 + rng.normal(0, N / 8, D)), 0, N - 1).astype(np.int64)
    pick[: D // 4] = rng.integers(0, N, D // 4)
    x, y = tx[pick], ty[pick]
    ch = W.challenges(f"virt{d}.{n}.{seed}", d)
    return x, y, tx, ty, ch


@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
@pytest.mark.parametrize("d,n,want_A,use_async", [(10, 8, True, False), (12, 8, False, True), (12, 12, True, False),
                                                   (16, 10, False, False), (19, 16, False, True),
                                                   (20, 12, True, False), (21, 16, False, True)])
def test_virtual_s_matches_oracle(ctx, d, n, want_A, use_async, variant):
    x, y, tx, ty, ch = _pair_workload(d, n, d * 7 + n)
    D, N = 1 << d, 1 << n
    chal = C.chal_array(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)
    ref = C.prove_pair_stream(x, y, tx, ty, ch.alpha_f, chal, variant, min(d, 2))
    ctx.reserve(D, N)
    tab = ctx.table(ctx.import_pair(tx, ty, ch.alpha_f))
    assert ctx.table_attach_pair(tab, tx, ty, ch.alpha_f)
    if use_async:
        ctx.set_async(True)
    S, m = ctx.prepare_pair(x, y, ch.alpha_f, D, tab, virtual_s=True)
    assert S is None
    pf = ctx.prove(None, D, tab, m, _chal(ch), variant, want_A=want_A, want_B=True)
    if use_async:
        ctx.wait()
        ctx.set_async(False)
        pf = pf.result()
    assert np.array_equal(m.cpu().numpy().astype(np.uint32), ref.m)
    assert pf.evals == ref.evals
    assert pf.finals == ref.finals
    assert ctx.export_ints(pf.B) == C.limbs_to_ints(ref.B)
    if want_A:
        A = ctx.export_ints(pf.A)
        af = ch.alpha_f % TL.R
        idx = np.random.default_rng(d).choice(D, 256, replace=False)
        for i in idx:
            s = (int(x[i]) + af * int(y[i])) % TL.R
            assert A[i] * (s + ch.beta) % TL.R == 1


def test_virtual_s_fiat_shamir_equals_materialised(ctx):
    """prove_fs on a virtual S: the same transcript and derived challenges as on the materialised S."""
    d, n = 19, 16
    x, y, tx, ty, ch = _pair_workload(d, n, 5)
    D, N = 1 << d, 1 << n
    ctx.reserve(D, N)
    tab = ctx.table(ctx.import_pair(tx, ty, ch.alpha_f))
    assert ctx.table_attach_pair(tab, tx, ty, ch.alpha_f)
    seed = hashlib.sha256(b"virtual-fs").digest()
    S, m = ctx.prepare_pair(x, y, ch.alpha_f, D, tab)
    ref, dref = ctx.prove_fs(S, D, tab, m, seed, TL.PAPER)
    _, m2 = ctx.prepare_pair(x, y, ch.alpha_f, D, tab, virtual_s=True)
    got, dgot = ctx.prove_fs(None, D, tab, m2, seed, TL.PAPER)
    assert dgot == dref
    assert got.evals == ref.evals and got.finals == ref.finals
    # and the oracle, on the challenges the device derived
    chal = C.chal_array(dref["beta"], dref["alpha1"], dref["alpha2"], dref["u"], dref["r"])
    o = C.prove_pair_stream(x, y, tx, ty, ch.alpha_f, chal, TL.PAPER, 2)
    assert got.evals == o.evals and got.finals == o.finals


def test_virtual_s_needs_its_prepare(ctx):
    from paper_2404_16109_b200 import zkl
    d, n = 14, 8
    x, y, tx, ty, ch = _pair_workload(d, n, 9)
    D, N = 1 << d, 1 << n
    ctx.reserve(D, N)
    tab = ctx.table(ctx.import_pair(tx, ty, ch.alpha_f))
    S, m = ctx.prepare_pair(x, y, ch.alpha_f, D, tab)          # materialised: no virtual S to prove on
    with pytest.raises(zkl.ZklError) as e:
        ctx.prove(None, D, tab, m, _chal(ch), TL.PAPER)
    assert e.value.name == "ZKL_E_ARG"
    tab2 = ctx.table(ctx.import_pair(tx, ty, ch.alpha_f))
    _, m = ctx.prepare_pair(x, y, ch.alpha_f, D, tab, virtual_s=True)
    with pytest.raises(zkl.ZklError) as e:                      # another table than the prepared one
        ctx.prove(None, D, tab2, m, _chal(ch), TL.PAPER)
    assert e.value.name == "ZKL_E_ARG"


def _golden(cfg):
    path = os.path.join(ROOT, "tests", "golden", f"full_{cfg}.json")
    with open(path) as f:
        return json.load(f)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_bench_step_at_H_matches_golden():
    """bench.py's exact step at H (D = 2^26, SiLU table): import T, table + pair-range attachment, async
    prepare_pair with a virtual S and the background histogram, prove on the virtual S, wait -- compared with the
    golden the CPU oracle wrote (tests/golden/full_H.json): m, B, all 26 x 4 evaluations and the 5 finals."""
    import torch
    from paper_2404_16109_b200 import zkl
    g = _golden("H")
    wl = W.activation("H")
    assert _sha(wl.x.astype("<i4")) == g["inputs_sha256"]["x"] and _sha(wl.y.astype("<i4")) == g["inputs_sha256"]["y"]
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    ctx = zkl.Context(0, stream=stream)
    try:
        D, N = wl.D, wl.N
        ctx.reserve(D, N)
        xd, yd = torch.from_numpy(wl.x).to(dev), torch.from_numpy(wl.y).to(dev)
        txd, tyd = torch.from_numpy(wl.tx).to(dev), torch.from_numpy(wl.ty).to(dev)
        T = ctx.vec(N)
        tmem = ctx.table_mem(N)
        m = torch.empty(N, dtype=torch.int32, device=dev)
        ch = wl.chal
        chal = zkl.Context.challenges(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)
        for _ in range(2):   # twice: the second step reuses the workspace, table memory and m of the first
            ctx.import_pair(txd, tyd, ch.alpha_f, T)
            tab = ctx.table(T, tmem)
            assert ctx.table_attach_pair(tab, txd, tyd, ch.alpha_f)
            ctx.set_async(True)
            ctx.prepare_pair(xd, yd, ch.alpha_f, D, tab, m=m, virtual_s=True)
            pend = ctx.prove(None, D, tab, m, chal, TL.PAPER, want_B=True)
            ctx.wait()
            ctx.set_async(False)
            pf = pend.result()
            assert _sha(m.cpu().numpy().astype("<u4")) == g["m_sha256"]
            B = np.asarray(C.ints_to_limbs(ctx.export_ints(pf.B)), dtype="<u8")
            assert _sha(B) == g["B_sha256"]
            assert [[hex(v) for v in e] for e in pf.evals] == g["evals"]
            assert {k: hex(v) for k, v in pf.finals.items()} == g["finals"]
    finally:
        ctx.close()
        torch.cuda.set_stream(torch.cuda.default_stream(dev))


@pytest.mark.parametrize("d,n", [(12, 8), (20, 16)])
def test_prove_pair_host_matches_oracle(ctx, d, n):
    """The end-to-end entry point from host buffers (zkl_tlookup_prove_pair_host) against the oracle."""
    x, y, tx, ty, ch = _pair_workload(d, n, 31 + d)
    D, N = 1 << d, 1 << n
    chal = C.chal_array(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)
    ref = C.prove_pair_stream(x, y, tx, ty, ch.alpha_f, chal, TL.PAPER, 2)
    ctx.reserve(D, N)
    pf, m = ctx.prove_pair_host(x, y, tx, ty, ch.alpha_f, D, _chal(ch), TL.PAPER, want_m=True)
    assert np.array_equal(m, ref.m)
    assert pf.evals == ref.evals and pf.finals == ref.finals


@pytest.mark.parametrize("d,n", [(20, 8), (21, 16)])
def test_async_prepare_then_fiat_shamir(ctx, d, n):
    """The bench's Fiat-Shamir step: async prepare_pair (the histogram on the low-priority stream, its workspace
    beside the proof's) then prove_fs, at large D with a small and a full table: the transcript and derived
    challenges equal the synchronous run's, and the oracle's on those challenges."""
    x, y, tx, ty, ch = _pair_workload(d, n, 3 * d + n)
    D, N = 1 << d, 1 << n
    seed = hashlib.sha256(f"async-fs-{d}-{n}".encode()).digest()
    ctx.reserve(D, N)
    tab = ctx.table(ctx.import_pair(tx, ty, ch.alpha_f))
    assert ctx.table_attach_pair(tab, tx, ty, ch.alpha_f)
    _, m = ctx.prepare_pair(x, y, ch.alpha_f, D, tab, virtual_s=True)
    ref, dref = ctx.prove_fs(None, D, tab, m, seed, TL.PAPER)
    ctx.set_async(True)
    _, m2 = ctx.prepare_pair(x, y, ch.alpha_f, D, tab, virtual_s=True)
    res = ctx.prove_fs(None, D, tab, m2, seed, TL.PAPER)
    ctx.wait()
    ctx.set_async(False)
    got, dgot = res.result()
    assert dgot == dref and got.evals == ref.evals and got.finals == ref.finals
    chal = C.chal_array(dref["beta"], dref["alpha1"], dref["alpha2"], dref["u"], dref["r"])
    o = C.prove_pair_stream(x, y, tx, ty, ch.alpha_f, chal, TL.PAPER, 2)
    assert ref.evals == o.evals and ref.finals == o.finals
