"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck; one tool per gpurun call, VERDICT r01
item 9): every kernel family of the tlookup path at sizes the tools finish in minutes, each transcript checked
against the CPU oracle so a run that exits 0 also computed the right thing.

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py
    python tools/sanitize_cases.py --check      # the same cases on libzkl_check.so (device bounds asserts)

Cases: C1 (D = 2^10 range check, one-CTA prove, both variants), a 2^14 random-table proof (inversion hierarchy,
hash index), a 2^19 function lookup with a virtual S (pair-range prepare, histogram, round-1 gather, round-2
gather, k_round, cooperative chunked rounds, tail), the async mode (background histogram) and Fiat-Shamir (the
cooperative Fiat-Shamir rounds kernel), and a 2-rank loopback proof.
"""
import os
import random
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if "--check" in sys.argv:   # compute-sanitizer is closed on this pool: device asserts on every access instead
    os.environ["ZKL_LIB"] = os.path.join(ROOT, "paper_2404_16109_b200", "libzkl_check.so")

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from oracle import c_oracle as C  # noqa: E402
from oracle import tlookup as TL  # noqa: E402
from paper_2404_16109_b200 import zkl  # noqa: E402


def chal_gpu(ch):
    return zkl.Context.challenges(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)


def main(small=False):
    ctx = zkl.Context(0)
    # C1
    wl = W.range_check()
    S, T = C.inputs_from_workload(wl)
    ch = TL.challenges_from(wl.chal)
    for variant in (TL.PAPER, TL.LOGUP):
        ref = C.prove(S, T, C.chal_array(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r), variant)
        ctx.reserve(wl.D, wl.N)
        Sv = ctx.import_ints(np.asarray(wl.s, dtype=np.int64))
        tab = ctx.table(ctx.import_ints(np.asarray(wl.t, dtype=np.int64)))
        m = ctx.prepare(Sv, wl.D, tab)
        pf = ctx.prove(Sv, wl.D, tab, m, chal_gpu(ch), variant, want_A=True, want_B=True)
        assert pf.evals == ref.evals and pf.finals == ref.finals, "C1"
    # 2^14 random table (hash index, inversion hierarchy through the tampered-S fallback is in the tests)
    rng = random.Random(7)
    d, n = 14, 8
    R = TL.R
    Tl = [rng.randrange(R) for _ in range(1 << n)]
    Sl = [Tl[rng.randrange(1 << n)] for _ in range(1 << d)]
    chk = TL.Challenges(rng.randrange(R), rng.randrange(R), 0, [rng.randrange(R) for _ in range(d)],
                        [rng.randrange(R) for _ in range(d)])
    chk.alpha2 = chk.alpha1 ** 2 % R
    ref = C.prove(C.ints_to_limbs(Sl), C.ints_to_limbs(Tl), C.chal_array(chk.beta, chk.alpha1, chk.alpha2, chk.u,
                                                                         chk.r), TL.LOGUP)
    ctx.reserve(1 << d, 1 << n)
    Sv = ctx.import_canon(zkl.ints_to_canon(Sl))
    tab = ctx.table(ctx.import_canon(zkl.ints_to_canon(Tl)))
    m = ctx.prepare(Sv, 1 << d, tab)
    pf = ctx.prove(Sv, 1 << d, tab, m, chal_gpu(chk), TL.LOGUP)
    assert pf.evals == ref.evals and pf.finals == ref.finals, "2^14"
    # function lookup, virtual S; explicit (sync and async) and Fiat-Shamir
    d = 17 if small else 19
    wl = W.activation("H", D=1 << d)
    chl = TL.challenges_from(wl.chal)
    chal = C.chal_array(chl.beta, chl.alpha1, chl.alpha2, chl.u, chl.r)
    ref = C.prove_pair_stream(wl.x, wl.y, wl.tx, wl.ty, wl.chal.alpha_f, chal, TL.PAPER, 2)
    ctx.reserve(wl.D, wl.N)
    tab = ctx.table(ctx.import_pair(wl.tx, wl.ty, wl.chal.alpha_f))
    assert ctx.table_attach_pair(tab, wl.tx, wl.ty, wl.chal.alpha_f)
    for use_async in (False, True):
        if use_async:
            ctx.set_async(True)
        _, m = ctx.prepare_pair(wl.x, wl.y, wl.chal.alpha_f, wl.D, tab, virtual_s=True)
        pf = ctx.prove(None, wl.D, tab, m, chal_gpu(chl), TL.PAPER)
        if use_async:
            ctx.wait()
            ctx.set_async(False)
            pf = pf.result()
        assert pf.evals == ref.evals and pf.finals == ref.finals, f"virtual S (async={use_async})"
    _, m = ctx.prepare_pair(wl.x, wl.y, wl.chal.alpha_f, wl.D, tab, virtual_s=True)
    fpf, der = ctx.prove_fs(None, wl.D, tab, m, bytes(range(32)), TL.PAPER)
    o = C.prove_pair_stream(wl.x, wl.y, wl.tx, wl.ty, wl.chal.alpha_f,
                            C.chal_array(der["beta"], der["alpha1"], der["alpha2"], der["u"], der["r"]), TL.PAPER, 2)
    assert fpf.evals == o.evals and fpf.finals == o.finals, "Fiat-Shamir"
    ctx.close()
    # two loopback ranks
    import torch
    P, D = 2, 1 << 17
    wl = W.activation("H", D=D)
    chl = TL.challenges_from(wl.chal)
    ref = C.prove_pair_stream(wl.x, wl.y, wl.tx, wl.ty, wl.chal.alpha_f,
                              C.chal_array(chl.beta, chl.alpha1, chl.alpha2, chl.u, chl.r), TL.PAPER, 2)
    group = zkl.LoopbackGroup(P, max_D_local=D // P, max_N=wl.N)
    out = [None] * P

    def rank(p):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            c = zkl.Context(0, stream=st, rank=p, group=group)
            c.reserve(D // P, wl.N)
            tb = c.table(c.import_pair(wl.tx, wl.ty, wl.chal.alpha_f))
            _, mm = c.prepare_pair(wl.x[p * D // P:(p + 1) * D // P], wl.y[p * D // P:(p + 1) * D // P],
                                   wl.chal.alpha_f, D, tb, virtual_s=True)
            out[p] = c.prove(None, D, tb, mm, chal_gpu(chl), TL.PAPER)
            c.close()

    th = [threading.Thread(target=rank, args=(p,)) for p in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    group.close()
    for pf in out:
        assert pf.evals == ref.evals and pf.finals == ref.finals, "loopback"
    print("sanitize cases ok")


if __name__ == "__main__":
    main(small="--small" in sys.argv)
