"""Proofs in flight from several host threads (the bench's mode): each thread drives its own context
and stream through the whole step (import T, table, pair-range attach, async prepare with a virtual S, prove, wait)
on its own workload, concurrently and repeatedly; every transcript is compared element by element with the CPU
oracle (the C tier).  Guards the library against state shared between contexts (staging, error words, the
histogram's workspace) and the host threads against each other."""
import threading

import numpy as np
import pytest

import workloads as W
from oracle import c_oracle as C
from oracle import tlookup as TL

pytestmark = pytest.mark.gpu


def _pair_workload(d, n, seed):
    rng = np.random.default_rng(seed)
    D, N = 1 << d, 1 << n
    tx = (np.arange(N) - N // 2).astype(np.int32)
    ty = rng.integers(-2 ** 31, 2 ** 31, N, dtype=np.int64).astype(np.int32)
    pick = np.clip(np.rint(N / 2 + rng.normal(0, N / 8, D)), 0, N - 1).astype(np.int64)
    pick[: D // 4] = rng.integers(0, N, D // 4)
    return tx[pick], ty[pick], tx, ty, W.challenges(f"inflight{d}.{n}.{seed}", d)


@pytest.mark.parametrize("lanes,d,n,variant", [(2, 18, 16, TL.PAPER), (3, 16, 12, TL.LOGUP)])
def test_lanes_in_flight_match_oracle(lanes, d, n, variant):
    import torch
    from paper_2404_16109_b200 import zkl
    dev = torch.device("cuda", 0)
    D, N = 1 << d, 1 << n
    work = [_pair_workload(d, n, 100 * lanes + i) for i in range(lanes)]
    refs = []
    for x, y, tx, ty, ch in work:
        chal = C.chal_array(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)
        refs.append(C.prove_pair_stream(x, y, tx, ty, ch.alpha_f, chal, variant, 2))
    ctxs, inputs = [], []
    for x, y, tx, ty, ch in work:
        st = torch.cuda.Stream(device=dev)
        c = zkl.Context(0, stream=st)
        c.reserve(D, N)
        ctxs.append((c, st))
        inputs.append(tuple(torch.from_numpy(a).to(dev) for a in (x, y, tx, ty)))
    torch.cuda.synchronize()
    errors, results = [], [[] for _ in range(lanes)]

    def run(i):
        c, st = ctxs[i]
        xd, yd, txd, tyd = inputs[i]
        ch = work[i][4]
        chal = zkl.Context.challenges(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)
        T, tmem = c.vec(N), c.table_mem(N)
        m = torch.empty(N, dtype=torch.int32, device=dev)
        try:
            with torch.cuda.stream(st):
                for _ in range(3):
                    c.import_pair(txd, tyd, ch.alpha_f, T)
                    tab = c.table(T, tmem)
                    assert c.table_attach_pair(tab, txd, tyd, ch.alpha_f)
                    c.set_async(True)
                    c.prepare_pair(xd, yd, ch.alpha_f, D, tab, m=m, virtual_s=True)
                    pend = c.prove(None, D, tab, m, chal, variant)
                    c.wait()
                    c.set_async(False)
                    pf = pend.result()
                    results[i].append((pf.evals, pf.finals, m.cpu().numpy().astype(np.uint32)))
        except Exception as e:   # noqa: BLE001 -- reported below with the lane
            errors.append((i, repr(e)))

    th = [threading.Thread(target=run, args=(i,)) for i in range(lanes)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for c, _ in ctxs:
        c.close()
    assert not errors, errors
    for i in range(lanes):
        assert len(results[i]) == 3
        for evals, finals, m in results[i]:
            assert evals == refs[i].evals and finals == refs[i].finals
            assert np.array_equal(m, refs[i].m)
