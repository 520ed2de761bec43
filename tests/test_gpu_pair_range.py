"""Function-lookup fast path of the fused prepare (a3): a table attached as a pair range
(T_j = tx_j + alpha ty_j, tx_j = tx_0 + j) indexes (x, y) as j = x - tx_0, checked by ty_j == y, instead of hashing.

S, m, the cached keys (through the transcript of the following prove) must be exactly those of the hash path and
the oracle; a pair off the function's graph or outside the range falls back to the hash path inside the same call
and reports NOT_IN_TABLE with the smallest index; a table that is not a range refuses the attachment and keeps
working; the fast kernel is the one that runs when it applies."""
import numpy as np
import pytest

import workloads as W
from oracle import c_oracle as C
from oracle import tlookup as TL

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2404_16109_b200 import zkl
    c = zkl.Context(0)
    yield c
    c.close()


def _chal(ch):
    from paper_2404_16109_b200 import zkl
    return zkl.Context.challenges(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)


@pytest.mark.parametrize("variant", [TL.PAPER, TL.LOGUP])
def test_range_path_matches_oracle(ctx, variant):
    wl = W.activation("2")   # C2: GELU, D = 2^20, N = 2^16, tx = [-2^15, 2^15)
    S, T = C.inputs_from_workload(wl)
    ch = TL.challenges_from(wl.chal)
    ref = C.prove(S, T, C.chal_array(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r), variant, want_A=False)
    ctx.reserve(wl.D, wl.N)
    tab = ctx.table(ctx.import_pair(wl.tx, wl.ty, wl.chal.alpha_f))
    assert ctx.table_attach_pair(tab, wl.tx, wl.ty, wl.chal.alpha_f)
    ctx.set_profiling(True)
    try:
        Sv, m = ctx.prepare_pair(wl.x, wl.y, wl.chal.alpha_f, wl.D, tab)
        names = [r[0] for r in ctx.profile_read()]
    finally:
        ctx.set_profiling(False)
    assert "k_import_pair_range" in names and "k_import_pair_index" not in names
    assert ctx.export_ints(Sv) == C.limbs_to_ints(S)
    assert np.array_equal(m.cpu().numpy().astype(np.uint32), ref.m)
    pf = ctx.prove(Sv, wl.D, tab, m, _chal(ch), variant)
    assert pf.evals == ref.evals and pf.finals == ref.finals


def test_range_path_misses_fall_back(ctx):
    from paper_2404_16109_b200 import zkl
    D, N = 1 << 14, 1 << 8
    ctx.reserve(D, N)
    tx = np.arange(N, dtype=np.int32) - 128
    ty = tx * 3 + 1
    tab = ctx.table(ctx.import_pair(tx, ty, 12345))
    assert ctx.table_attach_pair(tab, tx, ty, 12345)
    rng = np.random.default_rng(1)
    x = rng.integers(-128, 128, D).astype(np.int32)
    y = (x * 3 + 1).astype(np.int32)
    S, m = ctx.prepare_pair(x, y, 12345, D, tab)
    assert list(m.cpu().numpy()) == list(np.bincount(x.astype(np.int64) + 128, minlength=N))
    x2, y2 = x.copy(), y.copy()
    y2[9000] += 1             # off the graph
    x2[12000] = 500           # outside the range
    with pytest.raises(zkl.ZklError) as e:
        ctx.prepare_pair(x2, y2, 12345, D, tab)
    assert e.value.name == "ZKL_E_NOT_IN_TABLE" and e.value.index == 9000
    # a different alpha than the attached one: the hash path, same result
    tab2 = ctx.table(ctx.import_pair(tx, ty, 777))
    assert ctx.table_attach_pair(tab2, tx, ty, 777)
    S3, m3 = ctx.prepare_pair(x, y, 777, D, tab2)
    assert list(m3.cpu().numpy()) == list(m.cpu().numpy())


def test_attach_refuses_non_range(ctx):
    D, N = 1 << 13, 1 << 6
    ctx.reserve(D, N)
    tx = (np.arange(N, dtype=np.int32) * 2)          # stride 2: not a range
    ty = tx + 5
    tab = ctx.table(ctx.import_pair(tx, ty, 99))
    assert not ctx.table_attach_pair(tab, tx, ty, 99)
    tx2 = np.arange(N, dtype=np.int32)
    assert not ctx.table_attach_pair(tab, tx2, ty, 99)   # a range, but not the table's entries
    rng = np.random.default_rng(2)
    idx = rng.integers(0, N, D)
    S, m = ctx.prepare_pair(tx[idx], ty[idx], 99, D, tab)
    assert list(m.cpu().numpy()) == list(np.bincount(idx, minlength=N))
