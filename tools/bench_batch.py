"""Many-instance throughput: K tlookup instances (prepare_pair + prove) one after another on one
context (synchronous API) vs. in flight on M contexts / CUDA streams (async mode).

    python tools/bench_batch.py [log2D] [K] [M]      defaults 16 64 8

Workload H's SiLU table (N = 2^16); each instance has its own lookups (a permutation of H's inputs), its own
challenges and its own copy of the table (imported + indexed per instance, as a prover does per layer).
Inputs resident in HBM; CUDA events around the whole batch.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2404_16109_b200 import zkl  # noqa: E402


def main():
    log2d = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    M = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    D = 1 << log2d
    dev = torch.device("cuda", 0)
    base = W.activation("H", D=D)
    rng = np.random.default_rng(5)
    insts = []
    tx, ty = torch.from_numpy(base.tx).to(dev), torch.from_numpy(base.ty).to(dev)
    for k in range(K):
        # same table, different lookups (a permutation of the base inputs) and challenges per instance
        xk = np.ascontiguousarray(rng.permutation(base.x))
        ch = base.chal
        insts.append((torch.from_numpy(xk).to(dev), _paired(base, xk, dev), tx, ty,
                      zkl.Context.challenges(ch.beta + k, ch.alpha1, ch.alpha2, ch.u, ch.r)))
    ctxs = [zkl.Context(0, stream=torch.cuda.Stream()) for _ in range(M)]
    lanes = []
    for c in ctxs:
        c.reserve(D, base.N)
        with torch.cuda.stream(c.stream):
            lanes.append((c.vec(D), c.vec(base.N), c.table_mem(base.N),
                          torch.empty(base.N, dtype=torch.int32, device=dev)))

    def run_sync():
        c = ctxs[0]
        S, T, tmem, m = lanes[0]
        for x, y, tx, ty, ch in insts:
            c.import_pair(tx, ty, base.chal.alpha_f, T)
            tab = c.table(T, tmem)
            c.table_attach_pair(tab, tx, ty, base.chal.alpha_f)   # pair-range fast path of prepare_pair
            c.prepare_pair(x, y, base.chal.alpha_f, D, tab, S, m)
            c.prove(S, D, tab, m, ch)

    def run_async():
        for b in range(0, K, M):
            live = []
            for c, lane, (x, y, tx, ty, ch) in zip(ctxs, lanes, insts[b:b + M]):
                S, T, tmem, m = lane
                with torch.cuda.stream(c.stream):
                    c.import_pair(tx, ty, base.chal.alpha_f, T)
                    tab = c.table(T, tmem)
                    c.table_attach_pair(tab, tx, ty, base.chal.alpha_f)   # pair-range fast path of prepare_pair
                c.set_async(True)
                c.prepare_pair(x, y, base.chal.alpha_f, D, tab, S, m)
                live.append((c, c.prove(S, D, tab, m, ch)))
            for c, pf in live:
                c.wait()
                c.set_async(False)
                pf.result()

    out = {}
    for name, fn in (("sequential", run_sync), ("async", run_async)):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        out[name] = {"ms": ms, "lookups_per_s": K * D / (ms / 1e3)}
    print(json.dumps({"D": D, "K": K, "streams": M, **out,
                      "speedup": out["sequential"]["ms"] / out["async"]["ms"]}))


def _paired(base, x, dev):
    """y such that (x, y) is a row of the table: y = f(x) looked up through the table's x column."""
    order = np.argsort(base.tx)
    pos = np.searchsorted(base.tx[order], x)
    return torch.from_numpy(np.ascontiguousarray(base.ty[order][pos])).to(dev)


if __name__ == "__main__":
    main()
