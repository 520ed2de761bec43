"""Time the tlookup step on every BASELINE.json configuration on one GPU (for BASELINE.md §5).

A step = a1 (import) + a2 (table) + a3 (prepare) + a4-a9 (prove), inputs resident in HBM, CUDA events, warm-up 2.
C4 runs its K = 5 digit instances back to back as one step (value = 5 * 2^27 / time).
    python tools/bench_configs.py [C1 C2 C3 H C4 C5]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2404_16109_b200 import zkl  # noqa: E402


def run_instances(ctx, wls, steps=5, warmup=2):
    dev = torch.device("cuda", 0)
    Dmax = max(w.D for w in wls)
    Nmax = max(w.N for w in wls)
    ctx.reserve(Dmax, Nmax)
    prepared = []
    for wl in wls:
        if wl.kind == "pair":
            ins = (torch.from_numpy(np.ascontiguousarray(wl.x)).to(dev), torch.from_numpy(np.ascontiguousarray(wl.y)).to(dev),
                   torch.from_numpy(np.ascontiguousarray(wl.tx)).to(dev), torch.from_numpy(np.ascontiguousarray(wl.ty)).to(dev))
        else:
            ins = (torch.from_numpy(np.asarray(wl.s, np.int64)).to(dev), torch.from_numpy(np.asarray(wl.t, np.int64)).to(dev))
        ch = wl.chal
        prepared.append((wl, ins, zkl.Context.challenges(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r), ctx.vec(wl.D),
                         ctx.vec(wl.N), ctx.table_mem(wl.N), torch.empty(wl.N, dtype=torch.int32, device=dev)))

    def step():
        for wl, ins, chal, S, T, tmem, m in prepared:
            if wl.kind == "pair":
                ctx.import_pair(ins[2], ins[3], wl.chal.alpha_f, T)
                tab = ctx.table(T, tmem)
                ctx.table_attach_pair(tab, ins[2], ins[3], wl.chal.alpha_f)   # pair-range fast path of prepare_pair
                ctx.prepare_pair(ins[0], ins[1], wl.chal.alpha_f, wl.D, tab, S, m)
            else:
                ctx.import_ints(ins[1], T)
                tab = ctx.table(T, tmem)
                ctx.import_ints(ins[0], S)
                ctx.prepare(S, wl.D, tab, m)
            ctx.prove(S, wl.D, tab, m, chal)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    total = sum(w.D for w in wls)
    return ms, total / (ms / 1e3)


def main(names):
    ctx = zkl.Context(0)
    out = []
    for name in names:
        t0 = time.time()
        if name == "C1":
            wls = [W.range_check()]
        elif name == "C4":
            wls = [W.zkattn_digits(k) for k in range(5)]
        else:
            wls = [W.activation({"C2": "2", "C3": "3", "H": "H", "C5": "5"}[name])]
        gen = time.time() - t0
        ms, lps = run_instances(ctx, wls, steps=3 if name in ("C4", "C5") else 5)
        rec = {"config": name, "lookups": sum(w.D for w in wls), "ms_per_step": ms, "lookups_per_s": lps,
               "instances": len(wls), "gen_s": gen}
        print(json.dumps(rec), flush=True)
        out.append(rec)
        del wls
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "C3", "H", "C4", "C5"])
