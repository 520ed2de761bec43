"""Time the tlookup step on every BASELINE.json configuration on one GPU (for BASELINE.md §5).

A step = a1 (import) + a2 (table) + a3 (prepare) + a4-a9 (prove), inputs resident in HBM, CUDA events, warm-up 2.
C4 runs its K = 5 digit instances (32 heads each) in flight together as one step (value = 5 * 2^27 / time).
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


def run_instances(wls, steps=5, warmup=2):
    """The bench step on every instance: import T, table (+ pair-range attachment), prepare_pair with a virtual S
    (range lookups as pairs with y = 0: T = [0, 2^16) + alpha * 0), prove.  Several instances are kept in flight on
    their own contexts and streams (async mode): instance i+1's setup overlaps instance i's proof."""
    dev = torch.device("cuda", 0)
    prepared = []
    for wl in wls:
        st = torch.cuda.Stream(device=dev)
        ctx = zkl.Context(0, stream=st)
        ctx.reserve(wl.D, wl.N)
        if wl.kind == "pair":
            x, y, tx, ty = wl.x, wl.y, wl.tx, wl.ty
        else:   # a range lookup: S = x + alpha * 0 over T = t + alpha * 0
            x = np.asarray(wl.s, np.int32)
            y = np.zeros_like(x)
            tx = np.asarray(wl.t, np.int32)
            ty = np.zeros_like(tx)
        ins = tuple(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (x, y, tx, ty))
        ch = wl.chal
        prepared.append((ctx, st, wl, ins, zkl.Context.challenges(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r),
                         ctx.vec(wl.N), ctx.table_mem(wl.N), torch.empty(wl.N, dtype=torch.int32, device=dev)))

    def step():
        pend = []
        for ctx, st, wl, ins, chal, T, tmem, m in prepared:
            ctx.import_pair(ins[2], ins[3], wl.chal.alpha_f, T)
            tab = ctx.table(T, tmem)
            ctx.table_attach_pair(tab, ins[2], ins[3], wl.chal.alpha_f)
            ctx.set_async(True)
            ctx.prepare_pair(ins[0], ins[1], wl.chal.alpha_f, wl.D, tab, m=m, virtual_s=True)
            pend.append((ctx, ctx.prove(None, wl.D, tab, m, chal), tab))
        for ctx, p, _ in pend:
            ctx.wait()
            ctx.set_async(False)
        return [p.result() for _, p, _ in pend]

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    streams = [p[1] for p in prepared]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    for s_ in streams[1:]:
        s_.wait_event(e0)
    for _ in range(steps):
        step()
    for s_ in streams[1:]:
        ev = torch.cuda.Event()
        ev.record(s_)
        streams[0].wait_event(ev)
    e1.record(streams[0])
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    for p in prepared:
        p[0].close()
    total = sum(w.D for w in wls)
    return ms, total / (ms / 1e3)


def main(names):
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
        ms, lps = run_instances(wls, steps=3 if name in ("C4", "C5") else 5)
        rec = {"config": name, "lookups": sum(w.D for w in wls), "ms_per_step": ms, "lookups_per_s": lps,
               "instances": len(wls), "gen_s": gen}
        print(json.dumps(rec), flush=True)
        out.append(rec)
        del wls
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "C3", "H", "C4", "C5"])
