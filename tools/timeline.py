"""Per-launch timeline of one step (library profiling events): start, duration, stream, kernel.

    python tools/timeline.py [log2D | C1] [fs]

log2D: workload H (SiLU pairs, N = 2^16) at D = 2^log2D (default 26); C1: the range-check config (ints, N = 2^8).
fs: Fiat-Shamir mode (challenges derived on the device).  Also prints the host wall time of the step.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2404_16109_b200 import zkl  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "26"
fs = len(sys.argv) > 2 and sys.argv[2] == "fs"
dev = torch.device("cuda", 0)
ctx = zkl.Context(0)
if arg == "C1":
    wl = W.range_check()
    D = wl.D
else:
    D = 1 << int(arg)
    wl = W.activation("H", D=D)
ctx.reserve(D, wl.N)
ch = wl.chal
chal = zkl.Context.challenges(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)
S, T, tmem = ctx.vec(D), ctx.vec(wl.N), ctx.table_mem(wl.N)
m = torch.empty(wl.N, dtype=torch.int32, device=dev)
if wl.kind == "pair":
    xd, yd = torch.from_numpy(wl.x).to(dev), torch.from_numpy(wl.y).to(dev)
    txd, tyd = torch.from_numpy(wl.tx).to(dev), torch.from_numpy(wl.ty).to(dev)
else:
    sd, td = torch.from_numpy(np.asarray(wl.s, np.int64)).to(dev), torch.from_numpy(np.asarray(wl.t, np.int64)).to(dev)


def step():
    if wl.kind == "pair":
        ctx.import_pair(txd, tyd, ch.alpha_f, T)
        tab = ctx.table(T, tmem)
        ctx.table_attach_pair(tab, txd, tyd, ch.alpha_f)   # pair-range fast path of prepare_pair
        ctx.prepare_pair(xd, yd, ch.alpha_f, D, tab, m=m, virtual_s=True)   # the bench step: S virtual
    else:
        ctx.import_ints(td, T)
        tab = ctx.table(T, tmem)
        ctx.import_ints(sd, S)
        ctx.prepare(S, D, tab, m)
    Sx = None if wl.kind == "pair" else S
    if fs:
        return ctx.prove_fs(Sx, D, tab, m, bytes(range(32)), zkl.PAPER)
    return ctx.prove(Sx, D, tab, m, chal)


for _ in range(2):
    step()
torch.cuda.synchronize()
ctx.set_profiling(True)
t0 = time.perf_counter()
step()
torch.cuda.synchronize()
wall = time.perf_counter() - t0
rec = ctx.profile_read(with_start=True)
print(f"wall {wall*1e3:.2f} ms  launches {len(rec)}")
for name, ms, st, tag in sorted(rec, key=lambda r: r[2]):
    print(f"{st:9.3f} {ms:8.3f}  {'main side aux low'.split()[tag]:4s} {name}")
