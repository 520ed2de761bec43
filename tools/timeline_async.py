"""Per-launch timeline of one H step in async mode (the bench's step): prepare_pair + prove enqueued together."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2404_16109_b200 import zkl  # noqa: E402

D = 1 << (int(sys.argv[1]) if len(sys.argv) > 1 else 26)
wl = W.activation("H", D=D)
dev = torch.device("cuda", 0)
ctx = zkl.Context(0)
ctx.reserve(D, wl.N)
ch = wl.chal
chal = zkl.Context.challenges(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)
xd, yd = torch.from_numpy(wl.x).to(dev), torch.from_numpy(wl.y).to(dev)
txd, tyd = torch.from_numpy(wl.tx).to(dev), torch.from_numpy(wl.ty).to(dev)
T, tmem = ctx.vec(wl.N), ctx.table_mem(wl.N)
m = torch.empty(wl.N, dtype=torch.int32, device=dev)


def step():
    ctx.import_pair(txd, tyd, ch.alpha_f, T)
    tab = ctx.table(T, tmem)
    ctx.table_attach_pair(tab, txd, tyd, ch.alpha_f)
    ctx.set_async(True)
    ctx.prepare_pair(xd, yd, ch.alpha_f, D, tab, m=m, virtual_s=True)   # the bench step: S virtual
    pf = ctx.prove(None, D, tab, m, chal)
    ctx.wait()
    ctx.set_async(False)
    return pf.result()


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
