"""Per-launch timeline of one H step (profiling events): name, stream order, start, duration."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from paper_2404_16109_b200 import zkl

log2d = int(sys.argv[1]) if len(sys.argv) > 1 else 26
fs = len(sys.argv) > 2 and sys.argv[2] == "fs"   # Fiat-Shamir mode (challenges derived on the device)
D = 1 << log2d
wl = W.activation("H", D=D)
dev = torch.device("cuda", 0)
ctx = zkl.Context(0)
ctx.reserve(D, wl.N)
ch = wl.chal
chal = zkl.Context.challenges(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)
xd, yd = torch.from_numpy(wl.x).to(dev), torch.from_numpy(wl.y).to(dev)
txd, tyd = torch.from_numpy(wl.tx).to(dev), torch.from_numpy(wl.ty).to(dev)
S, T, tmem = ctx.vec(D), ctx.vec(wl.N), ctx.table_mem(wl.N)
m = torch.empty(wl.N, dtype=torch.int32, device=dev)
def step():
    ctx.import_pair(txd, tyd, ch.alpha_f, T)
    tab = ctx.table(T, tmem); ctx.prepare_pair(xd, yd, ch.alpha_f, D, tab, S, m)
    if fs:
        return ctx.prove_fs(S, D, tab, m, bytes(range(32)), zkl.PAPER)
    return ctx.prove(S, D, tab, m, chal)
for _ in range(2): step()
torch.cuda.synchronize()
ctx.set_profiling(True)
t0 = time.perf_counter(); step(); torch.cuda.synchronize(); wall = time.perf_counter() - t0
rec = ctx.profile_read(with_start=True)
print(f"wall {wall*1e3:.2f} ms  launches {len(rec)}")
for name, ms, st, tag in sorted(rec, key=lambda r: r[2]):
    print(f"{st:9.3f} {ms:8.3f}  {'main side aux'.split()[tag]:4s} {name}")
