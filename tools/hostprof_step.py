import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import workloads as W
from paper_2404_16109_b200 import zkl
dev = torch.device("cuda", 0)
wl = W.activation("H", D=1 << 26)
D = wl.D
stream = torch.cuda.Stream(device=dev)
torch.cuda.set_stream(stream)
ctx = zkl.Context(0, stream=stream)
ctx.reserve(D, wl.N)
ch = wl.chal
chal = zkl.Context.challenges(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)
xd, yd = torch.from_numpy(wl.x).to(dev), torch.from_numpy(wl.y).to(dev)
txd, tyd = torch.from_numpy(wl.tx).to(dev), torch.from_numpy(wl.ty).to(dev)
T = ctx.vec(wl.N); tmem = ctx.table_mem(wl.N)
m = torch.empty(wl.N, dtype=torch.int32, device=dev)
def step(t):
    t.append(time.perf_counter()); ctx.import_pair(txd, tyd, ch.alpha_f, T)
    t.append(time.perf_counter()); tab = ctx.table(T, tmem)
    t.append(time.perf_counter()); ctx.table_attach_pair(tab, txd, tyd, ch.alpha_f)
    t.append(time.perf_counter()); ctx.set_async(True)
    ctx.prepare_pair(xd, yd, ch.alpha_f, D, tab, m=m, virtual_s=True)
    t.append(time.perf_counter()); pending = ctx.prove(None, D, tab, m, chal)
    t.append(time.perf_counter()); ctx.wait()
    t.append(time.perf_counter()); ctx.set_async(False); pending.result()
    t.append(time.perf_counter())
for _ in range(3): step([])
torch.cuda.synchronize()
for _ in range(3):
    t = []
    step(t)
    names = ["import_pair", "table", "attach", "prepare_pair", "prove", "wait", "result"]
    print(" ".join(f"{n}={(t[i+1]-t[i])*1e3:.3f}" for i, n in enumerate(names)), f"total={(t[-1]-t[0])*1e3:.3f}")
