"""Two proofs in flight on one GPU (two contexts, two streams, two host threads), the bench step on each:
aggregate lookups/s against one context stepping alone.  Timed with CUDA events on the device.

    python tools/bench_inflight.py [steps]
"""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2404_16109_b200 import zkl  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 10
dev = torch.device("cuda", 0)
wl = W.activation("H", D=1 << 26)
D = wl.D
ch = wl.chal
chal = zkl.Context.challenges(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)
xd, yd = torch.from_numpy(wl.x).to(dev), torch.from_numpy(wl.y).to(dev)
txd, tyd = torch.from_numpy(wl.tx).to(dev), torch.from_numpy(wl.ty).to(dev)


class Lane:
    def __init__(self):
        self.stream = torch.cuda.Stream(device=dev)
        self.ctx = zkl.Context(0, stream=self.stream)
        self.ctx.reserve(D, wl.N)
        self.T = self.ctx.vec(wl.N)
        self.tmem = self.ctx.table_mem(wl.N)
        self.m = torch.empty(wl.N, dtype=torch.int32, device=dev)

    def step(self):
        c = self.ctx
        c.import_pair(txd, tyd, ch.alpha_f, self.T)
        tab = c.table(self.T, self.tmem)
        c.table_attach_pair(tab, txd, tyd, ch.alpha_f)
        c.set_async(True)
        c.prepare_pair(xd, yd, ch.alpha_f, D, tab, m=self.m, virtual_s=True)
        pend = c.prove(None, D, tab, self.m, chal)
        c.wait()
        c.set_async(False)
        return pend.result()


lanes = [Lane(), Lane()]
ref = lanes[0].step()
for ln in lanes:
    for _ in range(3):
        assert ln.step().evals == ref.evals
torch.cuda.synchronize()


def timed(nl):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    done = [torch.cuda.Event() for _ in range(nl)]
    e0.record(lanes[0].stream)
    for ln in lanes[1:nl]:
        ln.stream.wait_event(e0)

    def run(i):
        with torch.cuda.stream(lanes[i].stream):
            for _ in range(K):
                lanes[i].step()
            done[i].record(lanes[i].stream)

    th = [threading.Thread(target=run, args=(i,)) for i in range(nl)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for i in range(1, nl):
        lanes[0].stream.wait_event(done[i])
    e1.record(lanes[0].stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return ms, nl * K * D / (ms / 1e3)


for nl in (1, 2, 1, 2):
    ms, v = timed(nl)
    print(f"lanes={nl} total_ms={ms:.2f} ms_per_step={ms / (nl * K):.3f} lookups_per_s={v:.4e}")
